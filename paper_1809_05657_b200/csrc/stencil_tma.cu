// stencil_tma.cu — TMA-ring 2-D stencils (the user kernels of configs[2], P:L462 as
// read in DESIGN R12, and the Jacobi of configs[1], P:L459 / R11) for a device's work box.
//
// Persistent, warp-specialised CTAs (2 per SM).  A tile is up to RB output rows x CW
// output columns of the box.  One producer lane streams the tile's RB+2 input rows
// through an NST-stage shared-memory ring as 2-D TMA boxes of RS rows x 256 columns
// (cp.async.bulk.tensor, mbarrier complete_tx); the box origin sits 16 bytes left of
// the strip, so every output column's horizontal neighbours are in the same smem row.
// Eight consumer warps march down the rows, one output column per thread, holding the
// two rows above in registers: 3 shared loads per point, no shuffles, no edge loads,
// no global loads on the compute path.  The tile sequence runs row-block-major over the
// persistent grid, so the strips and row blocks in flight at any moment are neighbours
// and their overlapping halo columns/rows hit L2.
//
// Operand order is the oracle's: JACOBI5 ((W+E)+N)+S then *0.25;
// STENCIL9 e=((W+E)+N)+S, c=((NW+NE)+SW)+SE, (4e+c)/20 — results are bit-identical
// to the register-march kernels in kernels.cu and to the oracle.
//
// Measured (tools/stencil_tma_tune.cu): with nvcc's IEEE fp64 division (the reciprocal
// of 20 rebuilt per point) the register-march 9-point kernel was latency-bound and this
// one ran up to 12-20% faster standalone; once the division uses a constant reciprocal
// (divc.cuh) the register march is ahead (0.873 vs 0.78 of HBM at N=1), so this kernel
// is opt-in: HDA_TMA=1 (9-point), 2 (both).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "divc.cuh"
#include "kernels.cuh"
#include "sync.cuh"
#include "tcgen05_common.cuh"

namespace hda {
namespace stma {

constexpr int BOXW = 256;                   // smem row = TMA box width (elements, the TMA maximum)
constexpr int NCONS = 8;                    // consumer warps
constexpr int THREADS = (NCONS + 1) * 32;  // + one producer warp
constexpr int RS = 8;                       // rows per stage (one TMA box)
constexpr int NST = 4;                      // ring stages
constexpr int MINB = 2;                     // CTAs per SM

template <typename T>
struct Geo {
  static constexpr int A = 16 / (int)sizeof(T);            // box origin: 16 bytes left of the strip
  static constexpr int CW = sizeof(T) == 8 ? 252 : 248;     // output columns per strip (32-byte multiple)
  static constexpr int ALIGN = 32 / (int)sizeof(T);         // strip base alignment (elements)
};

struct Tiles {
  int64_t r0, r1, c0, c1, cb;
  int32_t nstrip, nrb, spt;  // strips, row blocks, stages per tile (RB = spt*RS - 2)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// bounded wait: a protocol fault ends in the sticky error flag (HDA_ETIMEOUT) and wrong
// results that the parity tests catch, never in a hung GPU
__device__ __forceinline__ bool mbar_wait(uint64_t* b, uint32_t parity, const KSync& ks) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (ok) return true;
    if (clock64() - t0 > (1LL << 34)) {  // ~8 s
      if (ks.err) *reinterpret_cast<volatile int*>(ks.err) = -7;
      return false;
    }
  }
}

template <typename T>
__device__ __forceinline__ T st9(T w, T e, T n, T s, T nw, T ne, T sw, T se) {
  T a = ((w + e) + n) + s;
  T c = ((nw + ne) + sw) + se;
  T t = T(4) * a;
  t = t + c;
  return div20(t);
}

template <typename T, int KIND>
__global__ void __launch_bounds__(THREADS, MINB)
    stencil2d_tma_kernel(const __grid_constant__ CUtensorMap map, T* __restrict__ out, int64_t ld,
                         const __grid_constant__ Tiles tt, const __grid_constant__ KSync ks) {
  constexpr int A = Geo<T>::A, CW = Geo<T>::CW;
  pdl_enter();
  ks_pre(ks);  // WAR: peers finished reading the cells this launch overwrites
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);  // shared address space kept: LDS, not generic loads
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)NST * RS * BOXW * sizeof(T));
  uint64_t* empty = full + NST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
  }
  __syncthreads();
  const int64_t ntiles = (int64_t)tt.nstrip * tt.nrb;
  const int RB = tt.spt * RS - 2;
  if (warp == NCONS) {
    if (lane == 0) {  // producer
      int slot = 0;
      uint32_t ph = 0;
      bool ok = true;
      for (int64_t t = blockIdx.x; t < ntiles && ok; t += gridDim.x) {
        const int64_t rb = t / tt.nstrip, s = t - rb * tt.nstrip;
        const int x = (int)(tt.cb + s * CW - A);
        const int y = (int)(tt.r0 + rb * RB - 1);
        for (int j = 0; j < tt.spt && ok; j++) {
          ok = mbar_wait(&empty[slot], ph ^ 1, ks);
          mbar_expect_tx(&full[slot], RS * BOXW * sizeof(T));
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
              "[%2];" ::"r"(smem_u32(ring + slot * RS * BOXW)),
              "l"(&map), "r"(smem_u32(&full[slot])), "r"(x), "r"(y + j * RS)
              : "memory");
          if (++slot == NST) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else {
    int slot = 0;
    uint32_t ph = 0;
    bool ok = true;
    for (int64_t t = blockIdx.x; t < ntiles && ok; t += gridDim.x) {
      const int64_t rb = t / tt.nstrip, s = t - rb * tt.nstrip;
      const int64_t col = tt.cb + s * CW + tid;
      const bool live = tid < CW && col >= tt.c0 && col < tt.c1;
      const int64_t row0 = tt.r0 + (int64_t)rb * RB;  // output row of input row 2
      const int rem = (int)min((int64_t)RB, tt.r1 - row0);
      T* op = out + row0 * ld + col;
      T u0 = 0, u1 = 0, u2 = 0, c0 = 0, c1 = 0, c2 = 0;
#pragma unroll 1
      for (int j = 0; j < tt.spt; j++) {
        ok = mbar_wait(&full[slot], ph, ks);
        const T* base = ring + slot * RS * BOXW + tid + A - 1;
#pragma unroll
        for (int k = 0; k < RS; k++) {
          const int i = j * RS + k;
          const T d0 = base[k * BOXW], d1 = base[k * BOXW + 1], d2 = base[k * BOXW + 2];
          if (i >= 2) {
            T o;
            if (KIND == 0)
              o = (((c0 + c2) + u1) + d1) * T(0.25);
            else
              o = st9<T>(c0, c2, u1, d1, u0, u2, d0, d2);
            if (live && i - 2 < rem) *op = o;
            op += ld;
          }
          u0 = c0, u1 = c1, u2 = c2;
          c0 = d0, c1 = d1, c2 = d2;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == NST) {
          slot = 0;
          ph ^= 1;
        }
      }
    }
  }
  ks_post(ks);
}

// one tensor map per (replica, shape, dtype): encoding costs host time, and the
// ping-pong sweeps alternate between two replicas
struct MapKey {
  const void* p;
  int64_t ld, rows;
  int dtype;
  bool operator==(const MapKey& o) const { return p == o.p && ld == o.ld && rows == o.rows && dtype == o.dtype; }
};
struct MapHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.p) ^ (size_t)(k.ld * 1000003) ^ (size_t)(k.rows * 7919) ^ (size_t)k.dtype;
  }
};
static bool get_map(const void* in, int64_t ld, int64_t rows, int dtype, CUtensorMap* out) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapHash> cache;
  const MapKey key{in, ld, rows, dtype};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  tcc::EncodeTiled enc = tcc::get_encode();
  if (!enc) return false;
  const size_t es = dtype == 0 ? 8 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {BOXW, RS};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  CUresult r = enc(&m, dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(in), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  if (cache.size() > 256) cache.clear();
  cache[key] = m;
  *out = m;
  return true;
}

static int sm_count() {
  static const int n = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v > 0 ? v : 148;
  }();
  return n;
}

template <typename T, int KIND>
static cudaError_t launch_t(const T* in, T* out, const int64_t* shape, const int64_t* lb, const int64_t* ub,
                            const KSync& ks, cudaStream_t s) {
  constexpr int CW = Geo<T>::CW;
  const int64_t ld = shape[2], rows = shape[1];
  Tiles tt;
  tt.r0 = lb[1];
  tt.r1 = ub[1];
  tt.c0 = lb[2];
  tt.c1 = ub[2];
  tt.cb = tt.c0 - tt.c0 % Geo<T>::ALIGN;
  tt.nstrip = (int)((tt.c1 - tt.cb + CW - 1) / CW);
  const size_t smem = (size_t)NST * RS * BOXW * sizeof(T) + 2 * NST * sizeof(uint64_t);
  // the shared-memory opt-in is per device (launches may come from one thread per GPU)
  static std::atomic<int> attr_done[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorNotSupported;
  if (!attr_done[dev].load(std::memory_order_acquire)) {
    if (cudaFuncSetAttribute(stencil2d_tma_kernel<T, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return cudaErrorNotSupported;
    attr_done[dev].store(1, std::memory_order_release);
  }
  const int64_t grid_max = (int64_t)sm_count() * MINB;
  // tile height: the stage count per tile that minimises the busiest CTA's rows
  // (ceil(tiles / grid) * rows per tile), so small shares still balance
  const int64_t R = tt.r1 - tt.r0;
  int best = 2;
  int64_t best_cost = INT64_MAX;
  for (int spt = 2; spt <= 16; spt++) {
    const int64_t rb = (int64_t)spt * RS - 2;
    const int64_t tiles = (int64_t)tt.nstrip * ((R + rb - 1) / rb);
    const int64_t cost = ((tiles + grid_max - 1) / grid_max) * (rb + 2);
    if (cost < best_cost) {
      best_cost = cost;
      best = spt;
    }
  }
  tt.spt = best;
  const int64_t RB = (int64_t)best * RS - 2;
  tt.nrb = (int)((R + RB - 1) / RB);
  CUtensorMap map;
  if (!get_map(in, ld, rows, sizeof(T) == 8 ? 0 : 1, &map)) return cudaErrorNotSupported;
  const int64_t grid = std::min<int64_t>(grid_max, (int64_t)tt.nstrip * tt.nrb);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  static const int pdl = [] {
    const char* e = std::getenv("HDA_PDL");
    return e ? std::atoi(e) : 1;
  }();
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, stencil2d_tma_kernel<T, KIND>, map, out, ld, tt, ks);
}

}  // namespace stma

// HDA_TMA: 0 (default) = off, 1 = TMA ring for the 9-point kernel, 2 = 9-point and
// Jacobi.  With the constant-reciprocal division (divc.cuh) the register march is ahead
// for the 9-point too: 357.5-357.7 vs 320.2-320.9 GPoints/s at N=1, 691.9 vs 629.6-632.7
// at N=2 (profiles/r02/div20/)
int stencil_tma_mode() {
  static const int v = [] {
    const char* e = std::getenv("HDA_TMA");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

cudaError_t launch_stencil2d_tma(int kind, int dtype, const void* in, void* out, const int64_t* shape,
                                 const int64_t* lb, const int64_t* ub, const KSync& ks, cudaStream_t s) {
  const int es = dtype == 0 ? 8 : 4;
  if (dtype != 0 && dtype != 1) return cudaErrorNotSupported;
  if (shape[0] != 1 || lb[0] != 0 || ub[0] != 1) return cudaErrorNotSupported;
  if (ub[1] - lb[1] < 32 || ub[2] - lb[2] < 128) return cudaErrorNotSupported;  // thin strips: register march
  if ((uintptr_t)in % 16 || (shape[2] * es) % 16 || shape[2] >= (1LL << 31) || shape[1] >= (1LL << 31))
    return cudaErrorNotSupported;
  if (kind == 0) {
    return dtype == 0 ? stma::launch_t<double, 0>((const double*)in, (double*)out, shape, lb, ub, ks, s)
                      : stma::launch_t<float, 0>((const float*)in, (float*)out, shape, lb, ub, ks, s);
  }
  return dtype == 0 ? stma::launch_t<double, 1>((const double*)in, (double*)out, shape, lb, ub, ks, s)
                    : stma::launch_t<float, 1>((const float*)in, (float*)out, shape, lb, ub, ks, s);
}

}  // namespace hda
