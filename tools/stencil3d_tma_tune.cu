// stencil3d_tma_tune.cu — standalone timing of a TMA-ring fp32 3-D 7-point design on
// 1024^3 (configs[4] 3-D half) against a scalar reference; not part of the library.
//
// Tile = BW-column strip x BH-row block x ZC-plane chunk.  A producer lane streams the
// tile's ZC+2 planes, each a (BH+2) x (BW+8) TMA box (origin 4 columns left of the
// strip, 1 row above), through an NST-stage smem ring.  Consumer thread = one column x
// RPT rows, marching z with planes z-1, z, z+1 of its rows in registers; x and y
// neighbours from the current plane's stage.
//     nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//          tools/stencil3d_tma_tune.cu -o tools/stencil3d_tma_tune -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e = (x);                                               \
    if (e != cudaSuccess) {                                            \
      printf("CUDA %s at line %d\n", cudaGetErrorString(e), __LINE__); \
      exit(1);                                                         \
    }                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
}

struct T3 {
  long z0, z1, y0, y1, x0, x1, xb;  // work box, strip base
  int nsx, nby, nbz, zc;            // strips, row blocks, z chunks, planes per chunk
};

template <int BW, int BH, int RPT, int NST, int MINB, int TX = BW>
__global__ void __launch_bounds__(TX * (BH / RPT) + 32, MINB)
    k_tma3(const __grid_constant__ CUtensorMap map, float* __restrict__ out, long n1, long n2, const __grid_constant__ T3 t3) {
  constexpr int PW = BW + 8;  // smem row pitch (elements) = box width
  constexpr int NCONS = TX * (BH / RPT);
  constexpr int SROWS = BH + 2;
  constexpr int SSTR = (SROWS * PW + 31) / 32 * 32;  // stage stride: 128-byte aligned TMA destinations
  extern __shared__ __align__(128) float ring[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NST * SSTR);
  uint64_t* empty = full + NST;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
  }
  __syncthreads();
  const long ntiles = (long)t3.nsx * t3.nby * t3.nbz;
  const long pl = n1 * n2;
  if (tid >= NCONS) {
    if (tid == NCONS) {
      int slot = 0;
      uint32_t ph = 0;
      for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long sx = t % t3.nsx, r = t / t3.nsx, by = r % t3.nby, bz = r / t3.nby;
        const int x = (int)(t3.xb + sx * BW - 4), y = (int)(t3.y0 + by * BH - 1);
        const long zs = t3.z0 + bz * t3.zc, ze = min(zs + t3.zc, t3.z1);
        for (long z = zs - 1; z <= ze; z++) {
          mbar_wait(&empty[slot], ph ^ 1);
          mbar_expect_tx(&full[slot], SROWS * PW * 4);
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
              "[%2];" ::"r"(smem_u32(ring + slot * SSTR)),
              "l"(&map), "r"(smem_u32(&full[slot])), "r"(x), "r"(y), "r"((int)z)
              : "memory");
          if (++slot == NST) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }
  const int lane = tid & 31, col = tid % TX, rg = tid / TX;  // column, row group
  int slot = 0;
  uint32_t ph = 0;
  auto advance = [&]() {
    if (++slot == NST) {
      slot = 0;
      ph ^= 1;
    }
  };
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long sx = t % t3.nsx, r = t / t3.nsx, by = r % t3.nby, bz = r / t3.nby;
    const long x = t3.xb + sx * BW + col;
    const long yb = t3.y0 + by * BH + rg * RPT;  // first output row of this thread
    const long zs = t3.z0 + bz * t3.zc, ze = min(zs + t3.zc, t3.z1);
    const bool xl = col < BW && x >= t3.x0 && x < t3.x1;
    const int nr = (int)min((long)RPT, t3.y1 - yb);  // live rows (may be <= 0)
    float zm[RPT], zc[RPT], zp[RPT];
    // plane zs-1
    mbar_wait(&full[slot], ph);
    {
      const float* st = ring + slot * SSTR + (rg * RPT + 1) * PW + col + 4;
#pragma unroll
      for (int i = 0; i < RPT; i++) zm[i] = st[i * PW];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    advance();
    mbar_wait(&full[slot], ph);
    int cur = slot;
    uint32_t cph = ph;
    (void)cph;
    {
      const float* st = ring + cur * SSTR + (rg * RPT + 1) * PW + col + 4;
#pragma unroll
      for (int i = 0; i < RPT; i++) zc[i] = st[i * PW];
    }
    advance();
    float* op = out + zs * pl + yb * n2 + x;
    for (long z = zs; z < ze; z++) {
      mbar_wait(&full[slot], ph);  // plane z+1
      {
        const float* st = ring + slot * SSTR + (rg * RPT + 1) * PW + col + 4;
#pragma unroll
        for (int i = 0; i < RPT; i++) zp[i] = st[i * PW];
      }
      const float* st = ring + cur * SSTR + (rg * RPT) * PW + min(col, BW - 1) + 4;  // row above the first
      float up = st[0];
      float o[RPT];
#pragma unroll
      for (int i = 0; i < RPT; i++) {
        const float* rr = st + (i + 1) * PW;
        const float dn = i + 1 < RPT ? zc[i + 1] : rr[PW];
        float s = rr[-1] + rr[1];
        s = s + up;
        s = s + dn;
        s = s + zm[i];
        s = s + zp[i];
        o[i] = s / 6.0f;
        up = zc[i];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[cur]);  // plane z done
      if (xl) {
#pragma unroll
        for (int i = 0; i < RPT; i++)
          if (i < nr) op[i * n2] = o[i];
      }
      op += pl;
#pragma unroll
      for (int i = 0; i < RPT; i++) {
        zm[i] = zc[i];
        zc[i] = zp[i];
      }
      cur = slot;
      advance();
    }
    // plane ze's stage was waited (as z+1 of the last step) but not released
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[cur]);
  }
}

__global__ void k_ref(const float* __restrict__ in, float* __restrict__ out, long n1, long n2, long z0, long y0,
                      long y1, long x0, long x1) {
  const long x = x0 + (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long y = y0 + blockIdx.y, z = z0 + blockIdx.z;
  if (x < x1 && y < y1) {
    const long pl = n1 * n2;
    const float* p = in + z * pl + y * n2 + x;
    float s = p[-1] + p[1];
    s = s + p[-n2];
    s = s + p[n2];
    s = s + p[-pl];
    s = s + p[pl];
    out[z * pl + y * n2 + x] = s / 6.0f;
  }
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 1024;
  const size_t bytes = (size_t)n * n * n * 4;
  float *X, *Y, *R;
  CK(cudaMalloc(&X, bytes));
  CK(cudaMalloc(&Y, bytes));
  CK(cudaMalloc(&R, bytes));
  std::vector<float> h((size_t)n * n * n);
  for (size_t i = 0; i < h.size(); i++) h[i] = (float)((i * 2654435761u) % 1000) / 1000.0f;
  CK(cudaMemcpy(X, h.data(), bytes, cudaMemcpyHostToDevice));
  const long lo = 1, hi = n - 1;
  const double alg = (double)(hi - lo) * (hi - lo) * (hi - lo) * 8;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeTiled enc = (EncodeTiled)fn;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> o(h.size()), ref(h.size());
  CK(cudaMemset(R, 0, bytes));
  {
    dim3 g((unsigned)((hi - lo + 127) / 128), (unsigned)(hi - lo), (unsigned)(hi - lo));
    k_ref<<<g, 128>>>(X, R, n, n, lo, lo, hi, lo, hi);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(ref.data(), R, bytes, cudaMemcpyDeviceToHost));
  }
  auto time_it = [&](const char* name, auto launch) {
    CK(cudaMemset(Y, 0, bytes));
    launch();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(o.data(), Y, bytes, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (size_t i = 0; i < o.size(); i++) bad += o[i] != ref[i] ? 1 : 0;  // ghost ring: 0 in both (memset)
    for (int i = 0; i < 3; i++) launch();
    CK(cudaDeviceSynchronize());
    const int it = 20;
    cudaEventRecord(a);
    for (int i = 0; i < it; i++) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / it;
    printf("%-44s %9.1f us  %7.1f GB/s  mismatches=%ld\n", name, us, alg / us / 1e3, bad);
  };
#define TMA3(BW, BH, RPT, NST, MINB, ZC) TMA3X(BW, BH, RPT, NST, MINB, ZC, BW)
#define TMA3X(BW, BH, RPT, NST, MINB, ZC, TX)                                                                         \
  {                                                                                                              \
    CUtensorMap m;                                                                                               \
    cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)n};                                          \
    cuuint64_t str[2] = {(cuuint64_t)n * 4, (cuuint64_t)n * n * 4};                                              \
    cuuint32_t box[3] = {BW + 8, BH + 2, 1}, es[3] = {1, 1, 1};                                                  \
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,        \
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != \
        CUDA_SUCCESS) {                                                                                          \
      printf("encode failed\n");                                                                                 \
      exit(1);                                                                                                   \
    }                                                                                                            \
    T3 t3;                                                                                                       \
    t3.z0 = lo, t3.z1 = hi, t3.y0 = lo, t3.y1 = hi, t3.x0 = lo, t3.x1 = hi, t3.xb = 0;                           \
    t3.nsx = (int)((hi - t3.xb + BW - 1) / BW);                                                                  \
    t3.nby = (int)((hi - lo + BH - 1) / BH);                                                                     \
    t3.zc = ZC;                                                                                                  \
    t3.nbz = (int)((hi - lo + ZC - 1) / ZC);                                                                     \
    const size_t smem = (size_t)NST * (((BH + 2) * (BW + 8) + 31) / 32 * 32) * 4 + 2 * NST * 8;                                     \
    auto kf = k_tma3<BW, BH, RPT, NST, MINB, TX>;                                                                    \
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));                       \
    int occ = 0;                                                                                                 \
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kf, TX * (BH / RPT) + 32, smem));                    \
    const long tiles = (long)t3.nsx * t3.nby * t3.nbz;                                                           \
    const unsigned grid = (unsigned)std::min<long>(tiles, (long)sms * occ);                                      \
    char nm[128];                                                                                                \
    snprintf(nm, sizeof nm, "tma3 BW%d TX%d BH%d RPT%d NST%d minB%d ZC%d occ%d", BW, TX, BH, RPT, NST, MINB, ZC, occ);    \
    time_it(nm, [&] { kf<<<grid, TX * (BH / RPT) + 32, smem>>>(m, Y, n, n, t3); });                               \
  }
  TMA3(128, 32, 16, 4, 2, 64);
  TMA3(128, 32, 16, 5, 1, 64);
  TMA3(128, 32, 16, 6, 1, 64);
  TMA3(128, 64, 32, 3, 1, 64);
  TMA3X(248, 16, 16, 4, 2, 64, 256);
  TMA3X(248, 16, 16, 5, 2, 64, 256);
  TMA3X(248, 32, 32, 3, 1, 64, 256);
  TMA3X(248, 16, 8, 4, 1, 64, 256);
  TMA3(128, 32, 16, 4, 2, 256);
  {
    cudaEventRecord(a);
    for (int i = 0; i < 10; i++) cudaMemcpyAsync(Y, X, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-44s %9.1f us  %7.1f GB/s\n", "cudaMemcpy D2D", ms * 1e3 / 10, 2.0 * bytes / (ms * 1e-3 / 10) / 1e9);
  }
  return 0;
}
