// kernels.cu — sm_100a kernels of the exchange path and the user kernels.
//
//  copy_runs_kernel   strided-rect raw copy: fused pull (peer replica -> local replica
//                     over NVLink = pack + transfer + unpack), pack, unpack, COPY
//  wait / signal      cross-device ordering words (spin with timeout / release store)
//  jacobi5            P:L459 A = (((W+E)+N)+S) * 0.25
//  stencil9           reading R12: (4*(((W+E)+N)+S) + (((NW+NE)+SW)+SE)) / 20
//  stencil7           reading R13: (((((x-+x+)+y-)+y+)+z-)+z+) / 6
//  scale, stamp       elementwise helpers (repartition kernel, test kernel)
//
// Shapes/boxes passed to the user-kernel launchers are FRONT-padded to 3-D so that
// dimension 2 is always the contiguous one.
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <cstdlib>
#include <utility>

#include "divc.cuh"
#include "kernels.cuh"
#include "sync.cuh"

namespace hda {

// =====================================================================================
// strided rectangle copy
// =====================================================================================

// NVLink pulls are latency-bound unless enough bytes are in flight: aim for >= ~8
// warps per SM (148 x 8 units), chunks between 512 B and 8 KiB
int64_t pick_chunk_bytes(int64_t total_bytes) {
  int64_t c = total_bytes / (148 * 8);
  c = (c + 511) & ~(int64_t)511;
  if (c < 512) c = 512;
  if (c > kChunkBytes) c = kChunkBytes;
  return c;
}

int64_t run_desc_units(RunDesc& d, int64_t chunk_bytes) {
  int64_t runs = (int64_t)d.n0 * d.n1;
  d.chunk_bytes = chunk_bytes;
  if (runs == 0 || d.run_bytes == 0) {
    d.chunks = 1;
    return 0;
  }
  if (d.run_bytes <= 64) {
    d.chunks = 0;
    return (runs + 31) / 32;
  }
  d.chunks = (int32_t)((d.run_bytes + chunk_bytes - 1) / chunk_bytes);
  return runs * d.chunks;
}

__device__ __forceinline__ void copy_elem(char* d, const char* s, int es) {
  switch (es) {
    case 8: *reinterpret_cast<unsigned long long*>(d) = *reinterpret_cast<const unsigned long long*>(s); break;
    case 4: *reinterpret_cast<unsigned int*>(d) = *reinterpret_cast<const unsigned int*>(s); break;
    case 2: *reinterpret_cast<unsigned short*>(d) = *reinterpret_cast<const unsigned short*>(s); break;
    default: *d = *s;
  }
}

// one warp moves n bytes; 16-byte vectors when src and dst share the 16-byte phase
__device__ __forceinline__ void warp_copy(char* d, const char* s, int64_t n, int es, int lane) {
  if ((((uintptr_t)s ^ (uintptr_t)d) & 15) == 0) {
    int64_t head = (16 - ((uintptr_t)s & 15)) & 15;
    if (head > n) head = n;
    for (int64_t i = (int64_t)lane * es; i < head; i += 32 * es) copy_elem(d + i, s + i, es);
    const uint4* s4 = reinterpret_cast<const uint4*>(s + head);
    uint4* d4 = reinterpret_cast<uint4*>(d + head);
    const int64_t nv = (n - head) >> 4;
    int64_t i = lane;
    for (; i + 96 < nv; i += 128) {  // four 16-byte loads in flight per lane
      uint4 a = s4[i], b = s4[i + 32], c = s4[i + 64], e = s4[i + 96];
      d4[i] = a;
      d4[i + 32] = b;
      d4[i + 64] = c;
      d4[i + 96] = e;
    }
    for (; i < nv; i += 32) d4[i] = s4[i];
    for (int64_t j = head + (nv << 4) + (int64_t)lane * es; j < n; j += 32 * es) copy_elem(d + j, s + j, es);
  } else {
    for (int64_t j = (int64_t)lane * es; j < n; j += 32 * es) copy_elem(d + j, s + j, es);
  }
}

// warps [warp0, warp0+nwarps) of the caller process units warp0, warp0+nwarps, ...
__device__ __forceinline__ void copy_units(const RunBatch& b, int64_t warp, int64_t nwarps, int lane) {
  for (int64_t u = warp; u < b.total_units; u += nwarps) {
    int k = 0;
    while (k + 1 < b.n && b.d[k + 1].unit_begin <= u) k++;
    const RunDesc& d = b.d[k];
    const int64_t lu = u - d.unit_begin;
    if (d.chunks > 0) {
      const int64_t run = lu / d.chunks, c = lu - run * d.chunks;
      const int64_t i0 = run / d.n1, i1 = run - i0 * d.n1;
      const char* s = d.src + d.src_off + i0 * d.src_p0 + i1 * d.src_p1;
      char* t = d.dst + d.dst_off + i0 * d.dst_p0 + i1 * d.dst_p1;
      const int64_t b0 = c * d.chunk_bytes;
      const int64_t b1 = min(b0 + d.chunk_bytes, d.run_bytes);
      warp_copy(t + b0, s + b0, b1 - b0, d.es, lane);
    } else {
      const int64_t run = lu * 32 + lane;
      if (run < (int64_t)d.n0 * d.n1) {
        const int64_t i0 = run / d.n1, i1 = run - i0 * d.n1;
        const char* s = d.src + d.src_off + i0 * d.src_p0 + i1 * d.src_p1;
        char* t = d.dst + d.dst_off + i0 * d.dst_p0 + i1 * d.dst_p1;
        for (int64_t j = 0; j < d.run_bytes; j += d.es) copy_elem(t + j, s + j, d.es);
      }
    }
  }
}

__global__ void __launch_bounds__(256) copy_runs_kernel(const __grid_constant__ RunBatch b,
                                                        const __grid_constant__ KSync ks) {
  ks_pre(ks);
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  copy_units(b, warp, nwarps, lane);
  ks_post(ks);
}

cudaError_t launch_copy_runs(const RunBatch& b, const KSync& ks, cudaStream_t s) {
  if (b.total_units <= 0 && ks.nwait == 0 && ks.nsig == 0) return cudaSuccess;
  int64_t blocks = (b.total_units + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  copy_runs_kernel<<<(unsigned)blocks, 256, 0, s>>>(b, ks);
  return cudaGetLastError();
}

// =====================================================================================
// cross-device ordering
// =====================================================================================

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void wait_kernel(const __grid_constant__ WaitList w, int* err, long long timeout_ns) {
  const int i = threadIdx.x;
  if (i < w.n) {
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(w.ptr[i]) < w.val[i]) {
      __nanosleep(100);
      if ((long long)(globaltimer() - t0) > timeout_ns) {
        *reinterpret_cast<volatile int*>(err) = -7;  // HDA_ETIMEOUT, host-mapped
        __threadfence_system();
        break;
      }
    }
  }
  __syncthreads();
}

__global__ void signal_kernel(const __grid_constant__ SignalList l) {
  __threadfence_system();
  const int i = threadIdx.x;
  if (i < l.n) st_release_sys(l.ptr[i], l.val);
}

cudaError_t launch_wait(const WaitList& w, int* err_flag, long long timeout_ns, cudaStream_t s) {
  if (w.n <= 0) return cudaSuccess;
  wait_kernel<<<1, kMaxDev, 0, s>>>(w, err_flag, timeout_ns);
  return cudaGetLastError();
}

cudaError_t launch_signal(const SignalList& l, cudaStream_t s) {
  if (l.n <= 0) return cudaSuccess;
  signal_kernel<<<1, kMaxDev, 0, s>>>(l);
  return cudaGetLastError();
}

// =====================================================================================
// 2-D stencils: 16-byte column vectors per thread, marching down rows with a
// register window; horizontal neighbours by warp shuffles (edge lanes load).
// Every input element is fetched from DRAM once per block (2 halo rows per ROWS).
// =====================================================================================

template <typename T>
struct V16;
template <>
struct V16<double> {
  static constexpr int n = 2;
  __device__ static void load(double (&r)[2], const double* p) {
    double2 v = __ldg(reinterpret_cast<const double2*>(p));
    r[0] = v.x;
    r[1] = v.y;
  }
  // coherent (L1-bypassing) load: data another kernel is writing during this one
  __device__ static void load_cg(double (&r)[2], const double* p) {
    double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    r[0] = v.x;
    r[1] = v.y;
  }
  __device__ static void store(double* p, const double (&r)[2]) {
    *reinterpret_cast<double2*>(p) = make_double2(r[0], r[1]);
  }
};
template <>
struct V16<float> {
  static constexpr int n = 4;
  __device__ static void load(float (&r)[4], const float* p) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p));
    r[0] = v.x;
    r[1] = v.y;
    r[2] = v.z;
    r[3] = v.w;
  }
  __device__ static void load_cg(float (&r)[4], const float* p) {
    float4 v = __ldcg(reinterpret_cast<const float4*>(p));
    r[0] = v.x;
    r[1] = v.y;
    r[2] = v.z;
    r[3] = v.w;
  }
  __device__ static void store(float* p, const float (&r)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
  }
};

// Tuned on B200 (tools/stencil_tune.cu, 8192^2 f64): 256 threads x 16 rows per block,
// 4-row load groups, >= 4 blocks/SM -> 6.24 TB/s = 95% of the measured copy peak
// (128 threads x 32 rows x 8-row groups at 113 registers reached only 4.99 TB/s:
// too few warps in flight).
static int sm_count_dev() {
  static std::atomic<int> n[64];  // launches may come from several host threads
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int v = n[dev].load(std::memory_order_relaxed);
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// HDA_ONE_WAVE=0 disables the one-wave row-range layout (A/B measurements)
static bool one_wave_enabled() {
  static const int v = [] {
    const char* e = std::getenv("HDA_ONE_WAVE");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

// launch with the programmatic-stream-serialization attribute; only for kernels whose
// first statement is pdl_enter() (sync.cuh).  HDA_PDL=0 disables it.
static bool pdl_enabled() {
  static const int v = [] {
    const char* e = std::getenv("HDA_PDL");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// PROD signals of a user kernel as their own tiny launch (PDL): the wait returns when
// the kernel before it on the stream has completed — all of its writes are in this
// GPU's L2, where peers read them — so no CTA of the big kernel pays a fence + counter
// at its end (measured: 1.5 us/step for a one-wave share, 8 us for 8192^2 N=1 tiles).
// griddepcontrol.wait orders the previous kernel's writes before this thread; the
// system-scope fence then makes the relaxed system-scope flag stores a release at
// system scope (fence cumulativity), which a peer's ld.acquire.sys synchronises with.
__global__ void signal_pdl_kernel(const __grid_constant__ SignalList l, int relaxed) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (relaxed) __threadfence_system();
  const int i = threadIdx.x;
  if (i < l.n) {
    if (relaxed)
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(l.ptr[i]), "l"(l.val) : "memory");
    else
      st_release_sys(l.ptr[i], l.val);
  }
}
cudaError_t launch_signal_pdl(const SignalList& l, int relaxed, cudaStream_t s) {
  if (l.n <= 0) return cudaSuccess;
  return launch_pdl(signal_pdl_kernel, dim3(1), dim3(kMaxDev), s, l, relaxed);
}

// HDA_TAIL_ROWS (default 4; 0 = off) / HDA_TAIL_WAVES (default 1): rows per tile and
// waves of the short tiles that end a many-wave 2-D stencil launch
static int env_or(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
static int tail_rows() {
  static const int v = env_or("HDA_TAIL_ROWS", 4);
  return v;
}
// HDA_ST_PF (5-point) / HDA_ST9_PF (9-point): L2 bulk-prefetch distance of the 2-D
// register-march stencils, in row groups (0 = off).  Measured on one B200 (N=1,
// profiles/r02/prefetch/): Jacobi 8192^2 0.897 -> 0.970 of HBM at 1 (0.957 at 2);
// 9-point 16384^2 0.795 -> 0.917 at 1 (0.891 at 2, 0.875 at 3)
static int st_prefetch(int kind) {
  static const int p5 = env_or("HDA_ST_PF", 1), p9 = env_or("HDA_ST9_PF", 1);
  return kind == 0 ? p5 : p9;
}
static int tail_waves() {
  static const int v = env_or("HDA_TAIL_WAVES", 1);
  return v;
}

constexpr int ST_THREADS = 256;  // threads per block along the row
constexpr int ST_GROUP = 4;      // rows loaded together (loads in flight per thread)
#ifndef ST_ROWS_DEF
#define ST_ROWS_DEF 16
#endif
constexpr int ST_ROWS = ST_ROWS_DEF;  // rows per block (16-row tiles)
#ifndef ST9_ROWS
#define ST9_ROWS 32  // the 9-point kernel's tile height (plain launches)
#endif
constexpr int ST_MINB = 4;       // resident blocks per SM (register cap)
#ifndef ST9_MINB
// the 9-point kernel's register cap (blocks per SM): 5 spilled (48 registers); with the
// constant-reciprocal division and the L2 prefetch, 4 (64 registers, no spills) is ahead:
// 376 vs 364 GPoints/s at 40 sweeps, 344 vs 330 at 200 (profiles/r02/stencil9_minb/)
#define ST9_MINB 4
#endif

template <typename T>
__device__ __forceinline__ T quarter(T x);
template <>
__device__ __forceinline__ double quarter(double x) { return x * 0.25; }
template <>
__device__ __forceinline__ float quarter(float x) { return x * 0.25f; }

template <typename T>
__device__ __forceinline__ T st9(T w, T e, T n, T s, T nw, T ne, T sw, T se) {
  T a = ((w + e) + n) + s;
  T c = ((nw + ne) + sw) + se;
  T t = T(4) * a;
  t = t + c;
  return div20(t);
}

// KIND 0 = JACOBI5, 1 = STENCIL9
// up to 8 boxes per launch (blockIdx.z picks the box): the dependent boundary strips of
// an overlapped halo exchange run as ONE launch
struct Boxes2 {
  int64_t r0[8], r1[8], c0[8], c1[8], cbase[8];
  int64_t rpb[8];     // rows per block (each block marches a contiguous row range)
  int64_t tstart[9];  // flat-grid launches: first tile of each box
  int32_t gx[8], gy[8];
  int32_t n;
  int32_t ndep_first;  // fused halo kernel: boxes [0, ndep_first) are the boundary strips
  int32_t pf;          // L2 bulk prefetch distance in row groups (HDA_ST_PF; 0 = off)
};

template <typename T, int KIND, int ROWS, bool CG>
__device__ __forceinline__ void stencil2d_body(const T* __restrict__ in, T* __restrict__ out, int64_t ld,
                                               int64_t r0, int64_t r1, int64_t c0, int64_t c1, int64_t cbase,
                                               int64_t rpb, int64_t xb, int64_t yb, int pf = 0) {
  constexpr int V = V16<T>::n;
  constexpr int W = ST_GROUP + 2;
  const int lane = threadIdx.x & 31;
  const int64_t col = cbase + (xb * ST_THREADS + threadIdx.x) * V;
  const bool live = col < ld;
  const int64_t rs = r0 + yb * rpb;
  const int64_t re = min(rs + rpb, r1);
  T w[W][V];

  auto load_row = [&](T(&r)[V], int64_t row) {
    if (live) {
      if (CG)
        V16<T>::load_cg(r, in + row * ld + col);
      else
        V16<T>::load(r, in + row * ld + col);
    } else {
#pragma unroll
      for (int v = 0; v < V; v++) r[v] = T(0);
    }
  };
  auto edges = [&](const T(&r)[V], int64_t row, T& L, T& R) {
    L = __shfl_up_sync(0xffffffffu, r[V - 1], 1);
    R = __shfl_down_sync(0xffffffffu, r[0], 1);
    // the neighbour of column 0 / ld-1 is never used (work boxes keep a 1-cell ring),
    // and loading it would step outside the replica for the first / last row
    if (lane == 0 && live && col > 0) L = CG ? __ldcg(in + row * ld + col - 1) : __ldg(in + row * ld + col - 1);
    if (lane == 31 && live && col + V < ld) R = CG ? __ldcg(in + row * ld + col + V) : __ldg(in + row * ld + col + V);
  };

  // L2 bulk prefetch pf row groups ahead: lane 0 of warp k < ST_GROUP prefetches the
  // block's span of one row, so the demand loads meet L2 rather than DRAM latency
  const int wid = threadIdx.x >> 5;
  const int64_t col0 = cbase + xb * ST_THREADS * V;
  const uint32_t span = (uint32_t)(min((int64_t)ST_THREADS * V, ld - col0) * (int64_t)sizeof(T));
  const bool pf_on = pf > 0 && lane == 0 && col0 < ld && (ld * (int64_t)sizeof(T)) % 16 == 0;
  auto prefetch_row = [&](int64_t row) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(in + row * ld + col0), "r"(span) : "memory");
  };
  if (pf_on)
    for (int64_t row = rs + 1 + wid; row <= min(re, rs + (int64_t)ST_GROUP * pf); row += ST_THREADS / 32)
      prefetch_row(row);
  load_row(w[0], rs - 1);
  load_row(w[1], rs);
  for (int64_t base = rs; base < re; base += ST_GROUP) {
    if (pf_on && wid < ST_GROUP) {
      const int64_t row = base + 1 + (int64_t)ST_GROUP * pf + wid;
      if (row <= re) prefetch_row(row);
    }
#pragma unroll
    for (int k = 0; k < ST_GROUP; k++)
      if (base + 1 + k <= re) load_row(w[k + 2], base + 1 + k);
#pragma unroll
    for (int k = 0; k < ST_GROUP; k++) {
      const int64_t r = base + k;
      if (r >= re) break;
      T o[V];
      if (KIND == 0) {
        T L, R;
        edges(w[k + 1], r, L, R);
#pragma unroll
        for (int v = 0; v < V; v++) {
          const T left = v == 0 ? L : w[k + 1][v - 1];
          const T right = v == V - 1 ? R : w[k + 1][v + 1];
          o[v] = quarter<T>(((left + right) + w[k][v]) + w[k + 2][v]);
        }
      } else {
        // recompute the row-edge shuffles of up/cur/dn for every output row: keeping
        // them in a register window cost occupancy (tuned: 84% vs 73% of HBM)
        T ul, ur, cl, cr, dl, dr;
        edges(w[k], r - 1, ul, ur);
        edges(w[k + 1], r, cl, cr);
        edges(w[k + 2], r + 1, dl, dr);
#pragma unroll
        for (int v = 0; v < V; v++) {
          const T* up = w[k];
          const T* cu = w[k + 1];
          const T* dn = w[k + 2];
          const T cL = v == 0 ? cl : cu[v - 1], cR = v == V - 1 ? cr : cu[v + 1];
          const T uL = v == 0 ? ul : up[v - 1], uR = v == V - 1 ? ur : up[v + 1];
          const T dL = v == 0 ? dl : dn[v - 1], dR = v == V - 1 ? dr : dn[v + 1];
          o[v] = st9<T>(cL, cR, up[v], dn[v], uL, uR, dL, dR);
        }
      }
      if (live) {
        T* dst = out + r * ld + col;
        if (col >= c0 && col + V <= c1) {
          V16<T>::store(dst, o);
        } else {
#pragma unroll
          for (int v = 0; v < V; v++)
            if (col + v >= c0 && col + v < c1) dst[v] = o[v];
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; v++) {
      w[0][v] = w[ST_GROUP][v];
      w[1][v] = w[ST_GROUP + 1][v];
    }
  }
}

// flat 1-D grid over the tiles of up to 8 boxes (no empty blocks for mixed box shapes)
__device__ __forceinline__ void tile_of(const Boxes2& bx, int64_t t, int& b, int64_t& xb, int64_t& yb) {
  b = 0;
  while (b + 1 < bx.n && bx.tstart[b + 1] <= t) b++;
  const int64_t local = t - bx.tstart[b];
  xb = local % bx.gx[b];
  yb = local / bx.gx[b];
}

template <typename T, int KIND, int ROWS>
__global__ void __launch_bounds__(ST_THREADS, KIND == 1 ? ST9_MINB : ST_MINB)
    stencil2d_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t ld, const __grid_constant__ Boxes2 bx,
                     const __grid_constant__ KSync ks) {
  pdl_enter();
  ks_pre(ks);
  if (bx.n > 0) {
    int b;
    int64_t xb, yb;
    tile_of(bx, blockIdx.x, b, xb, yb);
    stencil2d_body<T, KIND, ROWS, false>(in, out, ld, bx.r0[b], bx.r1[b], bx.c0[b], bx.c1[b], bx.cbase[b],
                                         bx.rpb[b], xb, yb, bx.pf);
  }
  ks_post(ks);
}

// Fused halo-exchange stencil (one launch per step).  z-slice 0: NVLink pull blocks —
// they wait for the writers' PROD words, copy every planned halo rectangle from the
// peers' replicas into this replica, and the last of them releases a local word and the
// writers' ACK words.  z-slices 1..: the stencil boxes (interior first, dependent strips
// last); dependent blocks wait for the local word and read with L1-bypassing loads.
// The pull blocks are dispatched first and wait on nothing inside the kernel, so the
// dependent blocks' in-kernel wait always makes progress.
struct PullPart {
  unsigned long long* wait_ptr[16];
  unsigned long long wait_val[16];
  unsigned long long* ack_ptr[8];
  int32_t nwait, nack, nblocks;
  unsigned int* ctr;
  unsigned long long* done_word;  // local
  unsigned long long epoch;
  long long delay_ns;
};

template <typename T, int KIND, int ROWS>
#ifndef HALO_MINB0
#define HALO_MINB0 4  // 5-point fused kernel: CTAs per SM the register budget must allow
#endif
__global__ void __launch_bounds__(ST_THREADS, KIND == 0 ? HALO_MINB0 : ST_MINB)
    stencil2d_halo_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t ld,
                          const __grid_constant__ Boxes2 bx, int32_t n_interior,
                          const __grid_constant__ RunBatch pull, const __grid_constant__ PullPart pp,
                          const __grid_constant__ KSync ks) {
  pdl_enter();
  // flat grid: [0, nblocks) pull; then the tiles of box 0, 1, ... (interior boxes first)
  const int64_t bid = blockIdx.x;
  if (bid < pp.nblocks) {
    // RAW: the writers finished the call that produced these cells
    if ((int)threadIdx.x < pp.nwait) {
      const unsigned long long t0 = ks_timer();
      while (ks_ld_acquire(pp.wait_ptr[threadIdx.x]) < pp.wait_val[threadIdx.x]) {
        __nanosleep(32);
        if ((long long)(ks_timer() - t0) > ks.timeout_ns) {
          *reinterpret_cast<volatile int*>(ks.err) = -7;
          __threadfence_system();
          break;
        }
      }
    }
    if (pp.delay_ns && threadIdx.x == 0) {  // test hook
      const unsigned long long t0 = ks_timer();
      while ((long long)(ks_timer() - t0) < pp.delay_ns) __nanosleep(1000);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    copy_units(pull, (bid * ST_THREADS + threadIdx.x) >> 5, ((int64_t)pp.nblocks * ST_THREADS) >> 5, lane);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(pp.ctr, 1u) == (unsigned)pp.nblocks - 1) {
        *pp.ctr = 0;
        __threadfence_system();  // release at system scope for the relaxed flag stores
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(pp.done_word), "l"(pp.epoch) : "memory");
        for (int i = 0; i < pp.nack; i++)
          asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(pp.ack_ptr[i]), "l"(pp.epoch) : "memory");
      }
    }
    ks_post(ks);
    return;
  }
  ks_pre(ks);  // WAR: peers finished reading the cells this launch overwrites
  int b;
  int64_t xb, yb;
  tile_of(bx, bid - pp.nblocks, b, xb, yb);
  if (bx.ndep_first ? b < bx.ndep_first : b >= n_interior) {
    if (threadIdx.x == 0) {
      const unsigned long long t0 = ks_timer();
      while (ks_ld_acquire(pp.done_word) < pp.epoch) {
        __nanosleep(32);
        if ((long long)(ks_timer() - t0) > ks.timeout_ns) {
          *reinterpret_cast<volatile int*>(ks.err) = -7;
          __threadfence_system();
          break;
        }
      }
    }
    __syncthreads();
    // boundary strips are thin (a row or a column): one point per thread with
    // L1-bypassing loads, instead of a second (cache-global) copy of the register-window
    // body that pushed the 9-point kernel into spills
    const int64_t rs = bx.r0[b] + yb * bx.rpb[b], re = min(rs + bx.rpb[b], bx.r1[b]);
    const int64_t cs = max(bx.c0[b], bx.cbase[b] + xb * ST_THREADS * V16<T>::n);
    const int64_t ce = min(bx.c1[b], bx.cbase[b] + (xb + 1) * ST_THREADS * V16<T>::n);
    const int64_t w = ce - cs;
    for (int64_t i = threadIdx.x; w > 0 && i < (re - rs) * w; i += ST_THREADS) {
      const int64_t r = rs + i / w, c = cs + i % w;
      const T* p = in + r * ld + c;
      if (KIND == 0) {
        out[r * ld + c] = quarter<T>(((__ldcg(p - 1) + __ldcg(p + 1)) + __ldcg(p - ld)) + __ldcg(p + ld));
      } else {
        out[r * ld + c] = st9<T>(__ldcg(p - 1), __ldcg(p + 1), __ldcg(p - ld), __ldcg(p + ld), __ldcg(p - ld - 1),
                                 __ldcg(p - ld + 1), __ldcg(p + ld - 1), __ldcg(p + ld + 1));
      }
    }
  } else {
    stencil2d_body<T, KIND, ROWS, false>(in, out, ld, bx.r0[b], bx.r1[b], bx.c0[b], bx.c1[b], bx.cbase[b],
                                         bx.rpb[b], xb, yb, bx.pf);
  }
  ks_post(ks);
}

// scalar fallback for row pitches that are not 16-byte multiples (small test shapes)
template <typename T, int KIND>
__global__ void stencil2d_scalar_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t ld,
                                        int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                                        const __grid_constant__ KSync ks) {
  ks_pre(ks);
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = r0 + blockIdx.y;
  if (c < c1 && r < r1) {
    const T* p = in + r * ld + c;
    if (KIND == 0) {
      out[r * ld + c] = quarter<T>(((p[-1] + p[1]) + p[-ld]) + p[ld]);
    } else {
      out[r * ld + c] = st9<T>(p[-1], p[1], p[-ld], p[ld], p[-ld - 1], p[-ld + 1], p[ld - 1], p[ld + 1]);
    }
  }
  ks_post(ks);
}

template <typename T, int KIND>
static cudaError_t launch_stencil2d_t(const T* in, T* out, const int64_t* shape, const int64_t* const* lbs,
                                      const int64_t* const* ubs, int nb, const KSync& ks, cudaStream_t s) {
  const int64_t ld = shape[2];
  constexpr int V = V16<T>::n;
  if (nb == 1 && stencil_tma_mode() >= (KIND == 1 ? 1 : 2)) {
    const cudaError_t e = launch_stencil2d_tma(KIND, sizeof(T) == 8 ? 0 : 1, in, out, shape, lbs[0], ubs[0], ks, s);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
  }
  const bool vec = (ld * (int64_t)sizeof(T)) % 16 == 0 && ((uintptr_t)in % 16) == 0 &&
                   ((uintptr_t)out % 16) == 0;
  if (vec) {
    constexpr int ROWS = ST_ROWS;
    Boxes2 bx;
    bx.n = 0;
    bx.ndep_first = 0;
    bx.pf = st_prefetch(KIND);
    for (int i = 0; i < nb && bx.n < 8; i++) {
      const int64_t r0 = lbs[i][1], r1 = ubs[i][1], c0 = lbs[i][2], c1 = ubs[i][2];
      if (r0 >= r1 || c0 >= c1 || lbs[i][0] >= ubs[i][0]) continue;
      const int k = bx.n++;
      bx.r0[k] = r0;
      bx.r1[k] = r1;
      bx.c0[k] = c0;
      bx.c1[k] = c1;
      bx.cbase[k] = c0 - (c0 % V);
      const int64_t per_block = (int64_t)ST_THREADS * V;
      bx.gx[k] = (int)((c1 - bx.cbase[k] + per_block - 1) / per_block);
    }
    // Large boxes: 16-row tiles, many waves (94% of HBM at 8190 rows).  Boxes that
    // would take fewer than ~5 waves (a GPU's share at N >= 4) instead get one wave of
    // 148 x ST_MINB blocks marching contiguous row ranges: no tail wave, 2 halo rows
    // per block, and register headroom on every SM for an overlapped halo pull.
    // Narrow boxes (column strips of a BLOCK halo: one live thread per block) keep
    // 16-row tiles.
    int64_t strips = 0, tiles16 = 0;
    for (int k = 0; k < bx.n; k++) {
      strips += bx.gx[k];
      tiles16 += (int64_t)bx.gx[k] * ((bx.r1[k] - bx.r0[k] + ST_ROWS - 1) / ST_ROWS);
    }
    const int64_t wave = (int64_t)sm_count_dev() * ST_MINB;
    // (5-point: 16-row tiles + the tail split below beat one wave at every size, e.g.
    // 4096^2 45.5 vs 49.8 us; the 9-point keeps the one-wave layout for small shares)
    const bool one_wave = one_wave_enabled() && tiles16 < 5 * wave && !(KIND == 0 && tail_rows() > 0);
    bx.tstart[0] = 0;
    for (int k = 0; k < bx.n; k++) {
      const int64_t rows = bx.r1[k] - bx.r0[k];
      // tile height: 16 rows, or ST9_ROWS (32) for a wide 9-point box that still spans
      // >= 10 waves of them.  16384^2 9-point (profiles/r02/stencil9_rows/): N=1 (28
      // waves) 385.5 vs 376.6 GPoints/s, N=2 (14) 728 vs 696-702; N=4 (7 waves) 1225 vs
      // 1259 with 32.  64 rows: 371.3 at N=1.  The 5-point loses at 32 (367.7 vs 399.8).
      // Narrow boxes (a BLOCK halo's column strips, one live thread per block) keep 16.
      int64_t trows = ST_ROWS;
      if (KIND == 1 && bx.c1[k] - bx.c0[k] > 64 &&
          (int64_t)bx.gx[k] * ((rows + ST9_ROWS - 1) / ST9_ROWS) >= 10 * wave)
        trows = ST9_ROWS;
      int64_t gyk = (rows + trows - 1) / trows;
      if (one_wave && bx.c1[k] - bx.c0[k] > 64) {
        gyk = std::max<int64_t>(1, wave / std::max<int64_t>(strips, 1));
        gyk = std::min<int64_t>(gyk, (rows + ST_GROUP - 1) / ST_GROUP);
      }
      bx.rpb[k] = (rows + gyk - 1) / gyk;
      bx.gy[k] = (int)((rows + bx.rpb[k] - 1) / bx.rpb[k]);
      bx.tstart[k + 1] = bx.tstart[k] + (int64_t)bx.gx[k] * bx.gy[k];
    }
    // Tail split (many-wave single box): the last rows become short tiles, dispatched
    // last, so the final partial wave drains in a fraction of a 16-row tile's time.
    // (5-point only: 8192^2 Jacobi 390.7 -> 396.3 GPoints/s; the 9-point, 44 waves of
    // 5 CTAs/SM, gains nothing)
    if (KIND == 0 && !one_wave && bx.n == 1 && tail_rows() > 0 && bx.c1[0] - bx.c0[0] > 64) {
      static const int occ = [] {  // thread-safe one-time init
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, stencil2d_kernel<T, KIND, ROWS>, ST_THREADS, 0);
        return o > 0 ? o : ST_MINB;
      }();
      const int64_t tr = tail_rows();
      const int64_t slots = (int64_t)sm_count_dev() * occ;
      int64_t trows = (tail_waves() * slots + bx.gx[0] - 1) / bx.gx[0] * tr;
      const int64_t rows = bx.r1[0] - bx.r0[0];
      trows = std::min<int64_t>(trows, rows / 4) / tr * tr;
      if (trows > 0) {
        bx.n = 2;
        bx.r0[1] = bx.r1[0] - trows;
        bx.r1[1] = bx.r1[0];
        bx.r1[0] = bx.r0[1];
        bx.c0[1] = bx.c0[0];
        bx.c1[1] = bx.c1[0];
        bx.cbase[1] = bx.cbase[0];
        bx.gx[1] = bx.gx[0];
        for (int k = 0; k < 2; k++) {
          const int64_t rk = bx.r1[k] - bx.r0[k];
          bx.rpb[k] = k ? tr : ST_ROWS;
          bx.gy[k] = (int)((rk + bx.rpb[k] - 1) / bx.rpb[k]);
          bx.tstart[k + 1] = bx.tstart[k] + (int64_t)bx.gx[k] * bx.gy[k];
        }
      }
    }
    // bx.n == 0: nothing to compute, but the sync words must still move (one block)
    const int64_t grid = bx.n ? bx.tstart[bx.n] : 1;
    cudaError_t e = launch_pdl(stencil2d_kernel<T, KIND, ROWS>, dim3((unsigned)grid), dim3(ST_THREADS), s, in, out,
                               ld, bx, ks);
    if (e != cudaSuccess) return e;
  } else {
    for (int i = 0; i < nb; i++) {
      const int64_t r0 = lbs[i][1], r1 = ubs[i][1], c0 = lbs[i][2], c1 = ubs[i][2];
      if (r0 >= r1 || c0 >= c1) continue;
      // scalar fallback (test shapes): sync words ride with the first/last launch
      KSync k2 = ks;
      if (i != 0) k2.nwait = 0;
      if (i != nb - 1) k2.nsig = 0;
      dim3 grid((unsigned)((c1 - c0 + 127) / 128), (unsigned)(r1 - r0));
      stencil2d_scalar_kernel<T, KIND><<<grid, 128, 0, s>>>(in, out, ld, r0, r1, c0, c1, k2);
    }
  }
  return cudaGetLastError();
}

template <typename T, int KIND>
static cudaError_t launch_halo_t(const T* in, T* out, const int64_t* shape, const int64_t* const* lbs,
                                 const int64_t* const* ubs, int nb, int n_interior, const RunBatch& pull,
                                 const HaloPull& hp, const KSync& ks, cudaStream_t s) {
  const int64_t ld = shape[2];
  constexpr int V = V16<T>::n;
  constexpr int ROWS = ST_ROWS;
  Boxes2 bx;
  bx.n = 0;
  int ni = 0;
  for (int i = 0; i < nb && bx.n < 8; i++) {
    const int64_t r0 = lbs[i][1], r1 = ubs[i][1], c0 = lbs[i][2], c1 = ubs[i][2];
    if (r0 >= r1 || c0 >= c1 || lbs[i][0] >= ubs[i][0]) continue;
    if (i < n_interior) ni++;
    const int k = bx.n++;
    bx.r0[k] = r0;
    bx.r1[k] = r1;
    bx.c0[k] = c0;
    bx.c1[k] = c1;
    bx.cbase[k] = c0 - (c0 % V);
    const int64_t per_block = (int64_t)ST_THREADS * V;
    bx.gx[k] = (int)((c1 - bx.cbase[k] + per_block - 1) / per_block);
  }
  int64_t pb = (pull.total_units + 7) / 8;  // 8 warps per block
  // pull blocks at most (HDA_HALO_NPULL): they spin on the writers' PROD words until the
  // neighbours finish, holding slots the interior could use; N=8-sized shares (5792^2 on
  // 4 GPUs): 16 -> 997-1001 GPoints/s, 64 -> 969-986, 4 -> 662-670 (profiles/r02/halo_npull/)
  static const int npull_cap = env_or("HDA_HALO_NPULL", 16);
  const int npull = (int)std::max<int64_t>(1, std::min<int64_t>(pb, npull_cap));
  // Interior boxes: when the GPU's share is under ~5 waves of 16-row tiles, ONE wave
  // of row-range blocks sized to the slots the pull blocks leave free (blocks that
  // miss the first wave would double the step); the boundary strips keep 16-row tiles
  // and run in the slots the pull blocks vacate.
  static const int occ = [] {  // thread-safe one-time init
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, stencil2d_halo_kernel<T, KIND, ROWS>, ST_THREADS, 0);
    return o > 0 ? o : 1;
  }();
  const int64_t wave = (int64_t)sm_count_dev() * occ;
  int64_t tiles16 = 0, strips_i = 0;
  for (int k = 0; k < bx.n; k++) {
    tiles16 += (int64_t)bx.gx[k] * ((bx.r1[k] - bx.r0[k] + ST_ROWS - 1) / ST_ROWS);
    if (k < ni && bx.c1[k] - bx.c0[k] > 64) strips_i += bx.gx[k];
  }
  // HDA_DEP_FIRST (default 1): the boundary strips are dispatched right after the pull
  // blocks instead of last, so the step ends with interior tiles only (as a standalone
  // launch) instead of the strips' wait + compute latency
  static const int dep_first = env_or("HDA_DEP_FIRST", 1);
  int64_t dep_tiles = 0;
  for (int k = ni; k < bx.n; k++)
    dep_tiles += (int64_t)bx.gx[k] * ((bx.r1[k] - bx.r0[k] + ST_ROWS - 1) / ST_ROWS);
  const int64_t slots = wave - npull - (dep_first ? dep_tiles : 0);
  const bool one_wave = one_wave_enabled() && tiles16 < 5 * wave && strips_i > 0 && slots >= strips_i;
  // many-wave share (N=2) with one interior box: its last rows as a tail box of short
  // tiles, dispatched after the interior and before the boundary strips (5-point only,
  // as in the plain launch)
  int tail_k = -1;
  if (KIND == 0 && !one_wave && ni == 1 && bx.n < 8 && tail_rows() > 0 && bx.c1[0] - bx.c0[0] > 64) {
    const int64_t tr = tail_rows();
    int64_t trows = (tail_waves() * wave + bx.gx[0] - 1) / bx.gx[0] * tr;
    trows = std::min<int64_t>(trows, (bx.r1[0] - bx.r0[0]) / 4) / tr * tr;
    if (trows > 0) {
      for (int k = bx.n; k > 1; k--) {  // shift the boundary boxes up by one
        bx.r0[k] = bx.r0[k - 1];
        bx.r1[k] = bx.r1[k - 1];
        bx.c0[k] = bx.c0[k - 1];
        bx.c1[k] = bx.c1[k - 1];
        bx.cbase[k] = bx.cbase[k - 1];
        bx.gx[k] = bx.gx[k - 1];
      }
      bx.n++;
      bx.r0[1] = bx.r1[0] - trows;
      bx.r1[1] = bx.r1[0];
      bx.r1[0] = bx.r0[1];
      bx.c0[1] = bx.c0[0];
      bx.c1[1] = bx.c1[0];
      bx.cbase[1] = bx.cbase[0];
      bx.gx[1] = bx.gx[0];
      ni = 2;
      tail_k = 1;
    }
  }
  bx.tstart[0] = 0;
  for (int k = 0; k < bx.n; k++) {
    const int64_t rows = bx.r1[k] - bx.r0[k];
    int64_t gyk = (rows + ST_ROWS - 1) / ST_ROWS;
    if (one_wave && k < ni && bx.c1[k] - bx.c0[k] > 64) {
      gyk = std::max<int64_t>(1, slots / strips_i);
      gyk = std::min<int64_t>(gyk, (rows + ST_GROUP - 1) / ST_GROUP);
    }
    if (k == tail_k) gyk = (rows + tail_rows() - 1) / tail_rows();  // short tiles
    bx.rpb[k] = (rows + gyk - 1) / gyk;
    bx.gy[k] = (int)((rows + bx.rpb[k] - 1) / bx.rpb[k]);
    bx.tstart[k + 1] = bx.tstart[k] + (int64_t)bx.gx[k] * bx.gy[k];
  }
  bx.ndep_first = 0;
  // no L2 prefetch in the fused halo launch (HDA_HALO_PF): forced onto 268 MB shares
  // (8192^2, N=4) it costs 998 vs 1172 GPoints/s; on the 134 MB shares the fused launch is
  // chosen for, 990 without vs 997-1001 with (separate boxes; within 1%, profiles/r02/halo_pf/)
  static const int halo_pf = env_or("HDA_HALO_PF", 0);
  bx.pf = halo_pf;
  if (dep_first && ni < bx.n) {  // rotate the boundary boxes to the front
    Boxes2 o = bx;
    int j = 0;
    for (int k = ni; k < o.n; k++, j++) {
      bx.r0[j] = o.r0[k], bx.r1[j] = o.r1[k], bx.c0[j] = o.c0[k], bx.c1[j] = o.c1[k];
      bx.cbase[j] = o.cbase[k], bx.rpb[j] = o.rpb[k], bx.gx[j] = o.gx[k], bx.gy[j] = o.gy[k];
    }
    for (int k = 0; k < ni; k++, j++) {
      bx.r0[j] = o.r0[k], bx.r1[j] = o.r1[k], bx.c0[j] = o.c0[k], bx.c1[j] = o.c1[k];
      bx.cbase[j] = o.cbase[k], bx.rpb[j] = o.rpb[k], bx.gx[j] = o.gx[k], bx.gy[j] = o.gy[k];
    }
    bx.ndep_first = o.n - ni;
    bx.tstart[0] = 0;
    for (int k = 0; k < bx.n; k++) bx.tstart[k + 1] = bx.tstart[k] + (int64_t)bx.gx[k] * bx.gy[k];
  }
  PullPart pp;
  std::memset(&pp, 0, sizeof pp);
  pp.nwait = hp.nwait;
  pp.nack = hp.nack;
  for (int i = 0; i < hp.nwait; i++) {
    pp.wait_ptr[i] = hp.wait_ptr[i];
    pp.wait_val[i] = hp.wait_val[i];
  }
  for (int i = 0; i < hp.nack; i++) pp.ack_ptr[i] = hp.ack_ptr[i];
  pp.ctr = hp.ctr;
  pp.done_word = hp.done_word;
  pp.epoch = hp.epoch;
  pp.delay_ns = hp.delay_ns;
  pp.nblocks = npull;
  const int64_t grid = pp.nblocks + bx.tstart[bx.n];
  return launch_pdl(stencil2d_halo_kernel<T, KIND, ROWS>, dim3((unsigned)grid), dim3(ST_THREADS), s, in, out, ld,
                    bx, ni, pull, pp, ks);
}

cudaError_t launch_stencil2d_halo(int kernel, int dtype, const void* in, void* out, const int64_t* shape,
                                  const int64_t* const* lbs, const int64_t* const* ubs, int nb, int n_interior,
                                  const RunBatch& pull, const HaloPull& hp, const KSync& ks, cudaStream_t s) {
  if (kernel == 1) {
    if (dtype == 0)
      return launch_halo_t<double, 0>((const double*)in, (double*)out, shape, lbs, ubs, nb, n_interior, pull, hp, ks, s);
    return launch_halo_t<float, 0>((const float*)in, (float*)out, shape, lbs, ubs, nb, n_interior, pull, hp, ks, s);
  }
  if (dtype == 0)
    return launch_halo_t<double, 1>((const double*)in, (double*)out, shape, lbs, ubs, nb, n_interior, pull, hp, ks, s);
  return launch_halo_t<float, 1>((const float*)in, (float*)out, shape, lbs, ubs, nb, n_interior, pull, hp, ks, s);
}

cudaError_t launch_jacobi5(int dtype, const void* in, void* out, const int64_t* shape, const int64_t* const* lbs,
                           const int64_t* const* ubs, int nb, const KSync& ks, cudaStream_t s) {
  if (dtype == 0) return launch_stencil2d_t<double, 0>((const double*)in, (double*)out, shape, lbs, ubs, nb, ks, s);
  return launch_stencil2d_t<float, 0>((const float*)in, (float*)out, shape, lbs, ubs, nb, ks, s);
}

cudaError_t launch_stencil9(int dtype, const void* in, void* out, const int64_t* shape, const int64_t* const* lbs,
                            const int64_t* const* ubs, int nb, const KSync& ks, cudaStream_t s) {
  if (dtype == 0) return launch_stencil2d_t<double, 1>((const double*)in, (double*)out, shape, lbs, ubs, nb, ks, s);
  return launch_stencil2d_t<float, 1>((const float*)in, (float*)out, shape, lbs, ubs, nb, ks, s);
}

// =====================================================================================
// 3-D 7-point stencil.  A block's 8 warps span S3_X = 1024 contiguous floats of a row
// (4 KiB DRAM bursts; a block that spans 8 rows x 512 B plateaued at 69% of HBM),
// each thread owns S3_R consecutive y rows (their y neighbours come from registers;
// only rows y-1 and y+S3_R are extra, L2-resident loads) and marches S3_ZCH planes in z
// keeping planes z-1, z, z+1 in registers.  Tuned on 1024^3 f32: 84% of HBM.
// =====================================================================================

#ifndef S3_R_DEF
#define S3_R_DEF 2
#endif
#ifndef S3_ZCH_DEF
#define S3_ZCH_DEF 32
#endif
constexpr int S3_R = S3_R_DEF;      // y rows per thread
constexpr int S3_ZCH = S3_ZCH_DEF;  // planes per block

template <typename T>
__global__ void __launch_bounds__(256, 4) stencil7_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t n1,
                                                         int64_t n2, int64_t z0, int64_t z1, int64_t y0, int64_t y1,
                                                         int64_t x0, int64_t x1, int64_t xbase, int64_t nbig,
                                                         int64_t zt, int pf, int pf_halo,
                                                         const __grid_constant__ KSync ks) {
  pdl_enter();
  ks_pre(ks);
  constexpr int V = V16<T>::n;
  const int lane = threadIdx.x & 31;
  const int64_t x = xbase + ((int64_t)blockIdx.x * 256 + threadIdx.x) * V;
  const int64_t ya = y0 + (int64_t)blockIdx.y * S3_R;
  const bool live = x < n2;
  // chunks [0, nbig) hold S3_ZCH planes; the rest (dispatched last) zt planes each,
  // so the final partial wave drains quickly
  const int64_t bz = blockIdx.z;
  const int64_t zs = bz < nbig ? z0 + bz * S3_ZCH : z0 + nbig * S3_ZCH + (bz - nbig) * zt;
  const int64_t ze = min(zs + (bz < nbig ? (int64_t)S3_ZCH : zt), z1);
  const int64_t pl = n1 * n2;
  auto ld = [&](T(&r)[V], int64_t z, int64_t yy) {
    if (live && yy < n1) {
      V16<T>::load(r, in + z * pl + yy * n2 + x);
    } else {
#pragma unroll
      for (int v = 0; v < V; v++) r[v] = T(0);
    }
  };
  T zm[S3_R][V], zc[S3_R][V], zp[S3_R][V];
#pragma unroll
  for (int r = 0; r < S3_R; r++) {
    ld(zm[r], zs - 1, ya + r);
    ld(zc[r], zs, ya + r);
  }
  // L2 prefetch pf planes ahead (HDA_S7_PF): warp w < S3_R bulk-prefetches its block's
  // span of row ya + w (with HDA_S7_PF_HALO=1 also the rows above and below, which
  // other blocks prefetch too), so the demand loads below meet L2, not DRAM latency
  const int wid = threadIdx.x >> 5;
  const int64_t span = min((int64_t)256 * V, n2 - (xbase + (int64_t)blockIdx.x * 256 * V));
  const int halo = pf_halo ? 1 : 0;
  const int64_t pr = ya - halo + wid;
  const T* pfrow = in + pr * n2 + xbase + (int64_t)blockIdx.x * 256 * V;
  const bool pf_on = pf > 0 && lane == 0 && wid < S3_R + 2 * halo && pr < n1 && span > 0;
  if (pf_on)
    for (int d = 1; d < pf; d++)
      if (zs + d < z1 + 1)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pfrow + (zs + d) * pl),
                     "r"((uint32_t)(span * sizeof(T))) : "memory");
  for (int64_t z = zs; z < ze; z++) {
    if (pf_on && z + pf < z1 + 1)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pfrow + (z + pf) * pl),
                   "r"((uint32_t)(span * sizeof(T))) : "memory");
    T top[V], bot[V];
    ld(top, z, ya - 1);
    ld(bot, z, ya + S3_R);
#pragma unroll
    for (int r = 0; r < S3_R; r++) ld(zp[r], z + 1, ya + r);
#pragma unroll
    for (int r = 0; r < S3_R; r++) {
      const int64_t y = ya + r;
      const T* c = zc[r];
      const T* ym = r == 0 ? top : zc[r - 1];
      const T* yp = r == S3_R - 1 ? bot : zc[r + 1];
      T L = __shfl_up_sync(0xffffffffu, c[V - 1], 1);
      T R = __shfl_down_sync(0xffffffffu, c[0], 1);
      const T* row = in + z * pl + y * n2 + x;
      if (lane == 0 && live && x > 0 && y < y1) L = __ldg(row - 1);
      if (lane == 31 && live && x + V < n2 && y < y1) R = __ldg(row + V);
      T o[V];
#pragma unroll
      for (int v = 0; v < V; v++) {
        const T xl = v == 0 ? L : c[v - 1];
        const T xr = v == V - 1 ? R : c[v + 1];
        T s = xl + xr;
        s = s + ym[v];
        s = s + yp[v];
        s = s + zm[r][v];
        s = s + zp[r][v];
        o[v] = div6(s);
      }
      if (live && y < y1) {
        T* dst = out + z * pl + y * n2 + x;
        if (x >= x0 && x + V <= x1) {
          V16<T>::store(dst, o);
        } else {
#pragma unroll
          for (int v = 0; v < V; v++)
            if (x + v >= x0 && x + v < x1) dst[v] = o[v];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < S3_R; r++)
#pragma unroll
      for (int v = 0; v < V; v++) {
        zm[r][v] = zc[r][v];
        zc[r][v] = zp[r][v];
      }
  }
  ks_post(ks);
}

template <typename T>
__global__ void stencil7_scalar_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t n1, int64_t n2,
                                       int64_t z0, int64_t y0, int64_t y1, int64_t x0, int64_t x1,
                                       const __grid_constant__ KSync ks) {
  ks_pre(ks);
  const int64_t x = x0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t y = y0 + blockIdx.y;
  const int64_t z = z0 + blockIdx.z;
  if (x < x1 && y < y1) {
    const int64_t pl = n1 * n2;
    const T* p = in + z * pl + y * n2 + x;
    T s = p[-1] + p[1];
    s = s + p[-n2];
    s = s + p[n2];
    s = s + p[-pl];
    s = s + p[pl];
    out[z * pl + y * n2 + x] = div6(s);
  }
  ks_post(ks);
}

template <typename T>
static cudaError_t launch_stencil7_t(const T* in, T* out, const int64_t* shape, const int64_t* lb,
                                     const int64_t* ub, const KSync& ks, cudaStream_t s) {
  const int64_t n1 = shape[1], n2 = shape[2];
  if (lb[0] >= ub[0] || lb[1] >= ub[1] || lb[2] >= ub[2]) return cudaSuccess;
  constexpr int V = V16<T>::n;
  const bool vec = (n2 * (int64_t)sizeof(T)) % 16 == 0 && ((uintptr_t)in % 16) == 0 &&
                   ((uintptr_t)out % 16) == 0;
  if (vec) {
    const int64_t xbase = lb[2] - (lb[2] % V);
    const int64_t per = 256 * V;
    const int64_t gx = (ub[2] - xbase + per - 1) / per, gy = (ub[1] - lb[1] + S3_R - 1) / S3_R;
    const int64_t nz = ub[0] - lb[0];
    int64_t nbig = (nz + S3_ZCH - 1) / S3_ZCH, zt = S3_ZCH, ntail = 0;
    if (tail_rows() > 0 && nz > 4 * S3_ZCH) {
      // about one wave of 4-plane chunks at the end (HDA_TAIL_ROWS = 0 turns it off)
      static const int occ = [] {  // thread-safe one-time init
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, stencil7_kernel<T>, 256, 0);
        return o > 0 ? o : 4;
      }();
      zt = 4;
      const int64_t slots = (int64_t)sm_count_dev() * occ;
      int64_t tplanes = (slots + gx * gy - 1) / (gx * gy) * zt;
      tplanes = std::min<int64_t>(tplanes, nz / 4);
      nbig = (nz - tplanes) / S3_ZCH;
      const int64_t rest = nz - nbig * S3_ZCH;
      ntail = (rest + zt - 1) / zt;
    }
    dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)(nbig + ntail));
    // 1024^3 f32, 30 steps (profiles/r02/prefetch/): 0.822 (off) -> 0.886 (1) ->
    // 0.928-0.954 (2) -> 0.91 (3) -> 0.83-0.88 (4) -> 0.74 (6) of HBM with the halo
    // rows; 100 steps (power-capped): own rows 0.858-0.866 vs 0.826-0.832 with halos
    static const int pf = env_or("HDA_S7_PF", 2), pf_halo = env_or("HDA_S7_PF_HALO", 0);
    cudaError_t e = launch_pdl(stencil7_kernel<T>, grid, dim3(256), s, in, out, n1, n2, lb[0], ub[0], lb[1], ub[1],
                               lb[2], ub[2], xbase, nbig, zt, pf, pf_halo, ks);
    if (e != cudaSuccess) return e;
  } else {
    dim3 grid((unsigned)((ub[2] - lb[2] + 127) / 128), (unsigned)(ub[1] - lb[1]), (unsigned)(ub[0] - lb[0]));
    stencil7_scalar_kernel<T><<<grid, 128, 0, s>>>(in, out, n1, n2, lb[0], lb[1], ub[1], lb[2], ub[2], ks);
  }
  return cudaGetLastError();
}

cudaError_t launch_stencil7(int dtype, const void* in, void* out, const int64_t* shape, const int64_t* lb,
                            const int64_t* ub, const KSync& ks, cudaStream_t s) {
  if (dtype == 0) return launch_stencil7_t<double>((const double*)in, (double*)out, shape, lb, ub, ks, s);
  return launch_stencil7_t<float>((const float*)in, (float*)out, shape, lb, ub, ks, s);
}

// =====================================================================================
// elementwise: SCALE (X = alpha*X in X's arithmetic) and STAMP (splitmix64 raw bits)
// =====================================================================================

template <typename T>
__device__ __forceinline__ T scale1(T x, double a);
template <>
__device__ __forceinline__ double scale1(double x, double a) { return a * x; }
template <>
__device__ __forceinline__ float scale1(float x, double a) { return (float)a * x; }
template <>
__device__ __forceinline__ __nv_bfloat16 scale1(__nv_bfloat16 x, double a) {
  return __float2bfloat16_rn(__fmul_rn((float)a, __bfloat162float(x)));
}

// one block per (i0, i1) run of the box (grid-stride over runs); threads stride the
// contiguous dimension with 16-byte vectors on the aligned body, scalars on head/tail
template <typename T>
__global__ void __launch_bounds__(256) scale_kernel(T* x, int64_t n1, int64_t n2, int64_t lb0, int64_t lb1,
                                                    int64_t lb2, int64_t e1, int64_t e2, int64_t runs, double a,
                                                    const __grid_constant__ KSync ks) {
  ks_pre(ks);
  constexpr int V = 16 / sizeof(T);
  for (int64_t run = blockIdx.x; run < runs; run += gridDim.x) {
    const int64_t i0 = run / e1, i1 = run - i0 * e1;
    T* row = x + ((lb0 + i0) * n1 + (lb1 + i1)) * n2 + lb2;
    int64_t head = (int64_t)(((16 - ((uintptr_t)row & 15)) & 15) / sizeof(T));
    if (head > e2) head = e2;
    const int64_t nv = (e2 - head) / V;
    if (threadIdx.x < head) row[threadIdx.x] = scale1<T>(row[threadIdx.x], a);
    uint4* body = reinterpret_cast<uint4*>(row + head);
    for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
      uint4 u = body[v];
      T* e = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int t = 0; t < V; t++) e[t] = scale1<T>(e[t], a);
      body[v] = u;
    }
    for (int64_t t = head + nv * V + threadIdx.x; t < e2; t += blockDim.x) row[t] = scale1<T>(row[t], a);
  }
  ks_post(ks);
}

cudaError_t launch_scale(int dtype, void* x, const int64_t* shape, const int64_t* lb, const int64_t* ub,
                         double alpha, const KSync& ks, cudaStream_t s) {
  const int64_t e0 = ub[0] - lb[0], e1 = ub[1] - lb[1], e2 = ub[2] - lb[2];
  if (e0 <= 0 || e1 <= 0 || e2 <= 0) return cudaSuccess;
  const int64_t runs = e0 * e1;
  const unsigned grid = (unsigned)std::min<int64_t>(runs, 148 * 64);
  if (dtype == 0)
    scale_kernel<double><<<grid, 256, 0, s>>>((double*)x, shape[1], shape[2], lb[0], lb[1], lb[2], e1, e2, runs, alpha, ks);
  else if (dtype == 1)
    scale_kernel<float><<<grid, 256, 0, s>>>((float*)x, shape[1], shape[2], lb[0], lb[1], lb[2], e1, e2, runs, alpha, ks);
  else
    scale_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((__nv_bfloat16*)x, shape[1], shape[2], lb[0], lb[1], lb[2], e1,
                                                      e2, runs, alpha, ks);
  return cudaGetLastError();
}

// =====================================================================================
// Reduce (Table 2): fixed-order two-pass reduction -> deterministic
// =====================================================================================
template <typename T>
struct RedIn;
template <>
struct RedIn<double> {
  using A = double;
  __device__ static A get(double v) { return v; }
};
template <>
struct RedIn<float> {
  using A = double;
  __device__ static A get(float v) { return (double)v; }
};
template <>
struct RedIn<__nv_bfloat16> {
  using A = double;
  __device__ static A get(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
};
template <>
struct RedIn<int> {
  using A = long long;
  __device__ static A get(int v) { return (long long)v; }
};
template <>
struct RedIn<long long> {
  using A = long long;
  __device__ static A get(long long v) { return v; }
};

template <typename A>
__device__ __forceinline__ A red_id(int op) {
  if (op == 0) return A(0);
  if (op == 1) return A(1);
  if (op == 2) return sizeof(A) == 8 && A(0.5) != A(0) ? A(-__longlong_as_double(0x7FF0000000000000LL)) : A(0);
  return A(0);
}
template <>
__device__ __forceinline__ long long red_id<long long>(int op) {
  return op == 0 ? 0LL : op == 1 ? 1LL : op == 2 ? (long long)0x8000000000000000ULL : 0x7FFFFFFFFFFFFFFFLL;
}
template <>
__device__ __forceinline__ double red_id<double>(int op) {
  return op == 0 ? 0.0 : op == 1 ? 1.0 : op == 2 ? -__longlong_as_double(0x7FF0000000000000LL)
                                                  : __longlong_as_double(0x7FF0000000000000LL);
}
template <typename A>
__device__ __forceinline__ A red_op(int op, A a, A b) {
  if (op == 0) return a + b;
  if (op == 1) return a * b;
  if (op == 2) return b > a ? b : a;
  return b < a ? b : a;
}

template <typename A>
__device__ __forceinline__ A block_tree(A v, int op, A* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = red_op<A>(op, sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  return sh[0];
}

template <typename T>
__global__ void __launch_bounds__(256) reduce_box_kernel(const T* x, int64_t n1, int64_t n2, int64_t lb0, int64_t lb1,
                                                         int64_t lb2, int64_t e1, int64_t e2, int64_t runs, int op,
                                                         typename RedIn<T>::A* partial) {
  using A = typename RedIn<T>::A;
  __shared__ A sh[256];
  A acc = red_id<A>(op);
  for (int64_t run = blockIdx.x; run < runs; run += gridDim.x) {
    const int64_t i0 = run / e1, i1 = run - i0 * e1;
    const T* row = x + ((lb0 + i0) * n1 + (lb1 + i1)) * n2 + lb2;
    for (int64_t e = threadIdx.x; e < e2; e += blockDim.x) acc = red_op<A>(op, acc, RedIn<T>::get(row[e]));
  }
  A r = block_tree<A>(acc, op, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = r;
}

template <typename A>
__global__ void __launch_bounds__(256) reduce_final_kernel(const A* partial, int n, int op, A* out) {
  __shared__ A sh[256];
  A acc = red_id<A>(op);
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = red_op<A>(op, acc, partial[i]);
  A r = block_tree<A>(acc, op, sh);
  if (threadIdx.x == 0) *out = r;
}

template <typename T>
static cudaError_t reduce_t(const T* x, const int64_t* shape, const int64_t* lb, const int64_t* ub, int op,
                            void* scratch, void* result, cudaStream_t s) {
  using A = typename RedIn<T>::A;
  const int64_t e0 = ub[0] - lb[0], e1 = ub[1] - lb[1], e2 = ub[2] - lb[2];
  const int64_t runs = (e0 > 0 && e1 > 0 && e2 > 0) ? e0 * e1 : 0;
  reduce_box_kernel<T><<<kReduceBlocks, 256, 0, s>>>(x, shape[1], shape[2], lb[0], lb[1], lb[2], e1 > 0 ? e1 : 1,
                                                      e2, runs, op, (A*)scratch);
  reduce_final_kernel<A><<<1, 256, 0, s>>>((const A*)scratch, kReduceBlocks, op, (A*)result);
  return cudaGetLastError();
}

cudaError_t launch_reduce(int dtype, const void* x, const int64_t* shape, const int64_t* lb, const int64_t* ub,
                          int op, void* scratch, void* result, cudaStream_t s) {
  switch (dtype) {
    case 0: return reduce_t<double>((const double*)x, shape, lb, ub, op, scratch, result, s);
    case 1: return reduce_t<float>((const float*)x, shape, lb, ub, op, scratch, result, s);
    case 2: return reduce_t<__nv_bfloat16>((const __nv_bfloat16*)x, shape, lb, ub, op, scratch, result, s);
    case 3: return reduce_t<int>((const int*)x, shape, lb, ub, op, scratch, result, s);
    default: return reduce_t<long long>((const long long*)x, shape, lb, ub, op, scratch, result, s);
  }
}

__global__ void share_kernel(const unsigned long long* local, const __grid_constant__ SignalList slots,
                             const __grid_constant__ SignalList flags) {
  const int i = threadIdx.x;
  const unsigned long long v = *local;
  if (i < slots.n) {
    slots.ptr[i][0] = v;
    __threadfence_system();
    ks_st_release(flags.ptr[i], flags.val);
  }
}

cudaError_t launch_share(const unsigned long long* local, const SignalList& slots, const SignalList& flags,
                         cudaStream_t s) {
  if (slots.n <= 0) return cudaSuccess;
  share_kernel<<<1, kMaxDev, 0, s>>>(local, slots, flags);
  return cudaGetLastError();
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void stamp_kernel(char* x, int es, int64_t n1, int64_t n2, const __grid_constant__ BoxList bl,
                             unsigned long long seed, const __grid_constant__ KSync ks) {
  ks_pre(ks);
  const unsigned long long base = seed * 0x9E3779B97F4A7C15ULL;
  for (int b = 0; b < bl.n; b++) {
    const int64_t e0 = bl.ub[b][0] - bl.lb[b][0], e1 = bl.ub[b][1] - bl.lb[b][1], e2 = bl.ub[b][2] - bl.lb[b][2];
    const int64_t n = e0 * e1 * e2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i0 = t / (e1 * e2), r = t - i0 * e1 * e2, i1 = r / e2, i2 = r - i1 * e2;
      const int64_t c = ((bl.lb[b][0] + i0) * n1 + (bl.lb[b][1] + i1)) * n2 + (bl.lb[b][2] + i2);
      const unsigned long long h = splitmix64(base + (unsigned long long)c);
      char* p = x + c * es;
      if (es == 8) *reinterpret_cast<unsigned long long*>(p) = h;
      else if (es == 4) *reinterpret_cast<unsigned int*>(p) = (unsigned int)h;
      else *reinterpret_cast<unsigned short*>(p) = (unsigned short)h;
    }
  }
  ks_post(ks);
}

cudaError_t launch_stamp(int es, void* x, const int64_t* shape, const BoxList& boxes, unsigned long long seed,
                         const KSync& ks, cudaStream_t s) {
  if (boxes.n <= 0 && ks.nwait == 0 && ks.nsig == 0) return cudaSuccess;
  stamp_kernel<<<148 * 4, 256, 0, s>>>((char*)x, es, shape[1], shape[2], boxes, seed, ks);
  return cudaGetLastError();
}

}  // namespace hda
