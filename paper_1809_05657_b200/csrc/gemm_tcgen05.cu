// gemm_tcgen05.cu — the dense product of the paper's GEMM benchmark (Listing 2,
// P:L336-345): C[box] = alpha * A @ B + beta * C over a device's work box, bf16
// operands, fp32 accumulation in TMEM, on the 5th-generation tensor cores.
//
// Persistent warp-specialised kernel, one CTA per SM:
//   warp 0  TMA producer: A tile 128x64 (K-major) + B tile 64x256 (row-major B is
//           MN-major for UMMA) per stage, 128-byte swizzle, 4-stage mbarrier ring
//   warp 1  MMA issuer (one elected thread): tcgen05.mma.cta_group::1.kind::f16
//           M=128 N=256 K=16, accumulators double-buffered in TMEM (2 x 256 columns)
//   warp 2  TMEM allocator
//   warps 4-7  epilogue: tcgen05.ld 32x32b -> alpha*acc + beta*C -> f32/bf16 stores
// A and B replicas are full-size, so the tensor maps span whole arrays and
// the work box selects tiles; rows/cols outside the box are never stored.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kernels.cuh"
#include "sync.cuh"
#include "tcgen05_common.cuh"

namespace hda {

cudaError_t launch_gemm_simt(int c_dtype, const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                             const int64_t* lb, const int64_t* ub, float alpha, float beta, const KSync& ks,
                             cudaStream_t s);
cudaError_t launch_gemm_2sm(int c_dtype, const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                            const int64_t* lb, const int64_t* ub, float alpha, float beta, const KSync& ks,
                            cudaStream_t s, const KGate* gate);

namespace tc {

using namespace tcc;

constexpr int BM = 128, BN = 256, BK = 64, UK = 16;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;             // 16 KiB
constexpr int B_BYTES = BK * BN * 2;             // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // 48 KiB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int THREADS = 256;
constexpr int TMEM_COLS = 512;


__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// bounded wait: a protocol bug must end the kernel (wrong results, caught by the
// parity tests), never hang the GPU
__device__ unsigned int g_gemm_wait_timeouts = 0;
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
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
    if (ok) return;
    if (clock64() - t0 > (1LL << 34)) {  // ~8 s at 2 GHz
      atomicAdd(&g_gemm_wait_timeouts, 1u);
      return;
    }
  }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}


// instruction descriptor: D f32, A/B bf16, A K-major, B MN-major, M=128, N=256
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}


// Tile order: groups of GROUP_M M-tiles, N-major inside a group, so the ~148 tiles in
// flight share 16 A tiles and ~9 B tiles (both L2-resident) instead of streaming 148
// distinct A tiles per wave (measured 30.7 GB of DRAM reads for 1 GiB of operands).
constexpr int GROUP_M = 16;
__device__ __forceinline__ void tile_coords(int64_t t, int64_t tiles_m, int64_t tiles_n, int& mt, int& nt) {
  const int64_t per_group = (int64_t)GROUP_M * tiles_n;
  const int64_t g = t / per_group, local = t - g * per_group;
  const int64_t rows = min((int64_t)GROUP_M, tiles_m - g * GROUP_M);
  mt = (int)(g * GROUP_M + local % rows);
  nt = (int)(local / rows);
}

template <typename TC>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, TC* C,
                int64_t N, int64_t K, int64_t m0, int64_t m1, int64_t n0, int64_t n1, int64_t nbase, float alpha,
                float beta, const __grid_constant__ KSync ks) {
  ks_pre(ks);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t tiles_m = (m1 - m0 + BM - 1) / BM, tiles_n = (n1 - nbase + BN - 1) / BN;
  const int64_t n_tiles = tiles_m * tiles_n;
  const int kblocks = (int)((K + BK - 1) / BK);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        int mt, nt;
        tile_coords(t, tiles_m, tiles_n, mt, nt);
        const int row0 = (int)(m0 + (int64_t)mt * BM), col0 = (int)(nbase + (int64_t)nt * BN);
        for (int kb = 0; kb < kblocks; kb++) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(sa, &map_a, &full[s], kb * BK, row0);
#pragma unroll
          for (int j = 0; j < BN / 64; j++) tma_load_2d(sb + j * (BK * 128), &map_b, &full[s], col0 + 64 * j, kb * BK);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], aph ^ 1);
        fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < kblocks; kb++) {
          mbar_wait(&full[s], ph);
          fence_after();
          const uint32_t a_addr = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / UK; k++) {
            // A: K-major, advance 16 elements = 32 B inside the 128-B swizzled rows
            const uint64_t ad = smem_desc(a_addr + k * (UK * 2), 16, 1024);
            // B: MN-major, 16 K-rows = two 8-row atoms = 2048 B; 64-column blocks 8 KiB apart
            const uint64_t bd = smem_desc(b_addr + k * (UK * 128), BK * 128, 1024);
            mma_bf16(tmem_d, ad, bd, (kb | k) != 0);
          }
          mma_commit(&empty[s]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (TMEM lane quarter = warp % 4)
    const int q = warp % 4;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      int mt, nt;
      tile_coords(t, tiles_m, tiles_n, mt, nt);
      const int64_t row = m0 + (int64_t)mt * BM + q * 32 + lane;
      const int64_t colb = nbase + (int64_t)nt * BN;
      mbar_wait(&tfull[acc], aph);
      fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      for (int c = 0; c < BN / 32; c++) {
        uint32_t r[32];
        tmem_ld32(taddr + c * 32, r);
        if (row < m1) store_chunk<TC>(C + row * N, colb + c * 32, n0, n1, r, alpha, beta);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
  }
  ks_post(ks);
}

// ---------------------------------------------------------------- host side

}  // namespace tc

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_gemm(int c_dtype, const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                        const int64_t* lb, const int64_t* ub, float alpha, float beta, const KSync& ks,
                        cudaStream_t s, const KGate* gate) {
  const int64_t m0 = lb[1], m1 = ub[1], n0 = lb[2], n1 = ub[2];
  if (m0 >= m1 || n0 >= n1) return cudaSuccess;
  const bool gated = gate && (gate->n > 0 || gate->nseg > 0);  // flags or K ranges: CTA-pair kernel only
  // CTA-pair kernel (gemm_tcgen05_2sm.cu) by default: 16384^2 back-to-back 1655-1691
  // vs 1462-1482 TFLOP/s for this single-CTA kernel (HDA_GEMM_2SM=0 selects it)
  static const int two_sm = [] {
    const char* e = std::getenv("HDA_GEMM_2SM");
    return e ? std::atoi(e) : 1;
  }();
  if (two_sm) {
    const cudaError_t e = launch_gemm_2sm(c_dtype, A, B, C, M, N, K, lb, ub, alpha, beta, ks, s, gate);
    if (e != cudaErrorNotSupported) return e;
  }
  if (gated) return cudaErrorNotSupported;
  // TMA needs 16-byte row pitches and aligned bases; tiny problems use the CUDA-core path
  const bool tc_ok = (K % 8 == 0) && (N % 8 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) &&
                     K >= tc::BK && N >= 64 && M <= INT32_MAX && N <= INT32_MAX && K <= INT32_MAX;
  CUtensorMap ma, mb;
  if (!tc_ok || !tc::make_map(&ma, A, (uint64_t)K, (uint64_t)M, tc::BM) ||
      !tc::make_map(&mb, B, (uint64_t)N, (uint64_t)K, tc::BK))
    return launch_gemm_simt(c_dtype, A, B, C, M, N, K, lb, ub, alpha, beta, ks, s);
  // TMA inner coordinates must be 16-byte aligned (measured: an odd column offset traps
  // as an illegal instruction): tiles start at n0 rounded down to 8 columns, stores
  // still skip columns below n0
  const int64_t nbase = n0 & ~(int64_t)7;
  const int64_t tiles = ((m1 - m0 + tc::BM - 1) / tc::BM) * ((n1 - nbase + tc::BN - 1) / tc::BN);
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  if (c_dtype == 1) {
    cudaFuncSetAttribute(tc::gemm_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BYTES);
    tc::gemm_kernel<float><<<grid, tc::THREADS, tc::SMEM_BYTES, s>>>(ma, mb, (float*)C, N, K, m0, m1, n0, n1, nbase,
                                                                     alpha, beta, ks);
  } else {
    cudaFuncSetAttribute(tc::gemm_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         tc::SMEM_BYTES);
    tc::gemm_kernel<__nv_bfloat16><<<grid, tc::THREADS, tc::SMEM_BYTES, s>>>(ma, mb, (__nv_bfloat16*)C, N, K, m0,
                                                                             m1, n0, n1, nbase, alpha, beta, ks);
  }
  return cudaGetLastError();
}

}  // namespace hda
