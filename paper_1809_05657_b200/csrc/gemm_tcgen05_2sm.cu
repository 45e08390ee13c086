// gemm_tcgen05_2sm.cu — the product of Listing 2 on CTA pairs:
// tcgen05.mma.cta_group::2, M=256 (128 rows per CTA) x N=256 x K=16, so each SM
// stages A for its own 128 rows and only HALF of B (128 columns): 32 KiB per stage per
// CTA instead of 48, one third less L2->SM traffic than the single-CTA kernel.
//
// Cluster of 2 CTAs (one per SM of a TPC), persistent over 256x256 tiles:
//   warp 0  TMA producer (both CTAs): A 128x64 + B 64x128 per stage into its own smem,
//           completion counted on the LEADER's full barrier (.cta_group::2 TMA)
//   warp 1  MMA issuer (leader CTA only), commits multicast to both CTAs' barriers
//   warp 2  TMEM allocator (both CTAs, .cta_group::2, 2 x 256 columns)
//   warps 4-7  epilogue (both CTAs): each CTA drains its 128 rows of the accumulator
// Every mbarrier wait is bounded; a timeout aborts the whole grid quickly (wrong
// results, caught by the parity tests) instead of hanging the GPU.
// Optionally gated (KGate): B rows still arriving over NVLink are waited for per
// k-block by the producers, so the all-gather of B overlaps the product.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "sync.cuh"
#include "tcgen05_common.cuh"

namespace hda {
namespace tc2 {

using namespace tcc;

constexpr int BM = 128;   // rows per CTA (the pair covers 256)
constexpr int BN = 256;   // accumulator columns (each CTA stages 128 of B)
constexpr int BNH = 128;  // B columns staged per CTA
constexpr int BK = 64, UK = 16;
#ifndef GEMM2_STAGES
#define GEMM2_STAGES 6
#endif
#ifndef GEMM2_GROUP_M
#define GEMM2_GROUP_M 8
#endif
constexpr int STAGES = GEMM2_STAGES;
constexpr int A_BYTES = BM * BK * 2;            // 16 KiB
constexpr int B_BYTES = BK * BNH * 2;           // 16 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 32 KiB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int THREADS = 256;
constexpr int TMEM_COLS = 512;

__device__ int g_abort = 0;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ bool aborted() { return *reinterpret_cast<volatile int*>(&g_abort) != 0; }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// bounded wait; the abort flag (a global load) is polled only while a wait is slow,
// never on the fast path.  CLUSTER: acquire at cluster scope (remote arrivals).
template <bool CLUSTER = false>
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  for (int spin = 0;; spin++) {
    if (CLUSTER)
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n}"
          : "=r"(ok)
          : "r"(smem_u32(b)), "r"(parity)
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n}"
          : "=r"(ok)
          : "r"(smem_u32(b)), "r"(parity)
          : "memory");
    if (ok) return;
    if ((spin & 1023) == 1023) {
      if (aborted()) return;
      if (spin > (1 << 22)) {  // seconds: a protocol bug; stop the grid
        atomicExch(&g_abort, 1);
        return;
      }
    }
  }
}

// TMA into this CTA's smem, completion bytes counted on `bar` (the leader's barrier)
__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}

// Gated K (all-gather fused into the product, kernels.cuh KGate): before the first TMA
// load of k-block kb, wait for every source whose rows [lo, hi) meet it.  `ready` keeps
// the sources already seen for the rest of the launch.  The acquire of the flag orders
// the copy-engine writes before it (the stream write that set it carries a system
// fence); the proxy fence extends that order to the TMA (async proxy) reads that follow.
__device__ __forceinline__ void gate_wait(const KGate& g, int kb, uint32_t& ready) {
  const int64_t k0 = (int64_t)kb * BK, k1 = k0 + BK;
  bool waited = false;
  for (int i = 0; i < g.n; i++) {
    if ((ready >> i) & 1u) continue;
    if (g.lo[i] >= k1 || g.hi[i] <= k0) continue;
    for (long long spin = 0;; spin++) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(g.flag[i]) : "memory");
      if (v >= g.val[i]) break;
      if ((spin & 255) == 255) {
        if (aborted()) return;
        if (spin > (1LL << 26)) {  // seconds: the copies never landed; stop the grid
          atomicExch(&g_abort, 1);
          return;
        }
        __nanosleep(256);
      }
    }
    ready |= 1u << i;
    waited = true;
  }
  if (waited) asm volatile("fence.proxy.async.global;" ::: "memory");
}

// D f32, A/B bf16, A K-major, B MN-major, M = 256 (the pair), N = 256
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)((2 * BM) >> 4) << 24);

__device__ __forceinline__ void mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
// arrive on the barrier at this smem offset in BOTH CTAs once the MMAs issued so far complete
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}


constexpr int GROUP_M = GEMM2_GROUP_M;  // 256-row tiles per group (grouped raster, L2 reuse)
__device__ __forceinline__ void tile_coords(int64_t t, int64_t tiles_m, int64_t tiles_n, int& mt, int& nt) {
  const int64_t per_group = (int64_t)GROUP_M * tiles_n;
  const int64_t g = t / per_group, local = t - g * per_group;
  const int64_t rows = min((int64_t)GROUP_M, tiles_m - g * GROUP_M);
  mt = (int)(g * GROUP_M + local % rows);
  nt = (int)(local / rows);
}

template <typename TC>
__global__ void __launch_bounds__(THREADS, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, TC* C,
                 int64_t N, int64_t K, int64_t m0, int64_t m1, int64_t n0, int64_t n1, int64_t nbase, float alpha,
                 float beta, const __grid_constant__ KSync ks, const __grid_constant__ KGate gate) {
  ks_pre(ks);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2] (leader's are the ones used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int64_t tiles_m = (m1 - m0 + 2 * BM - 1) / (2 * BM), tiles_n = (n1 - nbase + BN - 1) / BN;
  const int64_t n_tiles = tiles_m * tiles_n;
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  // K segments (KGate): one pass over the tiles per segment when the output is fp32 and
  // the launch is gated (each pass accumulates into C), else one pass over all of them
  const bool multi = gate.multi != 0;
  const int npass = multi ? gate.nseg : 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);   // the leader's producer arrives (expect_tx of both CTAs)
      mbar_init(&empty[s], 1);  // one multicast commit per use
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's barrier)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
  }
  if (warp == 2) {  // same warp in both CTAs (joint allocation)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      const uint32_t full0 = mapa(smem_u32(&full[0]), 0);  // the leader's full[0]
      int s = 0;
      uint32_t ph = 0;
      uint32_t ready = 0;
      for (int pp = 0; pp < npass && !aborted(); pp++) {
        for (int64_t t = cid; t < n_tiles && !aborted(); t += ncl) {  // abort checked per tile only
          int mt, nt;
          tile_coords(t, tiles_m, tiles_n, mt, nt);
          const int row0 = (int)(m0 + (int64_t)mt * 2 * BM + rank * BM);
          const int col0 = (int)(nbase + (int64_t)nt * BN + rank * BNH);
          // K order: the segments of this pass (all of them when one pass covers K); the
          // MMA issuer only counts blocks, so the order changes nothing else
          for (int sg = multi ? pp : 0; sg < (multi ? pp + 1 : gate.nseg); sg++) {
            for (int kb = gate.skb0[sg]; kb < gate.skb1[sg]; kb++) {
              if (gate.n > 0) gate_wait(gate, kb, ready);
              mbar_wait(&empty[s], ph ^ 1);
              uint8_t* sa = smem + s * STAGE_BYTES;
              uint8_t* sb = sa + A_BYTES;
              if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
              const uint32_t fb = full0 + (uint32_t)(s * sizeof(uint64_t));
              tma_load_2sm(sa, &map_a, fb, kb * BK, row0);
#pragma unroll
              for (int j = 0; j < BNH / 64; j++)
                tma_load_2sm(sb + j * (BK * 128), &map_b, fb, col0 + 64 * j, kb * BK);
              if (++s == STAGES) {
                s = 0;
                ph ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader only)
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int pp = 0; pp < npass && !aborted(); pp++) {
        int nkb = 0;  // k-blocks per tile in this pass (all segments when one pass walks them)
        for (int sg = multi ? pp : 0; sg < (multi ? pp + 1 : gate.nseg); sg++) nkb += gate.skb1[sg] - gate.skb0[sg];
        for (int64_t t = cid; t < n_tiles && !aborted(); t += ncl) {
          mbar_wait<true>(&tempty[acc], aph ^ 1);  // arrivals from both CTAs' epilogues
          fence_after();
          const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
          for (int i = 0; i < nkb; i++) {
            mbar_wait(&full[s], ph);
            fence_after();
            const uint32_t a_addr = smem_u32(smem + s * STAGE_BYTES);
            const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / UK; k++) {
              const uint64_t ad = smem_desc(a_addr + k * (UK * 2), 16, 1024);
              const uint64_t bd = smem_desc(b_addr + k * (UK * 128), BK * 128, 1024);
              mma2(tmem_d, ad, bd, (i | k) != 0);
            }
            commit_both(&empty[s]);
            if (++s == STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
          commit_both(&tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            aph ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs; TMEM lane quarter = warp % 4)
    const int q = warp % 4;
    const uint32_t tempty0 = mapa(smem_u32(&tempty[0]), 0);
    int acc = 0;
    uint32_t aph = 0;
    for (int pp = 0; pp < npass && !aborted(); pp++) {
      // later passes add their K segment to what the earlier ones stored; the same
      // thread stores and re-reads each element, so program order suffices
      const float b = pp == 0 ? beta : 1.f;
      for (int64_t t = cid; t < n_tiles && !aborted(); t += ncl) {
        int mt, nt;
        tile_coords(t, tiles_m, tiles_n, mt, nt);
        const int64_t row = m0 + (int64_t)mt * 2 * BM + rank * BM + q * 32 + lane;
        const int64_t colb = nbase + (int64_t)nt * BN;
        mbar_wait(&tfull[acc], aph);
        fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
        for (int c = 0; c < BN / 32; c++) {
          uint32_t r[32];
          tmem_ld32(taddr + c * 32, r);
          if (row < m1) store_chunk<TC>(C + row * N, colb + c * 32, n0, n1, r, alpha, b);
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + (uint32_t)(acc * sizeof(uint64_t)));
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
  }
  // an aborted grid (a wait that never completed) surfaces as the sticky HDA_ETIMEOUT
  if (threadIdx.x == 0 && ks.err && aborted()) *reinterpret_cast<volatile int*>(ks.err) = -7;
  ks_post(ks);
}

template <typename TC>
static cudaError_t launch_t(const CUtensorMap& ma, const CUtensorMap& mb, TC* C, int64_t N, int64_t K, int64_t m0,
                            int64_t m1, int64_t n0, int64_t n1, float alpha, float beta, const KSync& ks,
                            cudaStream_t s, int sms, const KGate& gate) {
  const int64_t nbase = n0 & ~(int64_t)7;  // 16-byte aligned TMA column base (see gemm_tcgen05.cu)
  const int64_t tiles = ((m1 - m0 + 2 * BM - 1) / (2 * BM)) * ((n1 - nbase + BN - 1) / BN);
  const int clusters = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, sms / 2));
  cudaFuncSetAttribute(gemm2_kernel<TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm2_kernel<TC>, ma, mb, C, N, K, m0, m1, n0, n1, nbase, alpha, beta, ks, gate);
}

}  // namespace tc2

// Returns cudaErrorNotSupported when the 2-SM path does not apply (caller falls back).
cudaError_t launch_gemm_2sm(int c_dtype, const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                            const int64_t* lb, const int64_t* ub, float alpha, float beta, const KSync& ks,
                            cudaStream_t s, const KGate* gate) {
  const int64_t m0 = lb[1], m1 = ub[1], n0 = lb[2], n1 = ub[2];
  const bool ok = (K % 8 == 0) && (N % 8 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) &&
                  K >= tc2::BK && N >= 128 && M <= INT32_MAX && N <= INT32_MAX && K <= INT32_MAX &&
                  (m1 - m0) >= 2 * tc2::BM;
  CUtensorMap ma, mb;
  if (!ok || !tc2::make_map(&ma, A, (uint64_t)K, (uint64_t)M, tc2::BM) ||
      !tc2::make_map(&mb, B, (uint64_t)N, (uint64_t)K, tc2::BK))
    return cudaErrorNotSupported;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  KGate g;
  std::memset(&g, 0, sizeof g);
  const int kblocks = (int)((K + tc2::BK - 1) / tc2::BK);
  g.nseg = 1;
  g.skb1[0] = kblocks;
  if (gate && gate->n > 0) {
    if (gate->n > kMaxGate) return cudaErrorNotSupported;
    g = *gate;
    // segments: k-blocks ordered by the arrival rank of the last source they need
    // (-1 = resident), ties by k; runs of consecutive k-blocks with one rank
    std::vector<int> rdy(kblocks, -1);
    for (int i = 0; i < g.n; i++)
      for (int64_t kb = g.lo[i] / tc2::BK; kb < kblocks && kb * tc2::BK < g.hi[i]; kb++) rdy[kb] = i;
    std::vector<int> order(kblocks);
    for (int kb = 0; kb < kblocks; kb++) order[kb] = kb;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rdy[a] < rdy[b]; });
    int ns = 0;
    for (int j = 0; j < kblocks; j++) {
      const int kb = order[j];
      if (ns > 0 && g.skb1[ns - 1] == kb && rdy[g.skb0[ns - 1]] == rdy[kb]) {
        g.skb1[ns - 1] = kb + 1;
        continue;
      }
      if (ns == kMaxGate + 1) return cudaErrorNotSupported;
      g.skb0[ns] = kb;
      g.skb1[ns] = kb + 1;
      ns++;
    }
    g.nseg = ns;
    // per-segment passes: fp32 C only (a bf16 C would be rounded once per pass)
    static const int multi = [] {
      const char* e = std::getenv("HDA_GATE_PASSES");
      return e ? std::atoi(e) : 1;
    }();
    g.multi = (multi && c_dtype == 1 && ns > 1) ? 1 : 0;
  } else if (gate && gate->nseg > 0) {
    // explicit K ranges, no arrival flags (the two-launch split of a gated product)
    if (gate->nseg > kMaxGate + 1) return cudaErrorNotSupported;
    g = *gate;
    g.n = 0;
    for (int j = 0; j < g.nseg; j++)
      if (g.skb0[j] < 0 || g.skb1[j] > kblocks || g.skb0[j] >= g.skb1[j]) return cudaErrorInvalidValue;
  } else {
    // measurement hook: HDA_DEBUG_GEMM_SEGS=s splits an ungated K into s passes (fp32 C)
    static const int dbg = [] {
      const char* e = std::getenv("HDA_DEBUG_GEMM_SEGS");
      return e ? std::atoi(e) : 0;
    }();
    if (dbg > 1 && dbg <= kMaxGate && c_dtype == 1 && kblocks >= dbg) {
      g.nseg = dbg;
      g.multi = 1;
      for (int j = 0; j < dbg; j++) {
        g.skb0[j] = (int)((int64_t)kblocks * j / dbg);
        g.skb1[j] = (int)((int64_t)kblocks * (j + 1) / dbg);
      }
    }
  }
  if (c_dtype == 1)
    return tc2::launch_t<float>(ma, mb, (float*)C, N, K, m0, m1, n0, n1, alpha, beta, ks, s, sms, g);
  return tc2::launch_t<__nv_bfloat16>(ma, mb, (__nv_bfloat16*)C, N, K, m0, m1, n0, n1, alpha, beta, ks, s, sms, g);
}

}  // namespace hda
