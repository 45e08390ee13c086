// kernels.cuh — launch interfaces of the sm_100a kernels (library-internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hda {

// One strided rectangle copy, raw bytes: n0 x n1 runs of run_bytes contiguous bytes.
// Run (i0, i1) starts at src + src_off + i0*src_p0 + i1*src_p1 (same for dst).
// Used for the fused pull (peer replica -> local replica, same offsets on both sides:
// pack + NVLink transfer + unpack in one pass), for pack (replica -> contiguous
// staging), unpack (staging -> replica) and the COPY kernel (replica -> replica).
struct RunDesc {
  const char* src;
  char* dst;
  int64_t src_off, dst_off;
  int64_t src_p0, dst_p0;
  int64_t src_p1, dst_p1;
  int64_t run_bytes;
  int64_t unit_begin;   // first work unit of this descriptor (prefix sum)
  int32_t n0, n1;
  int32_t es;           // element size: granularity of heads/tails/misaligned copies
  int32_t chunks;       // >0: long runs, chunks per run (one warp per chunk)
                        // 0 : short runs, 32 runs per unit (one thread per run)
  int64_t chunk_bytes;  // bytes per chunk (multiple of 512)
};

constexpr int kMaxRunDescs = 8;  // per launch (kernel parameters stay small)
struct RunBatch {
  RunDesc d[kMaxRunDescs];
  int32_t n;
  int64_t total_units;
};
constexpr int64_t kChunkBytes = 8192;

// sets chunks/chunk_bytes and returns the number of units of one descriptor;
// chunk_bytes adapts so that small payloads still spread over many warps
int64_t run_desc_units(RunDesc& d, int64_t chunk_bytes);
int64_t pick_chunk_bytes(int64_t total_bytes);

// cross-device ordering words (see hda.cpp "sync protocol")
constexpr int kMaxDev = 64;
struct WaitList {
  unsigned long long* ptr[kMaxDev];
  unsigned long long val[kMaxDev];
  int32_t n;
};
struct SignalList {
  unsigned long long* ptr[kMaxDev];
  int32_t n;
  unsigned long long val;
};

// in-kernel cross-device ordering (sync.cuh); nwait == nsig == 0 means "none"
constexpr int kKSync = kMaxDev;
struct KSync {
  unsigned long long* wait_ptr[kKSync];
  unsigned long long wait_val[kKSync];
  unsigned long long* sig_ptr[kKSync];
  unsigned long long sig_val;
  unsigned int* ctr;
  int* err;
  long long timeout_ns;
  int32_t nwait, nsig;
  int32_t relaxed;  // experiment: signal with st.relaxed.sys after a gpu-scope fence
  long long delay_ns;  // test hook (HDA_DEBUG_PULL_DELAY_US): pulls sleep after their waits
};

struct BoxList {  // boxes in element coordinates of a 3-D padded shape
  int64_t lb[16][3];
  int64_t ub[16][3];
  int32_t n;
};

cudaError_t launch_copy_runs(const RunBatch& b, const KSync& ks, cudaStream_t s);
cudaError_t launch_wait(const WaitList& w, int* err_flag, long long timeout_ns, cudaStream_t s);
cudaError_t launch_signal(const SignalList& l, cudaStream_t s);
// after the previous kernel on s completes (programmatic dependent launch)
cudaError_t launch_signal_pdl(const SignalList& l, int relaxed, cudaStream_t s);

// user kernels over the work box [lb, ub) of one device's replica (padded 3-D shape)
// 2-D stencils over nb (<= 8) boxes in ONE launch (lbs[i], ubs[i] front-padded 3-D)
// Fused halo-exchange 2-D stencil (kernel 1 = JACOBI5, 3 = STENCIL9): pulls `pull`
// (peer replica -> this replica) in its first blocks, then computes boxes
// [0, n_interior) immediately and boxes [n_interior, nb) after the pull — one launch.
struct HaloPull {
  unsigned long long* wait_ptr[16];  // local PROD words of the sources, then the pull's WAR ACK words
  unsigned long long wait_val[16];
  unsigned long long* ack_ptr[8];   // sources' ACK words for this reader
  int32_t nwait, nack;
  unsigned int* ctr;                // local counter
  unsigned long long* done_word;    // local "pull done" word
  unsigned long long epoch;
  long long delay_ns;               // test hook (see KSync::delay_ns)
};
cudaError_t launch_stencil2d_halo(int kernel, int dtype, const void* in, void* out, const int64_t* shape,
                                  const int64_t* const* lbs, const int64_t* const* ubs, int nb, int n_interior,
                                  const RunBatch& pull, const HaloPull& hp, const KSync& ks, cudaStream_t s);
// TMA-ring 2-D stencil over ONE work box (stencil_tma.cu): kind 0 = JACOBI5, 1 = STENCIL9;
// cudaErrorNotSupported when the box/layout does not qualify (caller uses the register
// march).  stencil_tma_mode(): HDA_TMA, 0 off, 1 (default) 9-point only, 2 both.
cudaError_t launch_stencil2d_tma(int kind, int dtype, const void* in, void* out, const int64_t* shape,
                                 const int64_t* lb, const int64_t* ub, const KSync& ks, cudaStream_t s);
int stencil_tma_mode();
// up to 8 boxes in one launch (flat grid of tiles)
cudaError_t launch_jacobi5(int dtype, const void* in, void* out, const int64_t* shape,
                           const int64_t* const* lbs, const int64_t* const* ubs, int nb, const KSync& ks,
                           cudaStream_t s);
cudaError_t launch_stencil9(int dtype, const void* in, void* out, const int64_t* shape,
                            const int64_t* const* lbs, const int64_t* const* ubs, int nb, const KSync& ks,
                            cudaStream_t s);
cudaError_t launch_stencil7(int dtype, const void* in, void* out, const int64_t* shape,
                            const int64_t* lb, const int64_t* ub, const KSync& ks, cudaStream_t s);
cudaError_t launch_scale(int dtype, void* x, const int64_t* shape, const int64_t* lb,
                         const int64_t* ub, double alpha, const KSync& ks, cudaStream_t s);
cudaError_t launch_stamp(int es, void* x, const int64_t* shape, const BoxList& boxes,
                         unsigned long long seed, const KSync& ks, cudaStream_t s);
// Reduce: deterministic two-pass reduction of a box (fp64 accumulation, int64 for
// integer dtypes) into *result (8 bytes); op 0 SUM 1 PROD 2 MAX 3 MIN.  `scratch` holds
// kReduceBlocks partials.
constexpr int kReduceBlocks = 592;
cudaError_t launch_reduce(int dtype, const void* x, const int64_t* shape, const int64_t* lb, const int64_t* ub,
                          int op, void* scratch, void* result, cudaStream_t s);
// SPMD combine: copy *local (8 bytes) to every peer slot, then release `val` to their flags
cudaError_t launch_share(const unsigned long long* local, const SignalList& slots, const SignalList& flags,
                         cudaStream_t s);
// All-gather fused into the product (P:L424's B all-gather; 2MM's D): rows
// [lo[i], hi[i]) of B arrive from source i while the GEMM runs, and flag[i] reaches
// val[i] once they have landed in this replica (a stream write after the copy-engine
// copy).  The producers wait for a source's flag before the first TMA load that touches
// its rows.  K is walked in segments [skb0[j], skb1[j]) (k-blocks of 64, together
// exactly [0, K/64)), resident rows first, then the sources in arrival order.  multi:
// one pass over all output tiles per segment, each pass adding its partial product to C
// (fp32 C only), so the resident rows' work covers the first copies instead of every
// tile stalling on its first remote k-block.  n == 0 and nseg == 0: no gating, all of K;
// n == 0 and nseg > 0: only the listed K ranges, in one pass, no flags (the split form).
constexpr int kMaxGate = 16;
struct KGate {
  int32_t n, nseg, multi, pad_;
  int64_t lo[kMaxGate], hi[kMaxGate];
  const unsigned long long* flag[kMaxGate];
  unsigned long long val[kMaxGate];
  int32_t skb0[kMaxGate + 1], skb1[kMaxGate + 1];
};

// C[rows lb0..ub0, cols lb1..ub1] = alpha * A@B + beta*C ; A [M,K] bf16 row-major,
// B [K,N] bf16 row-major, C [M,N] f32 or bf16 row-major (full-array strides).
// A gated launch (gate && gate->n > 0) runs only on the CTA-pair kernel:
// cudaErrorNotSupported otherwise, and the caller joins the copies and launches ungated.
cudaError_t launch_gemm(int c_dtype, const void* A, const void* B, void* C, int64_t M, int64_t N,
                        int64_t K, const int64_t* lb, const int64_t* ub, float alpha, float beta,
                        const KSync& ks, cudaStream_t s, const KGate* gate = nullptr);

}  // namespace hda
