// hda.cpp — runtime and C-ABI of the B200-native HDArray hot path (see include/hdarray.h).
//
// Per hda_apply (Table 2 ApplyKernel):
//   1. tracker: compose LUSE/LDEF + plan (Eq. 1-2), or a plan-cache hit
//   2. exchange: every planned rectangle moves from its last writer to its reader
//      FUSED : one copy kernel on the reader's GPU loads the writer's replica through
//              NVLink peer memory and stores into its own replica (pack + transfer +
//              unpack in one pass, no staging)
//      STAGED: pack kernel on the writer -> copy engine -> unpack kernel on the reader
//   3. the built-in kernel on every local device's work box
//   4. tracker commit (Eq. 3-4 corrected), on the host while the GPUs run
//
// Sync protocol (no host barriers; works across processes through CUDA IPC):
// every device d owns 192 monotone 64-bit words in its own HBM:
//   PROD[p]  = last call epoch whose kernel/write on device p has completed (written by p)
//   PACK[p]  = last epoch for which p's staged payload for d is packed     (written by p)
//   ACK[r]   = last epoch at which device r finished reading from d       (written by r)
// A reader waits PROD[p] >= epoch of p's last definition before pulling (RAW); a
// writer waits ACK[r] >= epoch of r's last pull before overwriting (WAR).  Waits are
// 1-block spin kernels with a timeout (sticky HDA_ETIMEOUT, never a hang); signals
// are release stores at system scope.  Devices that share a CUDA stream (virtual
// devices on one GPU) are ordered by the stream and skip both.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hdarray.h"
#include "kernels.cuh"
#include "tracker.hpp"

using namespace hda;

namespace {

constexpr int SW_PROD = 0, SW_PACK = 64, SW_ACK = 128, SW_CTR_PULL = 192, SW_CTR_KERN = 193;
constexpr int SW_PULLDONE = 194;  // local: epoch of the last completed overlapped pull
constexpr int SW_RED = 256, SW_REDSIG = 320;  // reduce partials [P] and their epochs [P]
constexpr int SW_DEBUG = 195;                  // measurement hooks only
constexpr int SW_SCRATCH = 384;               // kReduceBlocks partials
constexpr int SW_RED_B = SW_SCRATCH + kReduceBlocks;  // second bank of reduce partials [P]
constexpr int SW_GATE = SW_RED_B + 64;  // [P] local: epoch at which source p's gated GEMM rows landed
constexpr int SW_WORDS = SW_GATE + 64;
constexpr uint32_t BLOB_MAGIC = 0x48444131u;  // "HDA1"
constexpr int64_t kCeBytes = 1 << 20;         // AUTO: messages >= 1 MiB go to the copy engine

struct Gpu {
  int ordinal = 0;
  cudaStream_t stream = nullptr;  // compute (and everything else)
  cudaStream_t comm = nullptr;    // overlapped halo pulls
  cudaEvent_t ev_fork = nullptr, ev_pull = nullptr;
  cudaEvent_t ev_src[kMaxGate] = {};  // gated pull: source i's block has landed
};

struct Dev {
  bool local = false;
  int gpu = -1;                        // index into ctx->gpus (local devices)
  unsigned long long* sync = nullptr;  // this device's sync words (local or IPC-mapped)
  bool sync_alloc = false, sync_ipc = false;
};

struct ArrRT {
  std::vector<char*> ptr;  // per device: local replica, IPC-mapped peer replica, or null
  std::vector<char> alloc, ipc;
  bool imported = false;
  size_t bytes = 0;
};

struct TimedEv {
  int kind;  // kernel id, or -100 for exchange
  cudaEvent_t a, b;
  int count;  // 1 for the first launch of a call, 0 for its continuation launches
  unsigned long long epoch;
  int dev, phase;  // phase: 0 exchange, 1 kernel (whole), 2 interior, 3 dependent
};

struct PullJob {
  int dst;
  std::vector<int> srcs;
  std::vector<RunBatch> batches;
  std::vector<std::pair<int, int>> pend;  // (array, src) pairs read by this pull
  bool cross = false;                     // some source lives on another stream/GPU
  // overlap split of the reader's work box: cells whose footprint does not touch any
  // incoming rectangle (run while the pull is in flight) and the rest (after it)
  bool split = false;
  std::vector<Box> interior, dependent;
  std::vector<cudaMemcpy3DParms> ce;  // AUTO transport: bulk messages on the copy engine
  std::vector<int> ce_src;            // source device of each ce copy
  // GEMM whose incoming messages are whole row blocks of B, all on the copy engine: the
  // product runs gated on their arrival (KGate) instead of after a join; rows [lo, hi)
  // of B per srcs[i]
  bool gate = false;
  std::vector<std::pair<int64_t, int64_t>> gate_rows;
  int64_t gate_k = 0;  // rows of B (the product's K)
};
struct PendEntry {
  int array, src, dst;
};
struct PackJob {
  int src;
  std::vector<int> dsts;
  std::vector<RunBatch> batches;
  size_t bytes = 0;
};
struct Seg {
  int src;
  size_t src_off, dst_off, bytes;
};
struct RecvJob {
  int dst;
  std::vector<int> srcs;
  std::vector<Seg> segs;
  std::vector<RunBatch> unpack;
  size_t bytes = 0;
};
struct ExecPlan {
  bool staged = false;
  int transport = HDA_XPORT_FUSED;
  std::vector<PullJob> pulls;
  std::vector<PackJob> packs;
  // every (array, src, dst) read of this call, local reader or not: in SPMD the writer's
  // rank must know its REMOTE readers too, to wait for their ACKs before overwriting
  std::vector<PendEntry> reads;
  std::vector<RecvJob> recvs;
};

}  // namespace

// One host thread per GPU for single-process contexts: a call's launches for the
// devices of different GPUs are issued concurrently (each GPU's own order is kept;
// across GPUs the device-side sync words order everything, as between SPMD ranks).
// Measured serial issue: ~10 us per device per call, i.e. host-bound beyond ~4 GPUs.
// Workers spin briefly between calls, then sleep on a condition variable.
class IssuePool {
 public:
  explicit IssuePool(const std::vector<int>& ordinals) : ord_(ordinals), rcs_(ordinals.size(), 0) {
    for (size_t g = 0; g < ord_.size(); g++) th_.emplace_back([this, g] { worker((int)g); });
  }
  ~IssuePool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // fn(gpu index) on every worker; returns the first nonzero result
  int run(const std::function<int(int)>& fn) {
    task_ = &fn;
    remaining_.store((int)ord_.size(), std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    while (remaining_.load(std::memory_order_acquire) > 0) std::this_thread::yield();
    for (int r : rcs_)
      if (r) return r;
    return 0;
  }

 private:
  void worker(int g) {
    cudaSetDevice(ord_[g]);
    uint64_t seen = 0;
    for (;;) {
      int spins = 0;
      uint64_t cur;
      while ((cur = gen_.load(std::memory_order_acquire)) == seen && !stop_.load()) {
        if (++spins < 4096) {
          std::this_thread::yield();
        } else {
          std::unique_lock<std::mutex> lk(mu_);
          cv_.wait(lk, [&] { return gen_.load() != seen || stop_.load(); });
          spins = 0;
        }
      }
      if (stop_.load()) return;
      seen = cur;
      rcs_[g] = (*task_)(g);
      remaining_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<int> ord_;
  std::vector<int> rcs_;
  std::vector<std::thread> th_;
  const std::function<int(int)>* task_ = nullptr;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> remaining_{0};
  std::atomic<bool> stop_{false};
  std::mutex mu_;
  std::condition_variable cv_;
};

struct hda_ctx {
  int P = 0;
  bool spmd = false, plan_only = false, sync_imported = true;
  int rank = -1;
  std::vector<Gpu> gpus;
  std::vector<Dev> dev;
  std::unique_ptr<Tracker> tr;
  std::vector<ArrRT> arr;
  unsigned long long epoch = 0;
  std::vector<unsigned long long> last_prod;
  std::vector<std::vector<std::vector<unsigned long long>>> pend;  // [array][src][dst]
  // [array][dev]: boxes peers pulled from dev's replica since dev last wrote the array
  // (per-box WAR: kernel parts disjoint from them need no WAR wait); over => unknown
  std::vector<std::vector<std::vector<Box>>> rread;
  std::vector<std::vector<char>> rread_over;
  std::vector<int> split_mode;  // per device: 2 = this call's boundary part ran on the comm stream
  // [P] WAR waits of this call's pull into device q's replica: (ACK word, epoch) of the
  // peers that pulled those cells from q earlier and may still be reading them
  std::vector<std::vector<std::pair<unsigned long long*, unsigned long long>>> pull_war;
  unsigned long long n_reduce = 0;  // reduce calls so far (identical on every SPMD rank)
  std::vector<char> war_done;   // per device: WAR waits already issued for this call
  std::vector<std::vector<std::pair<int, unsigned long long>>> stage_pend;  // [src]
  std::vector<char*> send_stage, recv_stage;
  std::vector<size_t> send_cap, recv_cap;
  std::unordered_map<uint64_t, ExecPlan> exec;
  int transport = HDA_XPORT_AUTO;
  bool cache_on = true, ktiming = false, overlap = true, tracing = false;
  std::vector<TimedEv> trace;  // kept (not drained) while tracing
  cudaEvent_t trace_ref = nullptr;
  int cur_dev = 0, cur_phase = 1;
  std::vector<char> pulled_on_comm;  // [P] this call's pull for device q ran on the comm stream
  std::vector<const PullJob*> cur_pull;
  std::vector<const PullJob*> halo_job;  // [P] pull deferred into the fused halo-stencil launch
  std::vector<KGate> gate;               // [P] this call's gated product (issue_gated_pull)
  std::vector<char> gated;               // [P] gate[q] is armed for this call
  std::vector<TimedEv> tev;
  std::vector<cudaEvent_t> ev_pool;
  double ktime_ms[KN_COUNT] = {};
  int64_t kcount[KN_COUNT] = {};
  double xtime_ms = 0;
  int64_t xcount = 0;
  int* err_host = nullptr;
  int sticky = 0;
  std::string err;
  hda_stats_t stats{};
  std::mutex err_mu;
  std::unique_ptr<IssuePool> pool;  // single-process, >= 2 GPUs (issue_pool)
  std::vector<hda_msg_t> last_plan;
  long long timeout_ns = 60LL * 1000 * 1000 * 1000;
};

// ====================================================================== helpers

static int fail(hda_ctx_t* c, int code, const std::string& m) {
  if (c) {
    std::lock_guard<std::mutex> lk(c->err_mu);
    c->err = m;
  }
  return code;
}

static int cuda_fail(hda_ctx_t* c, cudaError_t e, const char* what) {
  std::lock_guard<std::mutex> lk(c->err_mu);
  c->sticky = HDA_ECUDA;
  c->err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return HDA_ECUDA;
}

#define CK(x)                                          \
  do {                                                 \
    cudaError_t e_ = (x);                              \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #x); \
  } while (0)

#define GUARD()                                              \
  do {                                                       \
    if (!ctx) return HDA_EINVAL;                             \
    if (ctx->sticky) return fail(ctx, ctx->sticky, ctx->err); \
  } while (0)

struct DevGuard {
  int prev = -1;
  bool on;
  explicit DevGuard(bool enable) : on(enable) {
    if (on) cudaGetDevice(&prev);
  }
  ~DevGuard() {
    if (on && prev >= 0) cudaSetDevice(prev);
  }
};

static void front_shape(int ndim, const int64_t* s, int64_t* out) {
  int off = 3 - ndim;
  for (int k = 0; k < 3; k++) out[k] = k < off ? 1 : s[k - off];
}
static Box front_box(int ndim, const Box& b) {
  Box r = unit_box();
  int off = 3 - ndim;
  for (int k = 0; k < ndim; k++) {
    r.lb[k + off] = b.lb[k];
    r.ub[k + off] = b.ub[k];
  }
  return r;
}

static bool same_stream(const hda_ctx_t* ctx, int p, int q) {
  return ctx->dev[p].local && ctx->dev[q].local && ctx->dev[p].gpu == ctx->dev[q].gpu;
}

static cudaStream_t stream_of(const hda_ctx_t* ctx, int d) { return ctx->gpus[ctx->dev[d].gpu].stream; }
static int ordinal_of(const hda_ctx_t* ctx, int d) { return ctx->gpus[ctx->dev[d].gpu].ordinal; }

// strided descriptor of box `fb` (front-padded) in an array of front-padded shape S
static RunDesc rect_desc(const int64_t* S, const Box& fb, size_t es) {
  RunDesc d;
  std::memset(&d, 0, sizeof d);
  const int64_t e0 = fb.ub[0] - fb.lb[0], e1 = fb.ub[1] - fb.lb[1], e2 = fb.ub[2] - fb.lb[2];
  const int64_t off = ((fb.lb[0] * S[1] + fb.lb[1]) * S[2] + fb.lb[2]) * (int64_t)es;
  d.src_off = d.dst_off = off;
  d.es = (int32_t)es;
  if (e2 == S[2] && e1 == S[1]) {
    d.run_bytes = e0 * e1 * e2 * (int64_t)es;
    d.n0 = 1;
    d.n1 = 1;
  } else if (e2 == S[2]) {
    d.run_bytes = e1 * e2 * (int64_t)es;
    d.n0 = (int32_t)e0;
    d.n1 = 1;
    d.src_p0 = d.dst_p0 = S[1] * S[2] * (int64_t)es;
  } else {
    d.run_bytes = e2 * (int64_t)es;
    d.n0 = (int32_t)e0;
    d.n1 = (int32_t)e1;
    d.src_p0 = d.dst_p0 = S[1] * S[2] * (int64_t)es;
    d.src_p1 = d.dst_p1 = S[2] * (int64_t)es;
  }
  return d;
}

static void batch_descs(std::vector<RunDesc>& descs, std::vector<RunBatch>& out) {
  RunBatch b;
  std::memset(&b, 0, sizeof b);
  int64_t total = 0;
  for (const RunDesc& d : descs) total += d.run_bytes * d.n0 * d.n1;
  const int64_t chunk = pick_chunk_bytes(total);
  for (RunDesc d : descs) {
    if (b.n == kMaxRunDescs) {
      out.push_back(b);
      std::memset(&b, 0, sizeof b);
    }
    int64_t u = run_desc_units(d, chunk);
    if (u == 0) continue;
    d.unit_begin = b.total_units;
    b.total_units += u;
    b.d[b.n++] = d;
  }
  if (b.n) out.push_back(b);
}

// devices' launches may be issued from several host threads (IssuePool)
static void count_launch(hda_ctx_t* ctx, int n = 1) {
  __atomic_fetch_add(&ctx->stats.kernel_launches, (int64_t)n, __ATOMIC_RELAXED);
}
// trace/timing attribution of the next timed_end (serial issue only: timing and tracing
// turn the issue threads off)
static void mark(hda_ctx_t* ctx, int q, int phase) {
  if (ctx->ktiming || ctx->tracing) {
    ctx->cur_dev = q;
    ctx->cur_phase = phase;
  }
}

static cudaEvent_t get_event(hda_ctx_t* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

static int launch_waits(hda_ctx_t* ctx, int d, const WaitList& w) {
  if (w.n == 0) return HDA_OK;
  CK(launch_wait(w, ctx->err_host, ctx->timeout_ns, stream_of(ctx, d)));
  count_launch(ctx);
  return HDA_OK;
}
static int launch_signals(hda_ctx_t* ctx, int d, const SignalList& s) {
  if (s.n == 0) return HDA_OK;
  CK(launch_signal(s, stream_of(ctx, d)));
  count_launch(ctx);
  return HDA_OK;
}
static void wl_add(WaitList& w, unsigned long long* p, unsigned long long v) {
  if (v == 0) return;
  for (int i = 0; i < w.n; i++)
    if (w.ptr[i] == p) {
      if (w.val[i] < v) w.val[i] = v;
      return;
    }
  w.ptr[w.n] = p;
  w.val[w.n] = v;
  w.n++;
}

static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

static KSync ks_empty(hda_ctx_t* ctx) {
  // signals: one system-scope fence, then relaxed system-scope stores — a release at
  // system scope (sync.cuh); HDA_SIG_RELEASE=1 uses st.release.sys for every flag
  static const int relaxed = env_int("HDA_SIG_RELEASE", 0) ? 0 : 1;
  KSync k;
  k.relaxed = relaxed;
  k.nwait = 0;
  k.nsig = 0;
  k.sig_val = 0;
  k.ctr = nullptr;
  k.err = ctx->err_host;
  k.timeout_ns = ctx->timeout_ns;
  k.delay_ns = 0;
  return k;
}
// test hook: every pull (the reader side of an exchange) sleeps this long after its
// RAW waits, so a missing WAR wait on the writer shows up as a parity failure;
// HDA_DEBUG_PULL_DELAY_DEV=r delays only reader device r's pulls (an asymmetric slow
// reader: the WAR windows that only open while OTHER devices run ahead)
static long long pull_delay_ns(int q) {
  static const long long v = 1000LL * env_int("HDA_DEBUG_PULL_DELAY_US", 0);
  static const int only = env_int("HDA_DEBUG_PULL_DELAY_DEV", -1);
  return only < 0 || only == q ? v : 0;
}
static void ks_wait(KSync& k, unsigned long long* p, unsigned long long v) {
  if (v == 0) return;
  for (int i = 0; i < k.nwait; i++)
    if (k.wait_ptr[i] == p) {
      if (k.wait_val[i] < v) k.wait_val[i] = v;
      return;
    }
  k.wait_ptr[k.nwait] = p;
  k.wait_val[k.nwait] = v;
  k.nwait++;
}
static void ks_sig(KSync& k, unsigned long long* p) {
  if (k.nsig < kKSync) k.sig_ptr[k.nsig++] = p;
}

static int check_err_flag(hda_ctx_t* ctx) {
  if (ctx->err_host && *(volatile int*)ctx->err_host) {
    ctx->sticky = HDA_ETIMEOUT;
    ctx->err = "a cross-device wait timed out (a peer did not signal)";
    return HDA_ETIMEOUT;
  }
  return HDA_OK;
}

static int sync_all(hda_ctx_t* ctx) {
  for (auto& g : ctx->gpus) {
    CK(cudaSetDevice(g.ordinal));
    CK(cudaStreamSynchronize(g.comm));
    CK(cudaStreamSynchronize(g.stream));
  }
  return check_err_flag(ctx);
}

// ====================================================================== exec plans

// grows device d's staging buffer; the caller has synchronised EVERY GPU first (a
// peer's in-flight copy may still read the old send buffer)
static int ensure_stage(hda_ctx_t* ctx, std::vector<char*>& v, std::vector<size_t>& cap, int d, size_t need) {
  if (cap[d] >= need) return HDA_OK;
  CK(cudaSetDevice(ordinal_of(ctx, d)));
  if (v[d]) CK(cudaFree(v[d]));
  size_t n = std::max(need, (size_t)1 << 20);
  CK(cudaMalloc((void**)&v[d], n));
  cap[d] = n;
  return HDA_OK;
}

// AUTO transport threshold (HDA_CE_BYTES, default kCeBytes): tests lower it to put
// small bulk messages on the copy-engine (and gated-product) path
static int64_t ce_bytes() {
  static const int64_t v = [] {
    const char* e = std::getenv("HDA_CE_BYTES");
    return e ? std::atoll(e) : kCeBytes;
  }();
  return v;
}

static int build_exec(hda_ctx_t* ctx, const Transition* t, ExecPlan& ep) {
  const int P = ctx->P;
  ep.staged = ctx->transport == HDA_XPORT_STAGED;
  ep.transport = ctx->transport;
  if (t->msgs.empty()) return HDA_OK;
  for (const Msg& m : t->msgs) {
    bool seen = false;
    for (const PendEntry& e : ep.reads)
      if (e.array == m.array && e.src == m.src && e.dst == m.dst) seen = true;
    if (!seen) ep.reads.push_back({m.array, m.src, m.dst});
  }
  if (!ep.staged) {
    for (int q = 0; q < P; q++) {
      if (!ctx->dev[q].local) continue;
      PullJob job;
      job.dst = q;
      std::vector<RunDesc> descs;
      // permutation schedule: device q pulls from q+1, q+2, ... (mod P) so that at any
      // moment every source serves one reader instead of all readers hitting src 0
      std::vector<const Msg*> mine;
      for (const Msg& m : t->msgs)
        if (m.dst == q) mine.push_back(&m);
      std::stable_sort(mine.begin(), mine.end(), [&](const Msg* a, const Msg* b) {
        return (a->src - q + P) % P < (b->src - q + P) % P;
      });
      for (const Msg* mp : mine) {
        const Msg& m = *mp;
        const TArray& a = ctx->tr->array(m.array);
        int64_t S[3];
        front_shape(a.ndim, a.shape, S);
        const Box fb = front_box(a.ndim, m.box);
        RunDesc d = rect_desc(S, fb, a.es);
        d.src = ctx->arr[m.array].ptr[m.src];
        d.dst = ctx->arr[m.array].ptr[q];
        if (!d.src || !d.dst) return fail(ctx, HDA_ESTATE, "replica not mapped (SPMD handles missing?)");
        const int64_t bytes = box_volume(m.box) * (int64_t)a.es;
        if (ctx->transport == HDA_XPORT_AUTO && bytes >= ce_bytes() && !same_stream(ctx, m.src, q)) {
          // bulk: copy-engine peer copy of the strided box (no SM time, no staging)
          cudaMemcpy3DParms p;
          std::memset(&p, 0, sizeof p);
          p.srcPtr = make_cudaPitchedPtr(const_cast<char*>(d.src), (size_t)S[2] * a.es, (size_t)S[2], (size_t)S[1]);
          p.dstPtr = make_cudaPitchedPtr(d.dst, (size_t)S[2] * a.es, (size_t)S[2], (size_t)S[1]);
          p.srcPos = p.dstPos = make_cudaPos((size_t)fb.lb[2] * a.es, (size_t)fb.lb[1], (size_t)fb.lb[0]);
          p.extent = make_cudaExtent((size_t)(fb.ub[2] - fb.lb[2]) * a.es, (size_t)(fb.ub[1] - fb.lb[1]),
                                     (size_t)(fb.ub[0] - fb.lb[0]));
          p.kind = cudaMemcpyDefault;
          job.ce.push_back(p);
          job.ce_src.push_back(m.src);
        } else {
          descs.push_back(d);
        }
        if (std::find(job.srcs.begin(), job.srcs.end(), m.src) == job.srcs.end()) job.srcs.push_back(m.src);
        std::pair<int, int> pr(m.array, m.src);
        if (std::find(job.pend.begin(), job.pend.end(), pr) == job.pend.end()) job.pend.push_back(pr);
      }
      if (descs.empty() && job.ce.empty()) continue;
      batch_descs(descs, job.batches);
      for (int p : job.srcs)
        if (!same_stream(ctx, p, q)) job.cross = true;
      // overlap split (footprint radius r of the built-in kernel)
      const CallInfo& ci = *t->info;
      if (ci.kernel == KN_GEMM && descs.empty() && job.cross && job.srcs.size() <= (size_t)kMaxGate) {
        // gated product: every message is one full-width row block of B from another GPU
        const int Barr = ci.param_array[2];
        const TArray& B = ctx->tr->array(Barr);
        bool ok = B.ndim == 2;
        std::vector<std::pair<int64_t, int64_t>> rows(job.srcs.size(), {-1, -1});
        for (const Msg* mp : mine) {
          const size_t i = std::find(job.srcs.begin(), job.srcs.end(), mp->src) - job.srcs.begin();
          if (mp->array != Barr || same_stream(ctx, mp->src, q) || rows[i].first >= 0 || mp->box.lb[1] != 0 ||
              mp->box.ub[1] != B.shape[1])
            ok = false;
          else
            rows[i] = {mp->box.lb[0], mp->box.ub[0]};
        }
        if (ok) {
          job.gate = true;
          job.gate_rows = rows;
          job.gate_k = B.shape[0];
        }
      }
      int r = -1;
      if (ci.kernel == KN_JACOBI5 || ci.kernel == KN_STENCIL9 || ci.kernel == KN_STENCIL7_3D) r = 1;
      if (ci.kernel == KN_SCALE || ci.kernel == KN_COPY) r = 0;
      const Box& w = ctx->tr->part(ci.part).box[q];
      if (r >= 0 && !box_empty(w)) {
        const int nd = ctx->tr->part(ci.part).ndim;
        std::vector<Box> dil;
        for (const Msg& m : t->msgs) {
          if (m.dst != q) continue;
          Box b = m.box;
          for (int kk = 0; kk < nd; kk++) {
            b.lb[kk] -= r;
            b.ub[kk] += r;
          }
          dil.push_back(b);
        }
        Rects W{w};
        Rects D = intersect(W, canonicalize(dil));
        job.dependent = D;
        job.interior = subtract(W, D);
        job.split = true;
      }
      ep.pulls.push_back(std::move(job));
    }
    return HDA_OK;
  }
  // STAGED: p's send staging holds its outgoing messages ordered by (dst, array, lb),
  // 256-byte aligned per message, so each (p, q) pair is one contiguous segment.
  std::vector<const Msg*> order;
  for (const Msg& m : t->msgs) order.push_back(&m);
  std::stable_sort(order.begin(), order.end(), [](const Msg* a, const Msg* b) {
    if (a->src != b->src) return a->src < b->src;
    return a->dst < b->dst;
  });
  std::vector<size_t> src_off(order.size());
  std::vector<size_t> used(P, 0);
  for (size_t i = 0; i < order.size(); i++) {
    const Msg& m = *order[i];
    const TArray& a = ctx->tr->array(m.array);
    src_off[i] = used[m.src];
    used[m.src] += ((size_t)box_volume(m.box) * a.es + 255) & ~(size_t)255;
  }
  // packs (staging pointers are bound at issue, issue_staged: a cached plan must not
  // hold a buffer that a later, larger plan reallocates)
  for (int p = 0; p < P; p++) {
    if (!ctx->dev[p].local || used[p] == 0) continue;
    PackJob job;
    job.src = p;
    job.bytes = used[p];
    std::vector<RunDesc> descs;
    for (size_t i = 0; i < order.size(); i++) {
      const Msg& m = *order[i];
      if (m.src != p) continue;
      const TArray& a = ctx->tr->array(m.array);
      int64_t S[3];
      front_shape(a.ndim, a.shape, S);
      RunDesc d = rect_desc(S, front_box(a.ndim, m.box), a.es);
      d.src = ctx->arr[m.array].ptr[p];
      d.dst = nullptr;  // send_stage[p], bound at issue
      d.dst_off = (int64_t)src_off[i];
      d.dst_p1 = d.run_bytes;
      d.dst_p0 = d.run_bytes * d.n1;
      descs.push_back(d);
      if (std::find(job.dsts.begin(), job.dsts.end(), m.dst) == job.dsts.end()) job.dsts.push_back(m.dst);
    }
    batch_descs(descs, job.batches);
    ep.packs.push_back(std::move(job));
  }
  // receives
  for (int q = 0; q < P; q++) {
    if (!ctx->dev[q].local) continue;
    RecvJob job;
    job.dst = q;
    size_t off = 0;
    std::vector<RunDesc> descs;
    for (size_t i = 0; i < order.size(); i++) {
      const Msg& m = *order[i];
      if (m.dst != q) continue;
      const TArray& a = ctx->tr->array(m.array);
      size_t bytes = (size_t)box_volume(m.box) * a.es;
      size_t padded = (bytes + 255) & ~(size_t)255;
      if (!job.segs.empty() && job.segs.back().src == m.src &&
          job.segs.back().src_off + job.segs.back().bytes == src_off[i]) {
        job.segs.back().bytes += padded;
      } else {
        job.segs.push_back(Seg{m.src, src_off[i], off, padded});
      }
      int64_t S[3];
      front_shape(a.ndim, a.shape, S);
      RunDesc d = rect_desc(S, front_box(a.ndim, m.box), a.es);
      d.dst = ctx->arr[m.array].ptr[q];
      d.src_off = (int64_t)off;
      d.src_p1 = d.run_bytes;
      d.src_p0 = d.run_bytes * d.n1;
      descs.push_back(d);
      off += padded;
      if (std::find(job.srcs.begin(), job.srcs.end(), m.src) == job.srcs.end()) job.srcs.push_back(m.src);
    }
    if (descs.empty()) continue;
    job.bytes = off;
    for (RunDesc& d : descs) d.src = nullptr;  // recv_stage[q], bound at issue
    batch_descs(descs, job.unpack);
    ep.recvs.push_back(std::move(job));
  }
  return HDA_OK;
}

// ====================================================================== phases

static int timed_begin(hda_ctx_t* ctx, cudaStream_t st, cudaEvent_t* a) {
  *a = nullptr;
  if (!ctx->ktiming && !ctx->tracing) return HDA_OK;
  *a = get_event(ctx);
  CK(cudaEventRecord(*a, st));
  return HDA_OK;
}
static int timed_end(hda_ctx_t* ctx, cudaStream_t st, int kind, cudaEvent_t a, int count = 1) {
  if (!a) return HDA_OK;
  cudaEvent_t b = get_event(ctx);
  CK(cudaEventRecord(b, st));
  TimedEv e{kind, a, b, count, ctx->epoch, ctx->cur_dev, kind == -100 ? 0 : ctx->cur_phase};
  if (ctx->tracing) {
    ctx->trace.push_back(e);
  } else {
    ctx->tev.push_back(e);
  }
  return HDA_OK;
}

// WAR on the READER side: a pull overwrites cells of its reader q's own replica, so
// every peer r that pulled cells of that array from q since q last wrote it (pend,
// rread) and may still be reading them — r's stream can run far behind q's — must have
// acknowledged before the pull writes.  Three devices are enough: q writes c, r pulls
// c from q, p redefines c (waiting on no one: r read q's replica, not p's), then q
// pulls c back from p.  Filtered per box: a pull whose boxes miss every box peers read
// from q's replica waits on nothing (the steady state of every halo loop, where q's
// own definition of the array cleared both records first).  Computed from the records
// BEFORE this call's reads are added: within one call q pulls only cells it does not
// own and peers pull only cells it owns, and waiting on this call's own ACKs would
// deadlock a symmetric halo exchange.
static void pull_war_waits(hda_ctx_t* ctx, const Transition* t) {
  static const int no_war = env_int("HDA_DEBUG_NO_WAR", 0);
  for (auto& v : ctx->pull_war) v.clear();
  if (no_war) return;
  for (const Msg& m : t->msgs) {
    const int q = m.dst;
    if (!ctx->dev[q].local) continue;
    const auto& row = ctx->pend[m.array][q];
    bool any = false;
    for (int r = 0; r < ctx->P; r++) any |= row[r] && !same_stream(ctx, q, r);
    if (!any) continue;
    bool hit = ctx->rread_over[m.array][q] != 0;
    for (const Box& b : ctx->rread[m.array][q]) hit = hit || !box_empty(box_and(b, m.box));
    if (!hit) continue;
    auto& w = ctx->pull_war[q];
    for (int r = 0; r < ctx->P; r++) {
      if (!row[r] || same_stream(ctx, q, r)) continue;
      unsigned long long* p = ctx->dev[q].sync + SW_ACK + r;
      bool merged = false;
      for (auto& e : w)
        if (e.first == p) {
          e.second = std::max(e.second, row[r]);
          merged = true;
        }
      if (!merged) w.emplace_back(p, row[r]);
    }
  }
}

// exec plan of call t (cached per transition) and the WAR bookkeeping of its reads
// (`scratch` holds the plan when the cache is off; it must outlive the issue)
static int exchange_plan(hda_ctx_t* ctx, const Transition* t, unsigned long long k, ExecPlan& scratch,
                         ExecPlan** out) {
  *out = nullptr;
  pull_war_waits(ctx, t);
  if (t->msgs.empty()) return HDA_OK;
  ExecPlan* ep;
  if (ctx->cache_on) {
    auto it = ctx->exec.find(t->serial);
    if (it == ctx->exec.end() || it->second.transport != ctx->transport) {
      ExecPlan np;
      int rc = build_exec(ctx, t, np);
      if (rc) return rc;
      ctx->exec[t->serial] = std::move(np);
      it = ctx->exec.find(t->serial);
    }
    ep = &it->second;
  } else {
    int rc = build_exec(ctx, t, scratch);
    if (rc) return rc;
    ep = &scratch;
  }
  if (!ep->staged)
    for (const PendEntry& e : ep->reads) ctx->pend[e.array][e.src][e.dst] = k;
  for (const Msg& m : t->msgs) {
    if (same_stream(ctx, m.src, m.dst)) continue;
    auto& v = ctx->rread[m.array][m.src];
    if (v.size() >= 32) {
      ctx->rread_over[m.array][m.src] = 1;
    } else {
      bool dup = false;
      for (const Box& b : v) dup = dup || box_eq(b, m.box);
      if (!dup) v.push_back(m.box);
    }
  }
  *out = ep;
  return HDA_OK;
}

static void war_waits(hda_ctx_t* ctx, const CallInfo& ci, int q, KSync& ks);
static bool war_disjoint(hda_ctx_t* ctx, const CallInfo& ci, int q, const std::vector<Box>& boxes);
static int run_kernel(hda_ctx_t* ctx, const Transition* t, int q, const double* scalars, const KSync& ks,
                      const std::vector<Box>* boxes = nullptr, cudaStream_t stream = nullptr,
                      const KGate* gate = nullptr);

// Stream memory operations (driver API, no SM time): the gated product's comm stream
// waits for the sources' PROD words and publishes arrivals and ACKs without a kernel, so
// it makes progress while the GPU-filling GEMM spins on the arrival flags.
typedef CUresult (*StreamValue64Fn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*DeviceAttrFn)(int*, CUdevice_attribute, CUdevice);
struct MemOps {
  StreamValue64Fn wait = nullptr, write = nullptr;
  bool ok = false;
};
static const MemOps& memops() {
  static const MemOps m = [] {
    MemOps r;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      r.wait = (StreamValue64Fn)p;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      r.write = (StreamValue64Fn)p;
    int attr = 0, dev = 0;
    if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess && cudaGetDevice(&dev) == cudaSuccess)
      ((DeviceAttrFn)p)(&attr, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, (CUdevice)dev);
    r.ok = r.wait && r.write && attr;
    return r;
  }();
  return m;
}
#define CU(call)                                                              \
  do {                                                                        \
    const CUresult cr_ = (call);                                              \
    if (cr_ != CUDA_SUCCESS) return fail(ctx, HDA_ECUDA, "stream memory op failed: " #call); \
  } while (0)

// HDA_GEMM_GATE: how a GEMM whose B rows arrive from other GPUs (copy-engine blocks,
// arrival flags written by the comm stream) overlaps that all-gather.
//   2 (default) split: with an fp32 C and whole k-blocks per source, one launch over the
//     resident rows beside the copies, then one (C += ...) per source as its rows land;
//     otherwise joined.  2MM ROW 16384^2: N=2 5.09-5.12 vs 5.51 ms per step joined, N=4
//     2.67 (2.80 with one launch for all arrived rows) vs 3.09.
//   1 gated inside the kernel: producers wait per k-block for the sources' flags (with
//     fp32 C, K in per-segment passes).  Slower than joining (N=2: 5.62-5.70 vs 5.40):
//     the copies take 0.43 ms either way, the gated product 0.68 ms longer.
//   0 joined: copies, then the product.
static int gate_mode() {
  static const int v = env_int("HDA_GEMM_GATE", 2);
  return v;
}
static bool gate_enabled() { return gate_mode() != 0; }

// The gated product's exchange (reader q): on the comm stream, forked after everything
// issued before this call, per source in the permutation order (q+1, q+2, ...): wait for
// its PROD word, copy its row block of B on the copy engine, then publish the arrival
// flag (local) and the source's ACK.  The GEMM on the main stream starts at once with
// the resident rows and waits per k-block (KGate).
static int issue_gated_pull(hda_ctx_t* ctx, PullJob& job, unsigned long long k) {
  const int q = job.dst;
  const MemOps& mo = memops();
  CK(cudaSetDevice(ordinal_of(ctx, q)));
  Gpu& g = ctx->gpus[ctx->dev[q].gpu];
  CK(cudaEventRecord(g.ev_fork, g.stream));
  CK(cudaStreamWaitEvent(g.comm, g.ev_fork, 0));
  ctx->pulled_on_comm[q] = 1;
  const CUstream cs = (CUstream)g.comm;
  // WAR: peers that pulled these cells of q's replica earlier must be done reading
  for (const auto& e : ctx->pull_war[q]) CU(mo.wait(cs, (CUdeviceptr)e.first, e.second, CU_STREAM_WAIT_VALUE_GEQ));
  cudaEvent_t a = nullptr;
  int rc;
  if ((rc = timed_begin(ctx, g.comm, &a))) return rc;
  KGate& kg = ctx->gate[q];
  std::memset(&kg, 0, sizeof kg);
  for (size_t i = 0; i < job.srcs.size(); i++) {
    const int p = job.srcs[i];
    if (ctx->last_prod[p])
      CU(mo.wait(cs, (CUdeviceptr)(ctx->dev[q].sync + SW_PROD + p), ctx->last_prod[p], CU_STREAM_WAIT_VALUE_GEQ));
    for (size_t c = 0; c < job.ce.size(); c++)
      if (job.ce_src[c] == p) CK(cudaMemcpy3DAsync(&job.ce[c], g.comm));
    // default flags: a system-wide fence precedes each write
    CU(mo.write(cs, (CUdeviceptr)(ctx->dev[q].sync + SW_GATE + p), k, CU_STREAM_WRITE_VALUE_DEFAULT));
    CU(mo.write(cs, (CUdeviceptr)(ctx->dev[p].sync + SW_ACK + q), k, CU_STREAM_WRITE_VALUE_DEFAULT));
    CK(cudaEventRecord(g.ev_src[i], g.comm));  // the split product's launch for these rows waits here
    kg.lo[i] = job.gate_rows[i].first;
    kg.hi[i] = job.gate_rows[i].second;
    kg.flag[i] = ctx->dev[q].sync + SW_GATE + p;
    kg.val[i] = k;
  }
  kg.n = (int32_t)job.srcs.size();  // arrival order = issue order; the launcher derives the K segments
  mark(ctx, q, 0);
  if ((rc = timed_end(ctx, g.comm, -100, a))) return rc;
  CK(cudaEventRecord(g.ev_pull, g.comm));
  ctx->gated[q] = 1;
  return HDA_OK;
}

// HDA_PULL_WAIT_KERNEL (default 1): a comm-stream SM pull waits for its writers in a
// one-CTA launch, then copies with no waits
static bool pull_wait_kernel_on() {
  static const int v = env_int("HDA_PULL_WAIT_KERNEL", 1);
  return v != 0;
}

// one device's pull (reader q = job.dst): thread-safe against the other devices' issue
static int issue_pull(hda_ctx_t* ctx, const Transition* t, PullJob& job, unsigned long long k, bool overlap_kernel,
                      bool halo_kernel, const double* scalars) {
  const int q = job.dst;
  CK(cudaSetDevice(ordinal_of(ctx, q)));
  Gpu& g = ctx->gpus[ctx->dev[q].gpu];
  // 2-D stencil with a cross-GPU halo: the pull runs inside the stencil launch
  if (ctx->overlap && halo_kernel && job.cross && job.split && job.ce.empty() && job.batches.size() == 1 &&
      job.srcs.size() <= 8 && job.srcs.size() + ctx->pull_war[q].size() <= 16 &&
      job.interior.size() + job.dependent.size() <= 8) {
    ctx->halo_job[q] = &job;
    return HDA_OK;
  }
  if (ctx->overlap && job.gate && gate_enabled() && memops().ok) return issue_gated_pull(ctx, job, k);
  const bool comm = ctx->overlap && job.cross && job.split && overlap_kernel;
  cudaStream_t st = comm ? g.comm : g.stream;
  // Stencils on the comm path: when the interior part touches no cell a peer pulled
  // from this replica (per-box WAR), the pull carries the WAR waits and the boundary
  // part runs on the comm stream right after it; the main stream runs the interior with
  // no waits and only joins before the PROD signal (HDA_COMM_BOUNDARY=0: boundary after
  // the interior on the main stream)
  static const int comm_boundary = env_int("HDA_COMM_BOUNDARY", 1);
  static const int sig_kernel_on = env_int("HDA_SIG_KERNEL", 1);
  const CallInfo& ci = *t->info;
  const bool stencil = ci.kernel == KN_JACOBI5 || ci.kernel == KN_STENCIL9 || ci.kernel == KN_STENCIL7_3D;
  const bool boundary_on_comm = comm && comm_boundary && sig_kernel_on && stencil && !job.interior.empty() &&
                                !job.dependent.empty() && war_disjoint(ctx, ci, q, job.interior);
  KSync war = ks_empty(ctx);
  if (boundary_on_comm) {
    war_waits(ctx, ci, q, war);
    ctx->war_done[q] = 1;
  }
  if (comm) {  // the pull may start as soon as everything issued before this call is done
    CK(cudaEventRecord(g.ev_fork, g.stream));
    CK(cudaStreamWaitEvent(g.comm, g.ev_fork, 0));
    ctx->pulled_on_comm[q] = 1;
    ctx->cur_pull[q] = &job;
  }
  // RAW waits and ACK signals ride in the pull kernel itself (sync.cuh)
  KSync pre = ks_empty(ctx), post = ks_empty(ctx);
  post.sig_val = k;
  post.ctr = (unsigned int*)(ctx->dev[q].sync + SW_CTR_PULL);
  for (int p : job.srcs)
    if (!same_stream(ctx, p, q)) {
      ks_wait(pre, ctx->dev[q].sync + SW_PROD + p, ctx->last_prod[p]);
      ks_sig(post, ctx->dev[p].sync + SW_ACK + q);
    }
  for (int i = 0; i < war.nwait; i++) ks_wait(pre, war.wait_ptr[i], war.wait_val[i]);
  for (const auto& e : ctx->pull_war[q]) ks_wait(pre, e.first, e.second);
  int rc;
  cudaEvent_t a = nullptr;
  const size_t nb = job.batches.size();
  // the exchange timer brackets the transfer, not the wait for the writers (below: the
  // copy-engine path and the comm-stream wait launch start it after their waits)
  const bool wait_first = nb > 0 && comm && pull_wait_kernel_on() && pre.nwait > 0;
  if (job.ce.empty() && !wait_first && (rc = timed_begin(ctx, st, &a))) return rc;
  if (!job.ce.empty()) {  // copy-engine part: RAW wait kernel, then the copies
    KSync w = ks_empty(ctx);
    std::memcpy(w.wait_ptr, pre.wait_ptr, sizeof w.wait_ptr);
    std::memcpy(w.wait_val, pre.wait_val, sizeof w.wait_val);
    w.nwait = pre.nwait;
    w.delay_ns = pull_delay_ns(q);
    RunBatch empty;
    std::memset(&empty, 0, sizeof empty);
    if (w.nwait || w.delay_ns) {
      CK(launch_copy_runs(empty, w, st));
      count_launch(ctx);
    }
    pre.nwait = 0;
    if ((rc = timed_begin(ctx, st, &a))) return rc;  // transfer time, not the wait
    for (const cudaMemcpy3DParms& p : job.ce) CK(cudaMemcpy3DAsync(&p, st));
    if (nb == 0) {
      CK(launch_copy_runs(empty, post, st));  // ACK signals after the copies
      count_launch(ctx);
    }
  }
  // Comm-stream SM pull: wait in one CTA, then launch the copy with no waits.  Folded
  // into the pull kernel, every one of its CTAs would spin on the writers' PROD words for
  // as long as the neighbours take to finish their previous step (~30 us at N=4), holding
  // SM slots the interior launch running beside it needs (HDA_PULL_WAIT_KERNEL=0: fold)
  bool waited_outside = false;
  if (wait_first && pre.nwait > 0) {
    KSync w = ks_empty(ctx);
    std::memcpy(w.wait_ptr, pre.wait_ptr, sizeof w.wait_ptr);
    std::memcpy(w.wait_val, pre.wait_val, sizeof w.wait_val);
    w.nwait = pre.nwait;
    w.delay_ns = pull_delay_ns(q);
    RunBatch empty;
    std::memset(&empty, 0, sizeof empty);
    CK(launch_copy_runs(empty, w, st));
    count_launch(ctx);
    pre.nwait = 0;
    waited_outside = true;
    if ((rc = timed_begin(ctx, st, &a))) return rc;
  }
  for (size_t i = 0; i < nb; i++) {
    KSync ks = ks_empty(ctx);
    if (i == 0) {
      std::memcpy(ks.wait_ptr, pre.wait_ptr, sizeof ks.wait_ptr);
      std::memcpy(ks.wait_val, pre.wait_val, sizeof ks.wait_val);
      ks.nwait = pre.nwait;
      ks.delay_ns = waited_outside ? 0 : pull_delay_ns(q);
    }
    if (i + 1 == nb) {
      std::memcpy(ks.sig_ptr, post.sig_ptr, sizeof ks.sig_ptr);
      ks.nsig = post.nsig;
      ks.sig_val = post.sig_val;
      ks.ctr = post.ctr;
    }
    CK(launch_copy_runs(job.batches[i], ks, st));
    count_launch(ctx);
  }
  mark(ctx, q, 0);
  if ((rc = timed_end(ctx, st, -100, a))) return rc;
  if (boundary_on_comm) {
    cudaEvent_t b;
    if ((rc = timed_begin(ctx, g.comm, &b))) return rc;
    if ((rc = run_kernel(ctx, t, q, scalars, ks_empty(ctx), &job.dependent, g.comm))) return rc;
    mark(ctx, q, 3);
    if ((rc = timed_end(ctx, g.comm, ci.kernel, b, 0))) return rc;
    ctx->split_mode[q] = 2;
  }
  if (comm) CK(cudaEventRecord(g.ev_pull, g.comm));
  return HDA_OK;
}

static RunBatch bind_stage(const RunBatch& b, char* dst, const char* src) {
  RunBatch o = b;
  for (int i = 0; i < o.n; i++) {
    if (dst) o.d[i].dst = dst;
    if (src) o.d[i].src = src;
  }
  return o;
}

// STAGED transport (single process, serial issue)
static int issue_staged(hda_ctx_t* ctx, ExecPlan* ep, unsigned long long k) {
  // size the staging buffers for this plan; growing one first drains every GPU, so no
  // pack, peer copy or unpack of an earlier call still uses the buffer being freed
  bool grow = false;
  for (const PackJob& job : ep->packs) grow |= ctx->send_cap[job.src] < job.bytes;
  for (const RecvJob& job : ep->recvs) grow |= ctx->recv_cap[job.dst] < job.bytes;
  if (grow) {
    int rc = sync_all(ctx);
    if (rc) return rc;
    for (const PackJob& job : ep->packs)
      if ((rc = ensure_stage(ctx, ctx->send_stage, ctx->send_cap, job.src, job.bytes))) return rc;
    for (const RecvJob& job : ep->recvs)
      if ((rc = ensure_stage(ctx, ctx->recv_stage, ctx->recv_cap, job.dst, job.bytes))) return rc;
  }
  for (PackJob& job : ep->packs) {
    const int p = job.src;
    CK(cudaSetDevice(ordinal_of(ctx, p)));
    WaitList wl;
    wl.n = 0;
    for (auto& e : ctx->stage_pend[p])
      if (!same_stream(ctx, p, e.first)) wl_add(wl, ctx->dev[p].sync + SW_ACK + e.first, e.second);
    ctx->stage_pend[p].clear();
    int rc = launch_waits(ctx, p, wl);
    if (rc) return rc;
    cudaEvent_t a;
    if ((rc = timed_begin(ctx, stream_of(ctx, p), &a))) return rc;
    for (const RunBatch& b : job.batches) {
      CK(launch_copy_runs(bind_stage(b, ctx->send_stage[p], nullptr), ks_empty(ctx), stream_of(ctx, p)));
      count_launch(ctx);
    }
    if ((rc = timed_end(ctx, stream_of(ctx, p), -100, a))) return rc;
    SignalList sl;
    sl.n = 0;
    sl.val = k;
    for (int q : job.dsts)
      if (!same_stream(ctx, p, q)) sl.ptr[sl.n++] = ctx->dev[q].sync + SW_PACK + p;
    if ((rc = launch_signals(ctx, p, sl))) return rc;
  }
  for (RecvJob& job : ep->recvs) {
    const int q = job.dst;
    CK(cudaSetDevice(ordinal_of(ctx, q)));
    WaitList wl;
    wl.n = 0;
    SignalList sl;
    sl.n = 0;
    sl.val = k;
    for (int p : job.srcs)
      if (!same_stream(ctx, p, q)) {
        wl_add(wl, ctx->dev[q].sync + SW_PACK + p, k);
        sl.ptr[sl.n++] = ctx->dev[p].sync + SW_ACK + q;
      }
    for (const auto& e : ctx->pull_war[q]) wl_add(wl, e.first, e.second);
    int rc = launch_waits(ctx, q, wl);
    if (rc) return rc;
    cudaEvent_t a;
    if ((rc = timed_begin(ctx, stream_of(ctx, q), &a))) return rc;
    for (const Seg& s : job.segs)
      CK(cudaMemcpyAsync(ctx->recv_stage[q] + s.dst_off, ctx->send_stage[s.src] + s.src_off, s.bytes,
                         cudaMemcpyDeviceToDevice, stream_of(ctx, q)));
    for (const RunBatch& b : job.unpack) {
      CK(launch_copy_runs(bind_stage(b, nullptr, ctx->recv_stage[q]), ks_empty(ctx), stream_of(ctx, q)));
      count_launch(ctx);
    }
    if ((rc = timed_end(ctx, stream_of(ctx, q), -100, a))) return rc;
    if ((rc = launch_signals(ctx, q, sl))) return rc;
    for (int p : job.srcs) ctx->stage_pend[p].push_back({q, k});
  }
  return HDA_OK;
}

// WAR before device q overwrites cells of the arrays it defines: every peer that
// pulled those arrays from q must have acknowledged the pull
static void war_waits(hda_ctx_t* ctx, const CallInfo& ci, int q, KSync& ks) {
  // HDA_DEBUG_NO_WAR=1 drops the WAR waits: UNSAFE, measurement of their cost only
  static const int no_war = env_int("HDA_DEBUG_NO_WAR", 0);
  if (no_war) return;
  for (size_t i = 0; i < ci.arrays.size(); i++) {
    if (ci.ldef[i][q].empty()) continue;
    auto& row = ctx->pend[ci.arrays[i]][q];
    for (int r = 0; r < ctx->P; r++) {
      if (row[r] && !same_stream(ctx, q, r)) ks_wait(ks, ctx->dev[q].sync + SW_ACK + r, row[r]);
      row[r] = 0;
    }
    ctx->rread[ci.arrays[i]][q].clear();
    ctx->rread_over[ci.arrays[i]][q] = 0;
  }
}

// true if no box in `boxes` touches a cell peers pulled from q's copy of an array q
// defines in this call (since q last wrote it): writing them needs no WAR wait
static bool war_disjoint(hda_ctx_t* ctx, const CallInfo& ci, int q, const std::vector<Box>& boxes) {
  for (size_t i = 0; i < ci.arrays.size(); i++) {
    if (ci.ldef[i][q].empty()) continue;
    const int a = ci.arrays[i];
    if (ctx->rread_over[a][q]) return false;
    for (const Box& r : ctx->rread[a][q])
      for (const Box& b : boxes)
        if (!box_empty(box_and(r, b))) return false;
  }
  return true;
}

// RAW: publish "device q completed call k" to every peer
static void signal_prod(hda_ctx_t* ctx, int q, unsigned long long k, KSync& ks) {
  ks.sig_val = k;
  ks.ctr = (unsigned int*)(ctx->dev[q].sync + SW_CTR_KERN);
  for (int r = 0; r < ctx->P; r++)
    if (r != q && !same_stream(ctx, q, r)) ks_sig(ks, ctx->dev[r].sync + SW_PROD + q);
}

// separate wait/signal kernels, for phases that launch no kernel of their own
static int sync_only(hda_ctx_t* ctx, int q, const KSync& ks) {
  if (ks.nwait == 0 && ks.nsig == 0) return HDA_OK;
  RunBatch empty;
  std::memset(&empty, 0, sizeof empty);
  CK(launch_copy_runs(empty, ks, stream_of(ctx, q)));
  count_launch(ctx);
  return HDA_OK;
}

// launch the built-in kernel of call t on device q over `boxes` (default: q's work box)
// in as few launches as possible; waits ride with the first launch, signals with the last
static KSync ks_part(hda_ctx_t* ctx, const KSync& ks, bool first, bool last) {
  KSync k2 = ks_empty(ctx);
  if (first) {
    std::memcpy(k2.wait_ptr, ks.wait_ptr, sizeof k2.wait_ptr);
    std::memcpy(k2.wait_val, ks.wait_val, sizeof k2.wait_val);
    k2.nwait = ks.nwait;
  }
  if (last) {
    std::memcpy(k2.sig_ptr, ks.sig_ptr, sizeof k2.sig_ptr);
    k2.nsig = ks.nsig;
    k2.sig_val = ks.sig_val;
    k2.ctr = ks.ctr;
  }
  return k2;
}

// HDA_GEMM_GATE=2, the split product (all-gather of B overlapped with the GEMM): with an
// fp32 C and whole k-blocks per source, the resident rows' product runs as one launch
// beside the copy-engine blocks, then one launch (C += alpha * A_i B_i) per source, in
// arrival order, each after the comm-stream event behind that source's block.  No
// in-kernel gating.  *done = false (nothing launched) when the resident rows are not one
// contiguous run of whole k-blocks or the CTA-pair kernel does not apply; the caller
// then joins the copies.
static int split_product(hda_ctx_t* ctx, int q, const void* A, const void* B, void* C, int64_t M, int64_t N,
                         int64_t K, const Box& fb, float alpha, float beta, const KSync& ks, cudaStream_t s,
                         const KGate& gate, bool* done) {
  constexpr int64_t BK = 64;  // the CTA-pair GEMM's k-block
  *done = false;
  const int64_t kb = (K + BK - 1) / BK;
  std::vector<char> remote(kb, 0);
  bool aligned = true;
  for (int i = 0; i < gate.n; i++) {
    if (gate.lo[i] % BK || (gate.hi[i] % BK && gate.hi[i] != K)) aligned = false;
    for (int64_t b = gate.lo[i] / BK; b * BK < gate.hi[i] && b < kb; b++) remote[b] = 1;
  }
  int64_t a = 0;  // resident k-blocks [a, b)
  while (a < kb && remote[a]) a++;
  int64_t b = a;
  while (b < kb && !remote[b]) b++;
  bool contiguous = a < b;
  for (int64_t x = b; x < kb; x++) contiguous &= remote[x] != 0;
  if (!aligned || !contiguous || b - a >= kb) return HDA_OK;
  KGate g1;
  std::memset(&g1, 0, sizeof g1);
  g1.nseg = 1, g1.skb0[0] = (int32_t)a, g1.skb1[0] = (int32_t)b;
  const cudaError_t e = launch_gemm(HDA_F32, A, B, C, M, N, K, fb.lb, fb.ub, alpha, beta,
                                    ks_part(ctx, ks, true, false), s, &g1);
  if (e == cudaErrorNotSupported) return HDA_OK;
  CK(e);
  const Gpu& gg = ctx->gpus[ctx->dev[q].gpu];
  for (int i = 0; i < gate.n; i++) {
    count_launch(ctx);  // the previous launch (the caller counts the last one)
    KGate gi;
    std::memset(&gi, 0, sizeof gi);
    gi.nseg = 1;
    gi.skb0[0] = (int32_t)(gate.lo[i] / BK);
    gi.skb1[0] = (int32_t)std::min<int64_t>(kb, (gate.hi[i] + BK - 1) / BK);
    CK(cudaStreamWaitEvent(s, gg.ev_src[i], 0));
    CK(launch_gemm(HDA_F32, A, B, C, M, N, K, fb.lb, fb.ub, alpha, 1.0f, ks_part(ctx, ks, false, i + 1 == gate.n),
                   s, &gi));
  }
  __atomic_fetch_add(&ctx->stats.gated_products, (int64_t)1, __ATOMIC_RELAXED);
  *done = true;
  return HDA_OK;
}

static int run_kernel(hda_ctx_t* ctx, const Transition* t, int q, const double* scalars, const KSync& ks,
                      const std::vector<Box>* boxes, cudaStream_t stream, const KGate* gate) {
  const CallInfo& ci = *t->info;
  const TPart& pt = ctx->tr->part(ci.part);
  const int X0 = ci.param_array[0];
  const TArray& a0 = ctx->tr->array(X0);
  int64_t S[3];
  front_shape(a0.ndim, a0.shape, S);
  std::vector<Box> fbs;
  if (boxes) {
    for (const Box& b : *boxes) fbs.push_back(front_box(a0.ndim, b));
  } else {
    fbs.push_back(front_box(a0.ndim, pt.box[q]));
  }
  const Box fb = fbs.empty() ? front_box(a0.ndim, pt.box[q]) : fbs[0];
  cudaStream_t s = stream ? stream : stream_of(ctx, q);
  auto P_ = [&](int param) { return ctx->arr[ci.param_array[param]].ptr[q]; };
  if (ci.kernel == KN_JACOBI5 || ci.kernel == KN_STENCIL9) {
    const size_t nb = fbs.size();
    for (size_t i0 = 0; i0 < std::max<size_t>(nb, 1); i0 += 8) {
      const int64_t* lbs[8];
      const int64_t* ubs[8];
      int n = 0;
      for (size_t i = i0; i < nb && n < 8; i++, n++) {
        lbs[n] = fbs[i].lb;
        ubs[n] = fbs[i].ub;
      }
      const KSync k2 = ks_part(ctx, ks, i0 == 0, i0 + 8 >= nb);
      if (ci.kernel == KN_JACOBI5)
        CK(launch_jacobi5(a0.dtype, P_(1), P_(0), S, lbs, ubs, n, k2, s));
      else
        CK(launch_stencil9(a0.dtype, P_(1), P_(0), S, lbs, ubs, n, k2, s));
      count_launch(ctx);
    }
    return HDA_OK;
  }
  if (fbs.size() > 1 && (ci.kernel == KN_STENCIL7_3D || ci.kernel == KN_SCALE || ci.kernel == KN_COPY)) {
    for (size_t i = 0; i < fbs.size(); i++) {
      std::vector<Box> one{boxes->at(i)};
      int rc = run_kernel(ctx, t, q, scalars, ks_part(ctx, ks, i == 0, i + 1 == fbs.size()), &one, stream);
      if (rc) return rc;
    }
    return HDA_OK;
  }
  switch (ci.kernel) {
    case KN_STENCIL7_3D:
      CK(launch_stencil7(a0.dtype, P_(1), P_(0), S, fb.lb, fb.ub, ks, s));
      break;
    case KN_COPY: {
      RunDesc d = rect_desc(S, fb, a0.es);
      d.src = P_(1);
      d.dst = P_(0);
      std::vector<RunDesc> v{d};
      std::vector<RunBatch> bs;
      batch_descs(v, bs);
      if (bs.size() == 1) {
        CK(launch_copy_runs(bs[0], ks, s));
      } else {
        for (auto& b : bs) CK(launch_copy_runs(b, ks_empty(ctx), s));
        int rc = sync_only(ctx, q, ks);
        if (rc) return rc;
      }
      break;
    }
    case KN_SCALE:
      CK(launch_scale(a0.dtype, P_(0), S, fb.lb, fb.ub, scalars[0], ks, s));
      break;
    case KN_STAMP: {
      const Rects& D = ci.ldef[0][q];
      for (size_t i = 0; i < D.size(); i += 16) {
        BoxList bl;
        bl.n = 0;
        for (size_t j = i; j < D.size() && j < i + 16; j++) {
          Box b = front_box(a0.ndim, D[j]);
          for (int k = 0; k < 3; k++) {
            bl.lb[bl.n][k] = b.lb[k];
            bl.ub[bl.n][k] = b.ub[k];
          }
          bl.n++;
        }
        // waits ride with the first launch, signals with the last
        KSync k2 = ks_empty(ctx);
        if (i == 0) {
          std::memcpy(k2.wait_ptr, ks.wait_ptr, sizeof k2.wait_ptr);
          std::memcpy(k2.wait_val, ks.wait_val, sizeof k2.wait_val);
          k2.nwait = ks.nwait;
        }
        if (i + 16 >= D.size()) {
          std::memcpy(k2.sig_ptr, ks.sig_ptr, sizeof k2.sig_ptr);
          k2.nsig = ks.nsig;
          k2.sig_val = ks.sig_val;
          k2.ctr = ks.ctr;
        }
        CK(launch_stamp((int)a0.es, P_(0), S, bl, (unsigned long long)scalars[0], k2, s));
      }
      break;
    }
    case KN_GEMM: {
      const TArray& A = ctx->tr->array(ci.param_array[1]);
      const TArray& B = ctx->tr->array(ci.param_array[2]);
      const int64_t K = A.shape[1];
      if (gate && gate->n > 0 && gate_mode() == 2 && a0.dtype == HDA_F32) {
        bool done = false;
        int rc = split_product(ctx, q, P_(1), P_(2), P_(0), A.shape[0], B.shape[1], K, fb, (float)scalars[0],
                               (float)scalars[1], ks, s, *gate, &done);
        if (rc) return rc;
        if (done) break;
      }
      if (gate && gate_mode() == 2) {  // not splittable: join the copies first
        CK(cudaStreamWaitEvent(s, ctx->gpus[ctx->dev[q].gpu].ev_pull, 0));
        gate = nullptr;
      }
      cudaError_t e = launch_gemm(a0.dtype, P_(1), P_(2), P_(0), A.shape[0], B.shape[1], A.shape[1], fb.lb, fb.ub,
                                  (float)scalars[0], (float)scalars[1], ks, s, gate);
      if (e == cudaSuccess && gate) __atomic_fetch_add(&ctx->stats.gated_products, (int64_t)1, __ATOMIC_RELAXED);
      if (e == cudaErrorNotSupported && gate) {  // no gated kernel for this shape: join the copies
        CK(cudaStreamWaitEvent(s, ctx->gpus[ctx->dev[q].gpu].ev_pull, 0));
        e = launch_gemm(a0.dtype, P_(1), P_(2), P_(0), A.shape[0], B.shape[1], A.shape[1], fb.lb, fb.ub,
                        (float)scalars[0], (float)scalars[1], ks, s);
      }
      CK(e);
      break;
    }
    default:
      break;
  }
  count_launch(ctx);
  return HDA_OK;
}

static void record_plan(hda_ctx_t* ctx, const Transition* t, bool hit, double us) {
  ctx->last_plan.clear();
  for (const Msg& m : t->msgs) {
    hda_msg_t o;
    o.array = m.array;
    o.src = m.src;
    o.dst = m.dst;
    o.ndim = ctx->tr->array(m.array).ndim;
    for (int k = 0; k < 3; k++) {
      o.lb[k] = m.box.lb[k];
      o.ub[k] = m.box.ub[k];
    }
    ctx->last_plan.push_back(o);
  }
  ctx->stats.n_apply++;
  if (hit)
    ctx->stats.plan_hits++;
  else
    ctx->stats.plan_misses++;
  ctx->stats.last_msgs = (int64_t)t->msgs.size();
  ctx->stats.last_bytes = t->bytes;
  ctx->stats.msgs_total += (int64_t)t->msgs.size();
  ctx->stats.bytes_total += t->bytes;
  ctx->stats.tracker_us += us;
}

static bool arrays_ready(hda_ctx_t* ctx, const CallInfo& ci) {
  if (ctx->plan_only) return true;
  if (!ctx->sync_imported) return false;
  for (int X : ci.arrays)
    if (!ctx->arr[X].imported) return false;
  return true;
}

using clk = std::chrono::steady_clock;

// the full per-call pipeline shared by apply / read / write
// the issue threads, when they apply: single process, >= 2 local GPUs, no kernel
// timing or tracing (their event bookkeeping is serial).  HDA_ISSUE_THREADS=0 disables.
static IssuePool* issue_pool(hda_ctx_t* ctx) {
  static const int on = env_int("HDA_ISSUE_THREADS", 1);
  if (!on || ctx->spmd || ctx->plan_only || ctx->gpus.size() < 2 || ctx->ktiming || ctx->tracing) return nullptr;
  if (!ctx->pool) {
    std::vector<int> ord;
    for (const Gpu& g : ctx->gpus) ord.push_back(g.ordinal);
    ctx->pool = std::make_unique<IssuePool>(ord);
  }
  return ctx->pool.get();
}

// the kernel part of a call whose pull runs on the comm stream (overlap): interior boxes
// while the pull is in flight, dependent boxes after it (or already on the comm stream)
static int issue_overlapped(hda_ctx_t* ctx, const Transition* t, int q, int32_t kernel, const double* scalars,
                            KSync& ks) {
  int rc;
  // interior boxes while the pull is in flight, dependent boxes after it
  const PullJob& job = *ctx->cur_pull[q];
  Gpu& g = ctx->gpus[ctx->dev[q].gpu];
  bool joined = false;
  const bool has_i = !job.interior.empty(), has_d = !job.dependent.empty();
  if (ctx->split_mode[q] == 2) {  // boundary already issued on the comm stream
    ctx->split_mode[q] = 0;
    cudaEvent_t a;
    if ((rc = timed_begin(ctx, g.stream, &a))) return rc;
    if ((rc = run_kernel(ctx, t, q, scalars, ks, &job.interior))) return rc;
    mark(ctx, q, 2);
    if ((rc = timed_end(ctx, g.stream, kernel, a, 1))) return rc;
    CK(cudaStreamWaitEvent(g.stream, g.ev_pull, 0));
    ctx->pulled_on_comm[q] = 0;
    return HDA_OK;
  }
  if (ks.nwait > 0) {
    // The peers' pulls this WAR wait depends on need SM time (their pull kernels)
    // or stall behind GPU-filling kernels (measured: cross-process 3-D peer copies
    // on the copy engine); if every CTA of the interior spun here while the peers
    // did the same, neither GPU would free what the other's pull needs.  Wait in
    // one CTA, then launch the interior with no waits.
    KSync w = ks_empty(ctx);
    std::memcpy(w.wait_ptr, ks.wait_ptr, sizeof w.wait_ptr);
    std::memcpy(w.wait_val, ks.wait_val, sizeof w.wait_val);
    w.nwait = ks.nwait;
    if ((rc = sync_only(ctx, q, w))) return rc;
    ks.nwait = 0;
  }
  if (has_i) {
    cudaEvent_t a;
    if ((rc = timed_begin(ctx, g.stream, &a))) return rc;
    if ((rc = run_kernel(ctx, t, q, scalars, ks_part(ctx, ks, true, !has_d), &job.interior))) return rc;
    mark(ctx, q, 2);
    if ((rc = timed_end(ctx, g.stream, kernel, a, 1))) return rc;
  }
  if (has_d) {
    CK(cudaStreamWaitEvent(g.stream, g.ev_pull, 0));
    joined = true;
    cudaEvent_t a;
    if ((rc = timed_begin(ctx, g.stream, &a))) return rc;
    if ((rc = run_kernel(ctx, t, q, scalars, ks_part(ctx, ks, !has_i, true), &job.dependent))) return rc;
    mark(ctx, q, 3);
    if ((rc = timed_end(ctx, g.stream, kernel, a, has_i ? 0 : 1))) return rc;
  }
  if (!joined) CK(cudaStreamWaitEvent(g.stream, g.ev_pull, 0));
  ctx->pulled_on_comm[q] = 0;
  return HDA_OK;
}

// everything device q issues for call k after its pull: WAR waits, the kernel (or the
// host copy of a write/read), PROD signals.  Thread-safe against other devices' issue.
static int issue_kernel(hda_ctx_t* ctx, const Transition* t, unsigned long long k, int q, int32_t kernel,
                        const double* scalars, const void* host_in, void* host_out) {
  const CallInfo& ci = *t->info;
  const TPart& pt = ctx->tr->part(ci.part);
  int rc;
  bool defines = false;
  for (size_t i = 0; i < ci.arrays.size(); i++)
    if (!ci.ldef[i][q].empty()) defines = true;
  const bool has_work = !box_empty(pt.box[q]);
  const bool kern = kernel > KN_NONE && (kernel == KN_STAMP ? defines : has_work);
  const bool io = (kernel == KN_WRITE && has_work) || (kernel == KN_READ && has_work);
  if (!defines && !kern && !io) return HDA_OK;
  CK(cudaSetDevice(ordinal_of(ctx, q)));
  KSync ks = ks_empty(ctx);
  if (defines) {
    if (!ctx->war_done[q]) war_waits(ctx, ci, q, ks);  // else: carried by the pull
    ctx->war_done[q] = 0;
    signal_prod(ctx, q, k, ks);
    // HDA_DEBUG_FAKE_SIGNAL=1: a kernel with no peer to signal still runs the
    // end-of-kernel fence + counter + store (to a local word) — measures their cost
    static const int fake_sig = env_int("HDA_DEBUG_FAKE_SIGNAL", 0);
    if (fake_sig && ks.nsig == 0) ks_sig(ks, ctx->dev[q].sync + SW_DEBUG);
  }
  // user kernels publish PROD from a trailing signal launch (HDA_SIG_KERNEL=0: from
  // the kernel's last CTA, after a fence in every CTA)
  static const int sig_kernel = env_int("HDA_SIG_KERNEL", 1);
  // the fused halo launch (one kernel per step) keeps its signal in its last CTA: one
  // launch instead of two per step, measured on 4 B200s with 134 MB shares (N=8-sized,
  // 5792^2): 962-968 vs 942-943 GPoints/s (HDA_HALO_SIG_TRAIL=1 restores the trailing
  // launch; profiles/r02/halo_sig/)
  static const int halo_sig_trail = env_int("HDA_HALO_SIG_TRAIL", 0);
  SignalList post_sig;
  post_sig.n = 0;
  const bool split_sig = sig_kernel && kern && !io && ks.nsig > 0 && (halo_sig_trail || !ctx->halo_job[q]);
  if (split_sig) {
    for (int i = 0; i < ks.nsig; i++) post_sig.ptr[i] = ks.sig_ptr[i];
    post_sig.n = ks.nsig;
    post_sig.val = ks.sig_val;
    ks.nsig = 0;
  }
  const int X0 = ci.param_array[0];
  const TArray& a0 = ctx->tr->array(X0);
  if (io) {
    // host copies cannot carry sync words: separate wait before, signal after
    KSync pre = ks_empty(ctx), post = ks_empty(ctx);
    std::memcpy(pre.wait_ptr, ks.wait_ptr, sizeof pre.wait_ptr);
    std::memcpy(pre.wait_val, ks.wait_val, sizeof pre.wait_val);
    pre.nwait = ks.nwait;
    std::memcpy(post.sig_ptr, ks.sig_ptr, sizeof post.sig_ptr);
    post.nsig = ks.nsig;
    post.sig_val = ks.sig_val;
    post.ctr = ks.ctr;
    if ((rc = sync_only(ctx, q, pre))) return rc;
    int64_t S[3];
    front_shape(a0.ndim, a0.shape, S);
    Box fb = front_box(a0.ndim, pt.box[q]);
    cudaMemcpy3DParms p;
    std::memset(&p, 0, sizeof p);
    const size_t es = a0.es;
    void* host = kernel == KN_WRITE ? const_cast<void*>(host_in) : host_out;
    cudaPitchedPtr hp = make_cudaPitchedPtr(host, (size_t)S[2] * es, (size_t)S[2], (size_t)S[1]);
    cudaPitchedPtr dp = make_cudaPitchedPtr(ctx->arr[X0].ptr[q], (size_t)S[2] * es, (size_t)S[2], (size_t)S[1]);
    cudaPos pos = make_cudaPos((size_t)fb.lb[2] * es, (size_t)fb.lb[1], (size_t)fb.lb[0]);
    p.extent = make_cudaExtent((size_t)(fb.ub[2] - fb.lb[2]) * es, (size_t)(fb.ub[1] - fb.lb[1]),
                               (size_t)(fb.ub[0] - fb.lb[0]));
    if (kernel == KN_WRITE) {
      p.srcPtr = hp;
      p.srcPos = pos;
      p.dstPtr = dp;
      p.dstPos = pos;
      p.kind = cudaMemcpyHostToDevice;
    } else {
      p.srcPtr = dp;
      p.srcPos = pos;
      p.dstPtr = hp;
      p.dstPos = pos;
      p.kind = cudaMemcpyDeviceToHost;
    }
    if (host) CK(cudaMemcpy3DAsync(&p, stream_of(ctx, q)));
    if ((rc = sync_only(ctx, q, post))) return rc;
  } else if (kern && ctx->halo_job[q]) {
    // fused halo-exchange stencil: pull + interior + dependent strips, one launch
    const PullJob& job = *ctx->halo_job[q];
    ctx->halo_job[q] = nullptr;
    const CallInfo& ci = *t->info;
    const TArray& a0 = ctx->tr->array(ci.param_array[0]);
    int64_t S[3];
    front_shape(a0.ndim, a0.shape, S);
    std::vector<Box> fb;
    for (const Box& b : job.interior) fb.push_back(front_box(a0.ndim, b));
    for (const Box& b : job.dependent) fb.push_back(front_box(a0.ndim, b));
    const int64_t* lbs[8];
    const int64_t* ubs[8];
    for (size_t i = 0; i < fb.size(); i++) {
      lbs[i] = fb[i].lb;
      ubs[i] = fb[i].ub;
    }
    HaloPull hp;
    std::memset(&hp, 0, sizeof hp);
    for (int p : job.srcs)
      if (!same_stream(ctx, p, q)) {
        if (ctx->last_prod[p]) {
          hp.wait_ptr[hp.nwait] = ctx->dev[q].sync + SW_PROD + p;
          hp.wait_val[hp.nwait++] = ctx->last_prod[p];
        }
        hp.ack_ptr[hp.nack++] = ctx->dev[p].sync + SW_ACK + q;
      }
    for (const auto& e : ctx->pull_war[q]) {
      hp.wait_ptr[hp.nwait] = e.first;
      hp.wait_val[hp.nwait++] = e.second;
    }
    hp.ctr = (unsigned int*)(ctx->dev[q].sync + SW_CTR_PULL);
    hp.done_word = ctx->dev[q].sync + SW_PULLDONE;
    hp.epoch = k;
    hp.delay_ns = pull_delay_ns(q);
    auto P_ = [&](int param) { return ctx->arr[ci.param_array[param]].ptr[q]; };
    cudaStream_t st = stream_of(ctx, q);
    cudaEvent_t a;
    if ((rc = timed_begin(ctx, st, &a))) return rc;
    CK(launch_stencil2d_halo(kernel, a0.dtype, P_(1), P_(0), S, lbs, ubs, (int)fb.size(),
                             (int)job.interior.size(), job.batches[0], hp, ks, st));
    count_launch(ctx);
    mark(ctx, q, 1);
    if ((rc = timed_end(ctx, st, kernel, a, 1))) return rc;
  } else if (kern && ctx->gated[q]) {
    // gated product: starts at once on the main stream, waits per k-block for the rows
    // the comm stream is still copying; joined right after (the next call's work)
    ctx->gated[q] = 0;
    Gpu& g = ctx->gpus[ctx->dev[q].gpu];
    cudaEvent_t a;
    if ((rc = timed_begin(ctx, g.stream, &a))) return rc;
    if ((rc = run_kernel(ctx, t, q, scalars, ks, nullptr, nullptr, &ctx->gate[q]))) return rc;
    mark(ctx, q, 1);
    if ((rc = timed_end(ctx, g.stream, kernel, a))) return rc;
    CK(cudaStreamWaitEvent(g.stream, g.ev_pull, 0));
    ctx->pulled_on_comm[q] = 0;
  } else if (kern && ctx->pulled_on_comm[q]) {
    if ((rc = issue_overlapped(ctx, t, q, kernel, scalars, ks))) return rc;
  } else if (kern) {
    cudaEvent_t a;
    if ((rc = timed_begin(ctx, stream_of(ctx, q), &a))) return rc;
    if ((rc = run_kernel(ctx, t, q, scalars, ks))) return rc;
    mark(ctx, q, 1);
    if ((rc = timed_end(ctx, stream_of(ctx, q), kernel, a))) return rc;
  } else if ((rc = sync_only(ctx, q, ks))) {  // K_NONE definitions
    return rc;
  }
  if (split_sig) {
    CK(launch_signal_pdl(post_sig, ks.relaxed, stream_of(ctx, q)));
    count_launch(ctx);
  }
  return HDA_OK;
}

static int call(hda_ctx_t* ctx, int32_t kernel, hda_part_t part, const AccessIn* acc, int32_t n_acc,
                const double* scalars, int32_t n_scalars, const void* host_in, void* host_out) {
  auto t0 = clk::now();
  const Transition* t = nullptr;
  bool hit = false;
  std::string err;
  int rc = ctx->tr->plan(kernel, part, acc, n_acc, scalars, n_scalars, ctx->cache_on, &t, &hit, err);
  if (rc) return fail(ctx, rc, err);
  double us = std::chrono::duration<double, std::micro>(clk::now() - t0).count();
  const CallInfo& ci = *t->info;
  if (!arrays_ready(ctx, ci)) return fail(ctx, HDA_ESTATE, "SPMD handles not imported for an array");
  const unsigned long long k = ++ctx->epoch;
  if (!ctx->plan_only) {
    DevGuard g(true);
    const bool overlap_kernel = kernel == KN_JACOBI5 || kernel == KN_STENCIL9 || kernel == KN_STENCIL7_3D ||
                                kernel == KN_SCALE || kernel == KN_COPY;
    // HDA_HALO_MODE: 0 split streams — pull + boundary part on the comm stream, interior
    // on the main stream (per-box WAR, HDA_COMM_BOUNDARY); 1 one fused launch (pull
    // blocks + interior + gated boundary strips); -1 fused for the 5-point Jacobi only;
    // -2 (default) split streams, except the fused launch for a 5-point share under
    // 200 MB of traffic per step, where the split shape's host issue (27 vs 14 us per
    // step at N=4, measured) would approach the device step.  Measured on 4 B200s
    // (profiles/r01/comm_boundary/): Jacobi N=4 (268 MB shares) 1297 split vs 1272 fused,
    // N=2 724 vs 712; 9-point N=4 1232 split (fused: 1045).
    static const int halo_mode = env_int("HDA_HALO_MODE", -2);
    bool small_share = false;
    if (halo_mode == -2 && kernel == KN_JACOBI5) {
      const TPart& wp = ctx->tr->part(part);
      const TArray& a0 = ctx->tr->array(ci.param_array[0]);
      for (int q = 0; q < ctx->P; q++)
        if (ctx->dev[q].local && box_volume(wp.box[q]) * 2 * (int64_t)a0.es < 200LL * 1000 * 1000) small_share = true;
    }
    const bool halo_kernel = (halo_mode == 1 && (kernel == KN_JACOBI5 || kernel == KN_STENCIL9)) ||
                             (halo_mode == -1 && kernel == KN_JACOBI5) || small_share;
    ExecPlan scratch;
    ExecPlan* ep = nullptr;
    if ((rc = exchange_plan(ctx, t, k, scratch, &ep))) return rc;
    if (ep && ep->staged && (rc = issue_staged(ctx, ep, k))) return rc;
    IssuePool* pool = issue_pool(ctx);
    if (pool) {
      // one host thread per GPU: its devices' pulls, then their kernels (stream order
      // within a GPU as in the serial path; across GPUs the sync words order everything)
      rc = pool->run([&](int gi) -> int {
        int r;
        if (ep && !ep->staged)
          for (PullJob& job : ep->pulls)
            if (ctx->dev[job.dst].gpu == gi && (r = issue_pull(ctx, t, job, k, overlap_kernel, halo_kernel, scalars))) return r;
        for (int q = 0; q < ctx->P; q++)
          if (ctx->dev[q].local && ctx->dev[q].gpu == gi &&
              (r = issue_kernel(ctx, t, k, q, kernel, scalars, host_in, host_out)))
            return r;
        return HDA_OK;
      });
      if (rc) return rc;
    } else {
      if (ep && !ep->staged)
        for (PullJob& job : ep->pulls)
          if ((rc = issue_pull(ctx, t, job, k, overlap_kernel, halo_kernel, scalars))) return rc;
      for (int q = 0; q < ctx->P; q++)
        if (ctx->dev[q].local && (rc = issue_kernel(ctx, t, k, q, kernel, scalars, host_in, host_out))) return rc;
    }
  }
  for (int q = 0; q < ctx->P && !ctx->plan_only; q++)
    if (ctx->pulled_on_comm[q]) {
      Gpu& g = ctx->gpus[ctx->dev[q].gpu];
      CK(cudaSetDevice(g.ordinal));
      CK(cudaStreamWaitEvent(g.stream, g.ev_pull, 0));
      ctx->pulled_on_comm[q] = 0;
    }
  // every rank knows every device's definitions (SPMD replicated tracker)
  for (int q = 0; q < ctx->P; q++)
    for (size_t i = 0; i < ci.arrays.size(); i++)
      if (!ci.ldef[i][q].empty()) ctx->last_prod[q] = k;
  auto t1 = clk::now();
  ctx->tr->commit(t);
  us += std::chrono::duration<double, std::micro>(clk::now() - t1).count();
  record_plan(ctx, t, hit, us);
  if (!ctx->plan_only && (kernel == KN_WRITE || kernel == KN_READ)) {
    DevGuard g(true);
    if ((rc = sync_all(ctx))) return rc;
  }
  return HDA_OK;
}

// ====================================================================== C-ABI

static hda_ctx_t* new_ctx(int P) {
  hda_ctx_t* ctx = new hda_ctx_t();
  ctx->P = P;
  ctx->tr = std::make_unique<Tracker>(P);
  ctx->dev.assign(P, Dev());
  ctx->last_prod.assign(P, 0);
  ctx->stage_pend.assign(P, {});
  ctx->send_stage.assign(P, nullptr);
  ctx->recv_stage.assign(P, nullptr);
  ctx->send_cap.assign(P, 0);
  ctx->recv_cap.assign(P, 0);
  ctx->pulled_on_comm.assign(P, 0);
  ctx->cur_pull.assign(P, nullptr);
  ctx->halo_job.assign(P, nullptr);
  ctx->gate.assign(P, KGate{});
  ctx->gated.assign(P, 0);
  ctx->split_mode.assign(P, 0);
  ctx->pull_war.assign(P, {});
  ctx->war_done.assign(P, 0);
  // HDA_TIMEOUT_MS: bound on every cross-device wait (default 60 s); a short value
  // turns a protocol deadlock into a prompt HDA_ETIMEOUT when debugging
  if (int ms = env_int("HDA_TIMEOUT_MS", 0)) ctx->timeout_ns = 1000000LL * ms;
  return ctx;
}

static int setup_gpu_common(hda_ctx_t* ctx) {
  for (auto& g : ctx->gpus) {
    CK(cudaSetDevice(g.ordinal));
    CK(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
    // halo pulls get the higher priority: their CTAs are scheduled ahead of the
    // interior kernel's as SM resources free up
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&g.comm, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&g.ev_fork, cudaEventDisableTiming));
    for (cudaEvent_t& e : g.ev_src) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g.ev_pull, cudaEventDisableTiming));
  }
  CK(cudaHostAlloc((void**)&ctx->err_host, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
  *ctx->err_host = 0;
  for (int d = 0; d < ctx->P; d++) {
    if (!ctx->dev[d].local) continue;
    CK(cudaSetDevice(ordinal_of(ctx, d)));
    CK(cudaMalloc((void**)&ctx->dev[d].sync, SW_WORDS * sizeof(unsigned long long)));
    CK(cudaMemset(ctx->dev[d].sync, 0, SW_WORDS * sizeof(unsigned long long)));
    ctx->dev[d].sync_alloc = true;
  }
  CK(cudaDeviceSynchronize());
  return HDA_OK;
}

extern "C" {

const char* hda_version(void) { return "hdarray-b200 0.1 (sm_100a)"; }

int hda_init(hda_ctx_t** out, int32_t n_gpus, const int32_t* gpu_ids, int32_t n_devices) {
  if (!out) return HDA_EINVAL;
  *out = nullptr;
  if (n_devices < 1 || n_devices > HDA_MAX_DEVICES || n_gpus < 0 || n_gpus > n_devices) return HDA_EINVAL;
  hda_ctx_t* ctx = new_ctx(n_devices);
  ctx->plan_only = n_gpus == 0;
  for (int d = 0; d < n_devices; d++) ctx->dev[d].local = true;
  if (!ctx->plan_only) {
    DevGuard g(true);
    for (int i = 0; i < n_gpus; i++) ctx->gpus.push_back(Gpu{gpu_ids ? gpu_ids[i] : i, nullptr});
    for (int d = 0; d < n_devices; d++) ctx->dev[d].gpu = d % n_gpus;
    for (int i = 0; i < n_gpus; i++) {
      cudaError_t e = cudaSetDevice(ctx->gpus[i].ordinal);
      if (e != cudaSuccess) {
        *out = ctx;
        return cuda_fail(ctx, e, "cudaSetDevice");
      }
      for (int j = 0; j < n_gpus; j++) {
        if (i == j || ctx->gpus[i].ordinal == ctx->gpus[j].ordinal) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, ctx->gpus[i].ordinal, ctx->gpus[j].ordinal);
        if (!can) {
          *out = ctx;
          return fail(ctx, HDA_EUNSUPPORTED, "GPUs without peer access");
        }
        e = cudaDeviceEnablePeerAccess(ctx->gpus[j].ordinal, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) {
          *out = ctx;
          return cuda_fail(ctx, e, "cudaDeviceEnablePeerAccess");
        }
      }
    }
    int rc = setup_gpu_common(ctx);
    if (rc) {
      *out = ctx;
      return rc;
    }
  }
  *out = ctx;
  return HDA_OK;
}

int hda_init_spmd(hda_ctx_t** out, int32_t n_devices, int32_t rank, int32_t gpu_id) {
  if (!out) return HDA_EINVAL;
  *out = nullptr;
  if (n_devices < 1 || n_devices > HDA_MAX_DEVICES || rank < 0 || rank >= n_devices) return HDA_EINVAL;
  hda_ctx_t* ctx = new_ctx(n_devices);
  ctx->spmd = true;
  ctx->rank = rank;
  ctx->plan_only = gpu_id < 0;
  ctx->dev[rank].local = true;
  if (ctx->plan_only) {
    for (int d = 0; d < n_devices; d++) ctx->dev[d].local = d == rank;
  } else {
    DevGuard g(true);
    ctx->gpus.push_back(Gpu{gpu_id, nullptr});
    ctx->dev[rank].gpu = 0;
    ctx->sync_imported = n_devices == 1;
    int rc = setup_gpu_common(ctx);
    *out = ctx;
    return rc;
  }
  *out = ctx;
  return HDA_OK;
}

int hda_finalize(hda_ctx_t* ctx) {
  if (!ctx) return HDA_EINVAL;
  ctx->pool.reset();  // join the issue threads before their streams go away
  if (!ctx->plan_only) {
    DevGuard g(true);
    for (auto& gp : ctx->gpus) {
      cudaSetDevice(gp.ordinal);
      cudaStreamSynchronize(gp.stream);
    }
    for (size_t X = 0; X < ctx->arr.size(); X++)
      for (int d = 0; d < ctx->P; d++) {
        if (ctx->arr[X].alloc.size() && ctx->arr[X].alloc[d]) {
          cudaSetDevice(ordinal_of(ctx, d));
          cudaFree(ctx->arr[X].ptr[d]);
        } else if (ctx->arr[X].ipc.size() && ctx->arr[X].ipc[d]) {
          cudaIpcCloseMemHandle(ctx->arr[X].ptr[d]);
        }
      }
    for (int d = 0; d < ctx->P; d++) {
      if (ctx->dev[d].sync_alloc) {
        cudaSetDevice(ordinal_of(ctx, d));
        cudaFree(ctx->dev[d].sync);
      } else if (ctx->dev[d].sync_ipc) {
        cudaIpcCloseMemHandle(ctx->dev[d].sync);
      }
      if (ctx->send_stage[d]) cudaFree(ctx->send_stage[d]);
      if (ctx->recv_stage[d]) cudaFree(ctx->recv_stage[d]);
    }
    for (auto& e : ctx->tev) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    for (auto& gp : ctx->gpus) {
      cudaSetDevice(gp.ordinal);
      cudaStreamDestroy(gp.stream);
      cudaStreamDestroy(gp.comm);
      cudaEventDestroy(gp.ev_fork);
      cudaEventDestroy(gp.ev_pull);
      for (cudaEvent_t e : gp.ev_src)
        if (e) cudaEventDestroy(e);
    }
    if (ctx->err_host) cudaFreeHost(ctx->err_host);
  }
  delete ctx;
  return HDA_OK;
}

int hda_num_devices(const hda_ctx_t* ctx, int32_t* n) {
  if (!ctx || !n) return HDA_EINVAL;
  *n = ctx->P;
  return HDA_OK;
}

int hda_is_local(const hda_ctx_t* ctx, int32_t dev, int32_t* is_local) {
  if (!ctx || !is_local || dev < 0 || dev >= ctx->P) return HDA_EINVAL;
  *is_local = ctx->dev[dev].local ? 1 : 0;
  return HDA_OK;
}

int hda_spmd_export(hda_ctx_t* ctx, hda_array_t arr, void* out) {
  GUARD();
  if (!out) return fail(ctx, HDA_EINVAL, "null blob");
  std::memset(out, 0, HDA_HANDLE_BYTES);
  if (!ctx->spmd || ctx->plan_only) return HDA_OK;
  char* base;
  if (arr == -1) {
    base = (char*)ctx->dev[ctx->rank].sync;
  } else {
    if (!ctx->tr->array_ok(arr)) return fail(ctx, HDA_EINVAL, "unknown array");
    base = ctx->arr[arr].ptr[ctx->rank];
  }
  DevGuard g(true);
  CK(cudaSetDevice(ctx->gpus[0].ordinal));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, base));
  uint32_t hdr[2] = {BLOB_MAGIC, (uint32_t)ctx->rank};
  std::memcpy(out, hdr, 8);
  std::memcpy((char*)out + 8, &h, sizeof h);
  return HDA_OK;
}

int hda_spmd_import(hda_ctx_t* ctx, hda_array_t arr, const void* all) {
  GUARD();
  if (!all) return fail(ctx, HDA_EINVAL, "null blobs");
  if (!ctx->spmd || ctx->plan_only) return HDA_OK;
  if (arr != -1 && !ctx->tr->array_ok(arr)) return fail(ctx, HDA_EINVAL, "unknown array");
  DevGuard g(true);
  CK(cudaSetDevice(ctx->gpus[0].ordinal));
  for (int p = 0; p < ctx->P; p++) {
    if (p == ctx->rank) continue;
    const char* b = (const char*)all + (size_t)p * HDA_HANDLE_BYTES;
    uint32_t hdr[2];
    std::memcpy(hdr, b, 8);
    if (hdr[0] != BLOB_MAGIC || (int)hdr[1] != p) return fail(ctx, HDA_EINVAL, "bad SPMD blob");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, b + 8, sizeof h);
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    if (arr == -1) {
      ctx->dev[p].sync = (unsigned long long*)ptr;
      ctx->dev[p].sync_ipc = true;
    } else {
      ctx->arr[arr].ptr[p] = (char*)ptr;
      ctx->arr[arr].ipc[p] = 1;
    }
  }
  if (arr == -1)
    ctx->sync_imported = true;
  else
    ctx->arr[arr].imported = true;
  return HDA_OK;
}

static int create_common(hda_ctx_t* ctx, int32_t dtype, int32_t ndim, const int64_t* shape, hda_array_t* out,
                         int* id_out) {
  if (!shape || !out) return fail(ctx, HDA_EINVAL, "null argument");
  std::string err;
  int id = ctx->tr->add_array(dtype, ndim, shape, err);
  if (id < 0) return fail(ctx, id, err);
  ArrRT a;
  a.ptr.assign(ctx->P, nullptr);
  a.alloc.assign(ctx->P, 0);
  a.ipc.assign(ctx->P, 0);
  const TArray& t = ctx->tr->array(id);
  a.bytes = (size_t)(t.shape[0] * t.shape[1] * t.shape[2]) * t.es;
  a.imported = !ctx->spmd || ctx->P == 1 || ctx->plan_only;
  ctx->arr.push_back(a);
  ctx->pend.emplace_back(ctx->P, std::vector<unsigned long long>(ctx->P, 0));
  ctx->rread.emplace_back(ctx->P);
  ctx->rread_over.emplace_back(ctx->P, 0);
  *id_out = id;
  return HDA_OK;
}

int hda_create(hda_ctx_t* ctx, int32_t dtype, int32_t ndim, const int64_t* shape, const void* init_host,
               hda_array_t* out) {
  GUARD();
  int id;
  int rc = create_common(ctx, dtype, ndim, shape, out, &id);
  if (rc) return rc;
  if (!ctx->plan_only) {
    DevGuard g(true);
    ArrRT& a = ctx->arr[id];
    for (int d = 0; d < ctx->P; d++) {
      if (!ctx->dev[d].local) continue;
      CK(cudaSetDevice(ordinal_of(ctx, d)));
      void* p = nullptr;
      cudaError_t e = cudaMalloc(&p, a.bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, HDA_ENOMEM, "cudaMalloc of a replica failed");
      }
      a.ptr[d] = (char*)p;
      a.alloc[d] = 1;
      if (init_host)
        CK(cudaMemcpy(p, init_host, a.bytes, cudaMemcpyHostToDevice));
      else
        CK(cudaMemset(p, 0, a.bytes));
    }
    CK(cudaDeviceSynchronize());
  }
  *out = id;
  return HDA_OK;
}

int hda_create_ext(hda_ctx_t* ctx, int32_t dtype, int32_t ndim, const int64_t* shape, void* const* dev_ptrs,
                   hda_array_t* out) {
  GUARD();
  if (ctx->spmd) return fail(ctx, HDA_EUNSUPPORTED, "hda_create_ext is single-process only");
  if (!dev_ptrs && !ctx->plan_only) return fail(ctx, HDA_EINVAL, "null device pointers");
  int id;
  int rc = create_common(ctx, dtype, ndim, shape, out, &id);
  if (rc) return rc;
  if (!ctx->plan_only)
    for (int d = 0; d < ctx->P; d++) ctx->arr[id].ptr[d] = (char*)dev_ptrs[d];
  *out = id;
  return HDA_OK;
}

int hda_free(hda_ctx_t* ctx, hda_array_t arr) {
  GUARD();
  if (!ctx->tr->array_ok(arr)) return fail(ctx, HDA_EINVAL, "unknown array");
  if (!ctx->plan_only) {
    DevGuard g(true);
    int rc = sync_all(ctx);
    if (rc) return rc;
    ArrRT& a = ctx->arr[arr];
    for (int d = 0; d < ctx->P; d++) {
      if (a.alloc[d]) {
        CK(cudaSetDevice(ordinal_of(ctx, d)));
        CK(cudaFree(a.ptr[d]));
      } else if (a.ipc[d]) {
        CK(cudaIpcCloseMemHandle(a.ptr[d]));
      }
      a.ptr[d] = nullptr;
      a.alloc[d] = a.ipc[d] = 0;
    }
  }
  ctx->tr->free_array(arr);
  ctx->exec.clear();
  return HDA_OK;
}

int hda_device_ptr(hda_ctx_t* ctx, hda_array_t arr, int32_t dev, void** out) {
  GUARD();
  if (!out || !ctx->tr->array_ok(arr) || dev < 0 || dev >= ctx->P) return fail(ctx, HDA_EINVAL, "bad argument");
  *out = ctx->arr[arr].ptr[dev];
  return HDA_OK;
}

int hda_partition(hda_ctx_t* ctx, int32_t kind, int32_t ndim, const int64_t* domain, const int64_t* lb,
                  const int64_t* ub, hda_part_t* out) {
  GUARD();
  if (!domain || !lb || !ub || !out) return fail(ctx, HDA_EINVAL, "null argument");
  std::string err;
  int id = ctx->tr->add_partition(kind, ndim, domain, lb, ub, err);
  if (id < 0) return fail(ctx, id, err);
  *out = id;
  return HDA_OK;
}

int hda_partition_manual(hda_ctx_t* ctx, int32_t ndim, const int64_t* domain, const int64_t* lbs,
                         const int64_t* ubs, hda_part_t* out) {
  GUARD();
  if (!domain || !lbs || !ubs || !out) return fail(ctx, HDA_EINVAL, "null argument");
  std::string err;
  int id = ctx->tr->add_partition_manual(ndim, domain, lbs, ubs, err);
  if (id < 0) return fail(ctx, id, err);
  *out = id;
  return HDA_OK;
}

int hda_partition_region(const hda_ctx_t* ctx, hda_part_t part, int32_t dev, int64_t* lb, int64_t* ub) {
  if (!ctx || !lb || !ub || !ctx->tr->part_ok(part) || dev < 0 || dev >= ctx->P) return HDA_EINVAL;
  const TPart& p = ctx->tr->part(part);
  for (int k = 0; k < p.ndim; k++) {
    lb[k] = p.box[dev].lb[k];
    ub[k] = p.box[dev].ub[k];
  }
  return HDA_OK;
}

int hda_apply(hda_ctx_t* ctx, int32_t kernel, hda_part_t part, const hda_access_t* acc, int32_t n_acc,
              const double* scalars, int32_t n_scalars) {
  GUARD();
  if (kernel < 0 || kernel >= KN_COUNT) return fail(ctx, HDA_EINVAL, "unknown kernel");
  if (n_acc < 0 || n_acc > 64 || (n_acc && !acc)) return fail(ctx, HDA_EINVAL, "bad access list");
  if (n_scalars < 0 || (n_scalars && !scalars)) return fail(ctx, HDA_EINVAL, "bad scalars");
  AccessIn in[64];
  for (int i = 0; i < n_acc; i++) in[i] = AccessIn{acc[i].array, acc[i].n_use, acc[i].use, acc[i].n_def, acc[i].def};
  return call(ctx, kernel, part, in, n_acc, scalars, n_scalars, nullptr, nullptr);
}

int hda_apply_abs(hda_ctx_t* ctx, int32_t kernel, hda_part_t part, const hda_abs_access_t* acc, int32_t n_acc,
                  const double* scalars, int32_t n_scalars) {
  GUARD();
  if (kernel < 0 || kernel >= KN_COUNT) return fail(ctx, HDA_EINVAL, "unknown kernel");
  if (n_acc < 1 || n_acc > 64 || !acc) return fail(ctx, HDA_EINVAL, "bad access list");
  if (n_scalars < 0 || (n_scalars && !scalars)) return fail(ctx, HDA_EINVAL, "bad scalars");
  AccessIn in[64];
  static const int32_t zeros[HDA_MAX_DEVICES] = {0};
  for (int i = 0; i < n_acc; i++) {
    in[i] = AccessIn{acc[i].array, 0, nullptr, 0, nullptr};
    in[i].n_use_abs = acc[i].n_use ? acc[i].n_use : zeros;
    in[i].use_abs = acc[i].use;
    in[i].n_def_abs = acc[i].n_def ? acc[i].n_def : zeros;
    in[i].def_abs = acc[i].def;
  }
  return call(ctx, kernel, part, in, n_acc, scalars, n_scalars, nullptr, nullptr);
}

// Table 2 SetTrapezoidUse/Def rasterized to per-row boxes
// (reading R20: inclusive corners, row edges interpolated and rounded half up)
static int64_t floordiv64(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) != 0 && ((a < 0) != (b < 0))) q--;
  return q;
}

int hda_trapezoid(const int64_t* c, int64_t* boxes, int32_t cap, int32_t* n_out) {
  if (!c || !n_out) return HDA_EINVAL;
  const int64_t top = c[0], bottom = c[4];
  if (c[2] != top || c[6] != bottom || bottom < top) return HDA_EINVAL;
  const int64_t h = bottom - top;
  int32_t n = 0;
  for (int64_t r = top; r <= bottom; r++) {
    const int64_t left = h ? c[1] + floordiv64((r - top) * (c[5] - c[1]) * 2 + h, 2 * h) : c[1];
    const int64_t right = h ? c[3] + floordiv64((r - top) * (c[7] - c[3]) * 2 + h, 2 * h) : c[3];
    if (left > right) continue;
    if (boxes && n < cap) {
      boxes[4 * n + 0] = r;
      boxes[4 * n + 1] = left;
      boxes[4 * n + 2] = r + 1;
      boxes[4 * n + 3] = right + 1;
    }
    n++;
  }
  *n_out = n;
  return HDA_OK;
}

int hda_sync(hda_ctx_t* ctx) {
  GUARD();
  if (ctx->plan_only) return HDA_OK;
  DevGuard g(true);
  return sync_all(ctx);
}

int hda_write(hda_ctx_t* ctx, hda_array_t arr, hda_part_t part, const void* host_full) {
  GUARD();
  if (!ctx->tr->array_ok(arr)) return fail(ctx, HDA_EINVAL, "unknown array");
  if (!host_full && !ctx->plan_only) return fail(ctx, HDA_EINVAL, "null host buffer");
  static const int32_t zero[3] = {0, 0, 0};
  AccessIn in{arr, 0, nullptr, 1, zero};
  return call(ctx, KN_WRITE, part, &in, 1, nullptr, 0, host_full, nullptr);
}

int hda_read(hda_ctx_t* ctx, hda_array_t arr, hda_part_t part, void* host_full) {
  GUARD();
  if (!ctx->tr->array_ok(arr)) return fail(ctx, HDA_EINVAL, "unknown array");
  static const int32_t zero[3] = {0, 0, 0};
  AccessIn in{arr, 1, zero, 0, nullptr};
  return call(ctx, KN_READ, part, &in, 1, nullptr, 0, nullptr, host_full);
}

int hda_reduce(hda_ctx_t* ctx, hda_array_t arr, hda_part_t part, int32_t op, double* out) {
  GUARD();
  if (!out || op < HDA_SUM || op > HDA_MIN) return fail(ctx, HDA_EINVAL, "bad reduce argument");
  if (!ctx->tr->array_ok(arr)) return fail(ctx, HDA_EINVAL, "unknown array");
  static const int32_t zero[3] = {0, 0, 0};
  AccessIn in{arr, 1, zero, 0, nullptr};
  int rc = call(ctx, KN_READ, part, &in, 1, nullptr, 0, nullptr, nullptr);  // coherence
  if (rc) return rc;
  if (ctx->plan_only) return fail(ctx, HDA_ESTATE, "reduce needs data (plan-only context)");
  const TArray& a = ctx->tr->array(arr);
  const TPart& pt = ctx->tr->part(part);
  const bool is_int = a.dtype == DT_I32 || a.dtype == DT_I64;
  const unsigned long long k = ++ctx->epoch;
  // SPMD: peers write their partials into this rank's slots.  Alternating two banks
  // keeps a fast rank's partial of the NEXT reduce out of the slots this rank's host
  // may still be reading: to start reduce n+2 (same bank as n) a rank must have seen
  // every peer's share of reduce n+1, which each peer issues only after its host
  // finished reading reduce n.
  const int red = (ctx->n_reduce++ & 1) ? SW_RED_B : SW_RED;
  DevGuard g(true);
  int64_t S[3];
  front_shape(a.ndim, a.shape, S);
  for (int q = 0; q < ctx->P; q++) {
    if (!ctx->dev[q].local) continue;
    CK(cudaSetDevice(ordinal_of(ctx, q)));
    unsigned long long* sw = ctx->dev[q].sync;
    const Box fb = front_box(a.ndim, pt.box[q]);
    CK(launch_reduce(a.dtype, ctx->arr[arr].ptr[q], S, fb.lb, fb.ub, op, sw + SW_SCRATCH, sw + red + q,
                     stream_of(ctx, q)));
    count_launch(ctx, 2);
    if (ctx->spmd && ctx->P > 1) {  // publish this rank's partial to every peer
      SignalList slots, flags;
      slots.n = flags.n = 0;
      flags.val = k;
      for (int r = 0; r < ctx->P; r++) {
        if (r == q) continue;
        slots.ptr[slots.n++] = ctx->dev[r].sync + red + q;
        flags.ptr[flags.n++] = ctx->dev[r].sync + SW_REDSIG + q;
      }
      CK(launch_share(sw + red + q, slots, flags, stream_of(ctx, q)));
      KSync w = ks_empty(ctx);
      for (int r = 0; r < ctx->P; r++)
        if (r != q) ks_wait(w, sw + SW_REDSIG + r, k);
      if ((rc = sync_only(ctx, q, w))) return rc;
      count_launch(ctx);
    }
  }
  if ((rc = sync_all(ctx))) return rc;
  // test hook: a host that reads its partials late (the window in which a fast peer's
  // next reduce could overwrite them without the bank alternation above)
  static const int read_delay_us = env_int("HDA_DEBUG_REDUCE_READ_DELAY_US", 0);
  if (read_delay_us) std::this_thread::sleep_for(std::chrono::microseconds(read_delay_us));
  // combine the P partials in device order (identical on every rank)
  double acc = op == HDA_SUM ? 0.0 : op == HDA_PROD ? 1.0 : op == HDA_MAX ? -HUGE_VAL : HUGE_VAL;
  long long iacc = op == HDA_PROD ? 1 : op == HDA_MAX ? LLONG_MIN : op == HDA_MIN ? LLONG_MAX : 0;
  for (int p = 0; p < ctx->P; p++) {
    int src = ctx->spmd ? ctx->rank : p;  // where p's partial lives in this process
    unsigned long long bits = 0;
    CK(cudaSetDevice(ordinal_of(ctx, src)));
    CK(cudaMemcpy(&bits, ctx->dev[src].sync + red + p, 8, cudaMemcpyDeviceToHost));
    if (is_int) {
      long long v;
      std::memcpy(&v, &bits, 8);
      iacc = op == HDA_SUM ? iacc + v : op == HDA_PROD ? iacc * v : op == HDA_MAX ? std::max(iacc, v) : std::min(iacc, v);
    } else {
      double v;
      std::memcpy(&v, &bits, 8);
      acc = op == HDA_SUM ? acc + v : op == HDA_PROD ? acc * v : op == HDA_MAX ? (v > acc ? v : acc) : (v < acc ? v : acc);
    }
  }
  *out = is_int ? (double)iacc : acc;
  return HDA_OK;
}

int hda_set_transport(hda_ctx_t* ctx, int32_t transport) {
  GUARD();
  if (transport != HDA_XPORT_FUSED && transport != HDA_XPORT_STAGED && transport != HDA_XPORT_AUTO)
    return fail(ctx, HDA_EINVAL, "transport");
  if (transport == HDA_XPORT_STAGED && ctx->spmd && ctx->P > 1)
    return fail(ctx, HDA_EUNSUPPORTED, "staged transport is single-process only");
  ctx->transport = transport;
  return HDA_OK;
}

int hda_set_overlap(hda_ctx_t* ctx, int32_t enabled) {
  GUARD();
  ctx->overlap = enabled != 0;
  return HDA_OK;
}

int hda_set_plan_cache(hda_ctx_t* ctx, int32_t enabled) {
  GUARD();
  ctx->cache_on = enabled != 0;
  return HDA_OK;
}

int hda_set_kernel_timing(hda_ctx_t* ctx, int32_t enabled) {
  GUARD();
  ctx->ktiming = enabled != 0 && !ctx->plan_only;
  return HDA_OK;
}

static int drain_timing(hda_ctx_t* ctx) {
  if (ctx->tev.empty()) return HDA_OK;
  DevGuard g(true);
  int rc = sync_all(ctx);
  if (rc) return rc;
  for (auto& e : ctx->tev) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e.a, e.b));
    if (e.kind == -100) {
      ctx->xtime_ms += ms;
      ctx->xcount += e.count;
    } else if (e.kind >= 0 && e.kind < KN_COUNT) {
      ctx->ktime_ms[e.kind] += ms;
      ctx->kcount[e.kind] += e.count;
    }
    ctx->ev_pool.push_back(e.a);
    ctx->ev_pool.push_back(e.b);
  }
  ctx->tev.clear();
  return HDA_OK;
}

int hda_kernel_time(hda_ctx_t* ctx, int32_t kernel, double* total_ms, int64_t* launches) {
  GUARD();
  if (kernel < 0 || kernel >= KN_COUNT || !total_ms || !launches) return fail(ctx, HDA_EINVAL, "bad argument");
  int rc = drain_timing(ctx);
  if (rc) return rc;
  *total_ms = ctx->ktime_ms[kernel];
  *launches = ctx->kcount[kernel];
  return HDA_OK;
}

int hda_exchange_time(hda_ctx_t* ctx, double* total_ms, int64_t* n) {
  GUARD();
  if (!total_ms || !n) return fail(ctx, HDA_EINVAL, "bad argument");
  int rc = drain_timing(ctx);
  if (rc) return rc;
  *total_ms = ctx->xtime_ms;
  *n = ctx->xcount;
  return HDA_OK;
}

int hda_set_trace(hda_ctx_t* ctx, int32_t enabled) {
  GUARD();
  if (ctx->plan_only) return HDA_OK;
  DevGuard g(true);
  if (enabled && !ctx->tracing) {
    for (auto& e : ctx->trace) {
      ctx->ev_pool.push_back(e.a);
      ctx->ev_pool.push_back(e.b);
    }
    ctx->trace.clear();
    if (!ctx->trace_ref) CK(cudaEventCreate(&ctx->trace_ref));
    const int d0 = ctx->spmd ? ctx->rank : 0;
    CK(cudaSetDevice(ordinal_of(ctx, d0)));
    CK(cudaEventRecord(ctx->trace_ref, stream_of(ctx, d0)));
  }
  ctx->tracing = enabled != 0;
  return HDA_OK;
}

int hda_trace(hda_ctx_t* ctx, double* out, int32_t cap, int32_t* n_out) {
  GUARD();
  if (!n_out) return fail(ctx, HDA_EINVAL, "null n_out");
  *n_out = (int32_t)ctx->trace.size();
  if (!out || ctx->trace.empty()) return HDA_OK;
  DevGuard g(true);
  int rc = sync_all(ctx);
  if (rc) return rc;
  for (int32_t i = 0; i < cap && i < *n_out; i++) {
    const TimedEv& e = ctx->trace[i];
    float t0 = 0, t1 = 0;
    CK(cudaEventElapsedTime(&t0, ctx->trace_ref, e.a));
    CK(cudaEventElapsedTime(&t1, ctx->trace_ref, e.b));
    out[5 * i + 0] = (double)e.epoch;
    out[5 * i + 1] = e.dev;
    out[5 * i + 2] = e.phase;
    out[5 * i + 3] = t0 * 1e3;
    out[5 * i + 4] = t1 * 1e3;
  }
  return HDA_OK;
}

int hda_stream(hda_ctx_t* ctx, int32_t dev, void** stream) {
  GUARD();
  if (!stream || dev < 0 || dev >= ctx->P || !ctx->dev[dev].local || ctx->plan_only)
    return fail(ctx, HDA_EINVAL, "no stream for that device");
  *stream = (void*)stream_of(ctx, dev);
  return HDA_OK;
}

int hda_last_plan(const hda_ctx_t* ctx, hda_msg_t* out, int32_t cap, int32_t* n_out) {
  if (!ctx || !n_out) return HDA_EINVAL;
  *n_out = (int32_t)ctx->last_plan.size();
  if (out)
    for (int32_t i = 0; i < cap && i < *n_out; i++) out[i] = ctx->last_plan[i];
  return HDA_OK;
}

int hda_owner_map(const hda_ctx_t* ctx, hda_array_t arr, int8_t* out) {
  if (!ctx || !out || !ctx->tr->array_ok(arr)) return HDA_EINVAL;
  ctx->tr->owner_map(arr, out);
  return HDA_OK;
}

int hda_read_replica(hda_ctx_t* ctx, hda_array_t arr, int32_t dev, void* host_full) {
  GUARD();
  if (!ctx->tr->array_ok(arr) || !host_full || dev < 0 || dev >= ctx->P || !ctx->dev[dev].local || ctx->plan_only)
    return fail(ctx, HDA_EINVAL, "bad argument");
  DevGuard g(true);
  int rc = sync_all(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ordinal_of(ctx, dev)));
  CK(cudaMemcpy(host_full, ctx->arr[arr].ptr[dev], ctx->arr[arr].bytes, cudaMemcpyDeviceToHost));
  return HDA_OK;
}

int hda_stats(const hda_ctx_t* ctx, hda_stats_t* out) {
  if (!ctx || !out) return HDA_EINVAL;
  *out = ctx->stats;
  return HDA_OK;
}

int hda_reset_stats(hda_ctx_t* ctx) {
  if (!ctx) return HDA_EINVAL;
  int rc = drain_timing(ctx);
  ctx->stats = hda_stats_t{};
  for (int k = 0; k < KN_COUNT; k++) {
    ctx->ktime_ms[k] = 0;
    ctx->kcount[k] = 0;
  }
  ctx->xtime_ms = 0;
  ctx->xcount = 0;
  return rc;
}

const char* hda_last_error(const hda_ctx_t* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

}  // extern "C"
