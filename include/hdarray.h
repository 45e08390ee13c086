/*
 * hdarray.h — C-ABI boundary of the B200-native HDArray def/use exchange runtime.
 *
 * Paper: Cho, Kwon, Midkiff, "HDArray: Parallel Array Interface for Distributed
 * Heterogeneous Devices", arXiv:1809.05657.  Citations "P:Lnnn" are lines of
 * /root/reference/PAPER.md (the LaTeX source; lines 1-595 are the paper).
 *
 * What this library computes (§1): "HDArray knows where the last written
 * copy of a datum is, and who needs that value".  For every kernel call k under a
 * work partition W, each device q's use set LUSE_q(X) is composed from the
 * kernel's use offsets and W_q; the message set is
 *     M_{p->q}(X) = LUSE_q(X) ∩ Own_p(X) − Valid_q(X)          (Eq. 1-2)
 * where Own_p = cells whose last writer is p and Valid_q = cells for which q holds
 * the current value; after the transfer and the kernel, the sets are updated with
 * last-writer semantics (Eq. 3-4, corrected: DESIGN.md reading R7).
 * Messages move device->device over NVLink (pack / transfer / unpack)
 * and then the built-in kernel runs on every device's work region.
 *
 * Conventions (apply to every call):
 *  - Arrays are dense, row-major (last dimension contiguous), 1 <= ndim <= 3.
 *    EVERY device holds a full-size replica of every array ("allocates host
 *    and device buffers with the same size of user-space arrays"), so a message is
 *    one rectangle at identical global coordinates on both sides.
 *  - Boxes are half-open [lb, ub) per dimension in global element coordinates
 *    (reading R1: the paper's "[LB:UB]", is not said to be inclusive).
 *  - Offsets: int32 per dimension; HDA_STAR ('*') means "the whole extent
 *    of that dimension of the accessed array".  Composition shifts W_p by each
 *    offset tuple and clamps to the array bounds (reading R6).
 *  - Return value: HDA_OK (0) or a negative HDA_E* code; hda_last_error() gives a
 *    message.  Validation errors (EINVAL, ERANGE, EOVERLAP, ERACE, EUNSUPPORTED)
 *    are detected before any state change: the call has no effect.  ECUDA and
 *    ETIMEOUT are sticky: the context is poisoned and only hda_finalize is valid.
 *  - Host pointers are borrowed for the duration of the call only.  Device memory
 *    allocated by hda_create is owned by the context; memory passed to
 *    hda_create_ext is borrowed and must outlive hda_free / hda_finalize.
 *  - One context per host thread; calls are not re-entrant.  Device work is
 *    asynchronous (hda_apply returns once everything is enqueued; the tracker
 *    commit for call k happens on the host while the GPUs run it);
 *    hda_sync, hda_read, hda_read_replica block.
 *
 * Process models:
 *  - hda_init: one process drives P "devices" mapped round-robin onto n_gpus
 *    physical GPUs (P > n_gpus gives virtual devices sharing a GPU, used for
 *    parity tests on one GPU).  n_gpus == 0 gives a PLAN-ONLY context: the
 *    tracker runs (plans, owner maps, stats) but no memory is touched.
 *  - hda_init_spmd: the paper's SPMD model ("Each MPI process that maps to a
 *    single OpenCL device"; P:L105 every process keeps copies of all sets): rank r
 *    drives device r on one GPU; every rank runs the same deterministic tracker and
 *    computes the same plans; replica buffers and sync words of peers are mapped
 *    with CUDA IPC after the ranks swap handles (hda_spmd_export/import; the
 *    Python binding does the swap over torch.distributed).  Every rank must issue
 *    the same sequence of calls.
 */
#ifndef HDARRAY_H
#define HDARRAY_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HDA_MAX_DIM 3
#define HDA_MAX_DEVICES 64
#define HDA_STAR INT32_MIN          /* '*' offset: whole extent of the dimension */
#define HDA_HANDLE_BYTES 128        /* size of one SPMD export blob */

/* element types (SPEC S:L126 lists f32/f64/i32/i64; bf16 for the dense product) */
enum hda_dtype { HDA_F64 = 0, HDA_F32 = 1, HDA_BF16 = 2, HDA_I32 = 3, HDA_I64 = 4 };

/* automatic partitions, P:L241 (Table 2 "Supported types: ROW, COL, and BLOCK") */
enum hda_part_kind { HDA_ROW = 0, HDA_COL = 1, HDA_BLOCK = 2 };

/* built-in kernels (the paper's benchmark kernels, §5.1, plus helpers).
 * Parameter order of the access list of hda_apply is fixed per kernel:
 *  HDA_K_NONE        any params; declared uses/defs are tracked, no device code runs
 *  HDA_K_JACOBI5     [dst A, src B]  A = (((B[i][j-1]+B[i][j+1])+B[i-1][j])+B[i+1][j])*0.25
 *                    (uses of B must cover (0,-1),(0,1),(-1,0),(1,0))
 *  HDA_K_COPY        [dst B, src A]  B = A, raw bits ("B[i][j]=A[i][j]")
 *  HDA_K_STENCIL9    [dst Y, src X]  e=((W+E)+N)+S; c=((NW+NE)+SW)+SE; Y=(4*e+c)/20
 *                    (Convolution, "eight neighbors"; weights: reading R12)
 *  HDA_K_STENCIL7_3D [dst Y, src X]  s=((((x-+x+)+y-)+y+)+z-)+z+; Y=s/6 (reading R13)
 *  HDA_K_SCALE       [X]            X = alpha*X in X's dtype (scalars[0] = alpha)
 *  HDA_K_GEMM        [C, A, B]      C = alpha*sum_k A[i][k]*B[k][j] + beta*C
 *                    (Listing 2; A,B bf16, C f32 or bf16, fp32 accumulate
 *                    on tensor cores; scalars = {alpha, beta}; uses A (0,*), B (*,0),
 *                    C (0,0) iff beta != 0)
 *  HDA_K_STAMP       [X, Y...]      every cell c of the composed DEF set of device p
 *                    gets the low bytes of splitmix64(seed*0x9E3779B97F4A7C15 + c)
 *                    (c = linear index; scalars[0] = seed); a test kernel that
 *                    writes arbitrary def shapes with distinctive raw bits.  Extra
 *                    parameters Y may declare uses (their data moves) but no defs.
 * Built-in kernels other than NONE/STAMP require def offsets == {(0,..,0)} and
 * declared uses covering their true footprint (EINVAL), and work ⊕ footprint
 * inside the array (ERANGE).  An array used at a non-zero offset and defined in
 * the same call is EINVAL (bulk-synchronous semantics, reading R15). */
enum hda_kernel {
  HDA_K_NONE = 0,
  HDA_K_JACOBI5 = 1,
  HDA_K_COPY = 2,
  HDA_K_STENCIL9 = 3,
  HDA_K_STENCIL7_3D = 4,
  HDA_K_SCALE = 5,
  HDA_K_GEMM = 6,
  HDA_K_STAMP = 7
};

/* transports for the exchange step (a5-a7).  Both move exactly the planned
 * rectangles, raw bits; they differ in who moves the bytes. */
enum hda_transport {
  HDA_XPORT_FUSED = 0,   /* one SM kernel on the receiver: peer loads -> local stores
                            (pack + NVLink transfer + unpack fused, no staging) */
  HDA_XPORT_STAGED = 1,  /* pack kernel on the sender into a contiguous staging buffer,
                            copy-engine transfer to the receiver, unpack kernel there */
  HDA_XPORT_AUTO = 2     /* default: messages >= 1 MiB from another GPU are strided
                            copy-engine peer copies (cudaMemcpy3DAsync, no staging, SMs
                            stay free for the overlapped compute); smaller ones FUSED */
};

enum hda_status {
  HDA_OK = 0,
  HDA_EINVAL = -1,       /* bad argument, unknown handle, arity mismatch, footprint not declared */
  HDA_ERANGE = -2,       /* region/box out of bounds; work ⊕ footprint leaves the array */
  HDA_EOVERLAP = -3,     /* manual partition regions overlap */
  HDA_ERACE = -4,        /* two devices' LDEFs intersect in one call */
  HDA_ENOMEM = -5,
  HDA_ECUDA = -6,        /* CUDA error (sticky) */
  HDA_ETIMEOUT = -7,     /* a cross-device wait did not complete (sticky) */
  HDA_EUNSUPPORTED = -8, /* e.g. COL/BLOCK on a 1-D domain, dtype not supported by kernel */
  HDA_ESTATE = -9        /* call not valid in this state (plan-only ctx, SPMD handles missing) */
};

typedef struct hda_ctx hda_ctx_t;
typedef int32_t hda_array_t;
typedef int32_t hda_part_t;

/* One access-list entry.  use/def point to n_use (n_def) offset tuples of ndim
 * int32 each (ndim of the array), tuple-major.  Positional: entry i binds
 * kernel parameter i ("Bind arguments to the kernel call"). */
typedef struct {
  hda_array_t array;
  int32_t n_use;
  const int32_t* use;
  int32_t n_def;
  const int32_t* def;
} hda_access_t;

/* One planned message: the cells [lb, ub) of `array` flow src -> dst. */
typedef struct {
  int32_t array, src, dst, ndim;
  int64_t lb[HDA_MAX_DIM], ub[HDA_MAX_DIM];
} hda_msg_t;

typedef struct {
  int64_t n_apply;          /* hda_apply + coherence-only calls (read) + writes */
  int64_t plan_hits;        /* transitions served by the plan cache */
  int64_t plan_misses;      /* transitions computed with rect algebra */
  int64_t msgs_total;       /* messages moved, cumulative */
  int64_t bytes_total;      /* payload bytes moved, cumulative */
  int64_t last_msgs;        /* messages of the last call */
  int64_t last_bytes;       /* payload bytes of the last call */
  int64_t kernel_launches;  /* CUDA kernels launched by this process, cumulative */
  double tracker_us;        /* host time in compose/plan/commit/cache, cumulative */
  int64_t gated_products;   /* GEMM launches gated on their B rows' arrival (all-gather
                               overlapped with the product), cumulative */
} hda_stats_t;

/* ---- lifetime (Table 2 Init/Exit) ----
 * hda_init: gpu_ids[n_gpus] (NULL => 0..n_gpus-1); n_devices = P >= n_gpus
 * (device d runs on gpu_ids[d % n_gpus]); n_gpus == 0 => plan-only.
 * Enables peer access between all listed GPUs.  EINVAL if P < 1, P > 64.
 * A context is used from one host thread at a time (calls are not re-entrant); with
 * >= 2 GPUs the context itself issues each GPU's launches from an internal per-GPU
 * thread (joined before every call returns; HDA_ISSUE_THREADS=0 disables). */
int hda_init(hda_ctx_t** out, int32_t n_gpus, const int32_t* gpu_ids, int32_t n_devices);
/* hda_init_spmd: this process is device `rank` of n_devices, on CUDA device gpu_id
 * (gpu_id < 0 => plan-only SPMD context: tracker only, used for host-logic tests). */
int hda_init_spmd(hda_ctx_t** out, int32_t n_devices, int32_t rank, int32_t gpu_id);
int hda_finalize(hda_ctx_t* ctx);
/* number of devices P, and whether device d is driven by this process */
int hda_num_devices(const hda_ctx_t* ctx, int32_t* n_devices);
int hda_is_local(const hda_ctx_t* ctx, int32_t dev, int32_t* is_local);

/* ---- SPMD handle swap ----
 * export: writes HDA_HANDLE_BYTES describing this rank's buffer for `arr`
 * (arr == -1: the rank's sync words).  import: `all` holds P blobs in rank order;
 * maps every peer's buffer.  Must be done for the sync words and for every array
 * before the array is used by apply/read/write (HDA_ESTATE otherwise).
 * No-ops returning HDA_OK on non-SPMD or plan-only contexts. */
int hda_spmd_export(hda_ctx_t* ctx, hda_array_t arr, void* out);
int hda_spmd_import(hda_ctx_t* ctx, hda_array_t arr, const void* all);

/* ---- arrays (Table 2 Create) ----
 * Allocates one full-size replica per local device.  init_host (global layout,
 * prod(shape) elements) is copied into every replica; NULL => zero-filled.
 * All sets start empty: owner NONE, every replica valid. */
int hda_create(hda_ctx_t* ctx, int32_t dtype, int32_t ndim, const int64_t* shape,
               const void* init_host, hda_array_t* out);
/* Borrowed replicas: dev_ptrs[P] full-size device buffers (e.g. torch data_ptr),
 * contents taken as identical on every device.  Not available in SPMD mode. */
int hda_create_ext(hda_ctx_t* ctx, int32_t dtype, int32_t ndim, const int64_t* shape,
                   void* const* dev_ptrs, hda_array_t* out);
int hda_free(hda_ctx_t* ctx, hda_array_t arr);
/* device pointer of a local replica (borrowed, valid until hda_free) */
int hda_device_ptr(hda_ctx_t* ctx, hda_array_t arr, int32_t dev, void** out);

/* ---- partitions (Table 2 Partition; Listing 1) ----
 * Even split of [lb,ub) into P disjoint boxes: ROW splits dim 0, COL dim 1,
 * BLOCK a pr x pc grid over dims 0-1 with pr >= pc closest to square (8 -> 4x2),
 * device = ir*pc + ic.  n cells over k parts: the first n%k parts get one extra
 * (reading R4).  Empty boxes are allowed (that device gets no work).
 * ERANGE if [lb,ub) leaves the domain; EUNSUPPORTED for COL/BLOCK on 1-D. */
int hda_partition(hda_ctx_t* ctx, int32_t kind, int32_t ndim, const int64_t* domain,
                  const int64_t* lb, const int64_t* ub, hda_part_t* out);
/* manual: lbs/ubs are P*ndim (device-major). EOVERLAP if two boxes intersect. */
int hda_partition_manual(hda_ctx_t* ctx, int32_t ndim, const int64_t* domain,
                         const int64_t* lbs, const int64_t* ubs, hda_part_t* out);
int hda_partition_region(const hda_ctx_t* ctx, hda_part_t part, int32_t dev,
                         int64_t* lb, int64_t* ub);

/* ---- the hot path (Table 2 ApplyKernel) ----
 * compose LUSE/LDEF -> plan (Eq. 1-2) or plan-cache hit -> exchange (pack,
 * transfer, unpack) -> kernel on every local device -> commit (Eq. 3-4 corrected).
 * scalars: kernel scalars (see enum hda_kernel). Asynchronous w.r.t. the GPUs. */
int hda_apply(hda_ctx_t* ctx, int32_t kernel, hda_part_t part, const hda_access_t* acc,
              int32_t n_acc, const double* scalars, int32_t n_scalars);
/* Absolute sections (Table 1 use@/def@; Table 2 SetAbsoluteUse/Def, P:L171-173,
 * P:L188-191): entry i names, per device q, the exact boxes it uses
 * (n_use[q] boxes) and defines (n_def[q] boxes) in this call, instead of offsets —
 * for non-rectangular or device-specific access (triangular Correlation-style
 * kernels).  Boxes: lb[ndim] then ub[ndim] (half-open), device-major.
 * n_use / n_def may be NULL (none).  Only HDA_K_NONE and HDA_K_STAMP (their device
 * code has no fixed footprint).  ERANGE if a box leaves the array; ERACE as usual. */
typedef struct {
  hda_array_t array;
  const int32_t* n_use; /* [P] */
  const int64_t* use;
  const int32_t* n_def; /* [P] */
  const int64_t* def;
} hda_abs_access_t;
int hda_apply_abs(hda_ctx_t* ctx, int32_t kernel, hda_part_t part, const hda_abs_access_t* acc,
                  int32_t n_acc, const double* scalars, int32_t n_scalars);
/* Trapezoid helper (Table 2 SetTrapezoidUse/Def): corners =
 * {top, ul_col, top, ur_col, bottom, bl_col, bottom, br_col} (inclusive cells); writes
 * one 2-D box {r, left, r+1, right+1} per row with left <= right, edges interpolated
 * linearly and rounded half up (reading R20).  *n_out = number of rows produced
 * (boxes may be NULL to query).  Pass the boxes to hda_apply_abs. */
int hda_trapezoid(const int64_t* corners, int64_t* boxes, int32_t cap, int32_t* n_out);

/* block until every local device has finished all enqueued work */
int hda_sync(hda_ctx_t* ctx);

/* ---- I/O utilities (Table 2 Read/Write) ----
 * write: every local device p copies region_p of host_full (global layout) into its
 * replica; this is a definition by p of region_p (reading R8).
 * read: coherence for LUSE_p = region_p (messages as in Eq. 1-2, no defs), then
 * region_p of device p's replica -> host_full, for every local device; blocks. */
int hda_write(hda_ctx_t* ctx, hda_array_t arr, hda_part_t part, const void* host_full);
int hda_read(hda_ctx_t* ctx, hda_array_t arr, hda_part_t part, void* host_full);

/* Reduce (Table 2 Reduce; "a device reduction is performed
 * followed by an MPI reduction"): coherence for LUSE_p = region_p (exactly as
 * hda_read), then a deterministic two-pass reduction of region_p on every device
 * (fp64 accumulation; int64 for integer dtypes), then the P partials are combined in
 * device order — over NVLink sync words in SPMD mode, so every rank returns the same
 * value.  Regions are disjoint, so every cell counts once.  Blocks.
 * ESTATE on plan-only contexts. */
enum hda_reduce_op { HDA_SUM = 0, HDA_PROD = 1, HDA_MAX = 2, HDA_MIN = 3 };
int hda_reduce(hda_ctx_t* ctx, hda_array_t arr, hda_part_t part, int32_t op, double* out);

/* ---- transport / tuning ---- */
int hda_set_transport(hda_ctx_t* ctx, int32_t transport);
/* overlap on/off (default on): when a device's halo comes from another GPU, its pull
 * runs on a second stream while the kernel computes the part of the work box whose
 * footprint touches no incoming rectangle; the rest runs after the pull lands. */
int hda_set_overlap(hda_ctx_t* ctx, int32_t enabled);
/* plan cache on/off (off => every call recomputes the plan; used to time the
 * baseline of P:L502 and to test cache transparency) */
int hda_set_plan_cache(hda_ctx_t* ctx, int32_t enabled);
/* kernel timing: when enabled, CUDA events bracket every built-in kernel launch on
 * its stream; hda_kernel_time returns the summed ms and launch count since the
 * last reset (blocks to read the events). */
int hda_set_kernel_timing(hda_ctx_t* ctx, int32_t enabled);
int hda_kernel_time(hda_ctx_t* ctx, int32_t kernel, double* total_ms, int64_t* launches);
/* exchange timing (same mechanism, brackets the pull / pack-copy-unpack work) */
int hda_exchange_time(hda_ctx_t* ctx, double* total_ms, int64_t* n);
/* tracing (SURVEY §5 "CUDA events per device per phase"): while enabled, every
 * exchange and kernel launch of every call is bracketed by CUDA events; hda_trace
 * returns rows {call epoch, device, phase, start_us, end_us} (phase 0 exchange,
 * 1 kernel, 2 interior part, 3 dependent part), times relative to enabling; blocks.
 * Events are recorded only on this process's devices and streams. */
int hda_set_trace(hda_ctx_t* ctx, int32_t enabled);
int hda_trace(hda_ctx_t* ctx, double* out, int32_t cap, int32_t* n_out);
/* cudaStream_t of a local device, for callers that record their own events */
int hda_stream(hda_ctx_t* ctx, int32_t dev, void** stream);

/* ---- introspection for parity tests ---- */
/* messages of the last apply/read, canonical order (array, src, dst, lb) */
int hda_last_plan(const hda_ctx_t* ctx, hda_msg_t* out, int32_t cap, int32_t* n_out);
/* last-writer map, prod(shape) int8: -1 = NONE (never written), else device */
int hda_owner_map(const hda_ctx_t* ctx, hda_array_t arr, int8_t* out);
/* full replica of a local device -> host (global layout); blocks */
int hda_read_replica(hda_ctx_t* ctx, hda_array_t arr, int32_t dev, void* host_full);
int hda_stats(const hda_ctx_t* ctx, hda_stats_t* out);
int hda_reset_stats(hda_ctx_t* ctx);
const char* hda_last_error(const hda_ctx_t* ctx);
const char* hda_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HDARRAY_H */
