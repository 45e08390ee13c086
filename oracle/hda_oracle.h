/*
 * hda_oracle.h — CPU oracle for the HDArray def/use exchange path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this.  It shares no code, header,
 * table or constant with the product library (paper_1809_05657_b200/csrc) and
 * never includes include/hdarray.h: the numeric codes below are restated here.
 *
 * Paper: Cho, Kwon, Midkiff, arXiv:1809.05657 (PAPER.md lines "P:Lnnn").
 *
 * The oracle is the plain definition ("HDArray knows where the last written
 * copy of a datum is, and who needs that value"): it simulates P devices in one
 * address space, each with a full-size replica, keeps an explicit
 * per-element last-writer map owner[c] (-1 = never written) and a per-element
 * bitmask valid[c] of devices holding the current value, and derives the message
 * set of every call by brute force over every used cell:
 *     (owner[c] -> q, c)  for c in LUSE_q, owner[c] not in {-1, q}, !valid_q[c]
 * which is what Eq. 1-2 compute with section sets.  Kernels are
 * evaluated naively cell by cell reading only the executing device's replica,
 * through a checked accessor that aborts the call if a read cell is not valid
 * there.  No blocking, fusion or reordering.
 *
 * Floating point: compiled with -O2 -ffp-contract=off -fno-fast-math; the operand
 * order of every kernel is the one written in the comments of hda_oracle.c.
 */
#ifndef HDA_ORACLE_H
#define HDA_ORACLE_H
#include <stdint.h>

#define ORC_STAR INT32_MIN

/* element types */
#define ORC_F64 0
#define ORC_F32 1
#define ORC_BF16 2
#define ORC_I32 3
#define ORC_I64 4
/* partitions */
#define ORC_ROW 0
#define ORC_COL 1
#define ORC_BLOCK 2
/* kernels */
#define ORC_K_NONE 0
#define ORC_K_JACOBI5 1
#define ORC_K_COPY 2
#define ORC_K_STENCIL9 3
#define ORC_K_STENCIL7_3D 4
#define ORC_K_SCALE 5
#define ORC_K_GEMM 6
#define ORC_K_STAMP 7
/* status */
#define ORC_OK 0
#define ORC_EINVAL -1
#define ORC_ERANGE -2
#define ORC_EOVERLAP -3
#define ORC_ERACE -4
#define ORC_ENOMEM -5
#define ORC_EUNSUPPORTED -8
#define ORC_ESTALE -10 /* checked accessor: a kernel read a cell not valid on its device */

typedef struct orc orc_t;

/* P devices (1..64). with_data = 0: plan-only (no replicas, no kernels). */
orc_t* orc_new(int P, int with_data);
void orc_free(orc_t* w);
const char* orc_error(const orc_t* w);

/* returns array id >= 0 or a negative status. init may be NULL (zeros). */
int orc_create(orc_t* w, int dtype, int ndim, const int64_t* shape, const void* init);
/* returns partition id >= 0 or a negative status */
int orc_partition(orc_t* w, int kind, int ndim, const int64_t* domain,
                  const int64_t* lb, const int64_t* ub);
int orc_partition_manual(orc_t* w, int ndim, const int64_t* domain,
                         const int64_t* lbs, const int64_t* ubs);
int orc_region(const orc_t* w, int part, int dev, int64_t* lb, int64_t* ub);

/* arrays[n_acc]; n_use[n_acc]; n_def[n_acc]; uses/defs: all tuples of entry 0,
 * then entry 1, ..., each tuple ndim(array) int32. */
int orc_apply(orc_t* w, int kernel, int part, int n_acc, const int32_t* arrays,
              const int32_t* n_use, const int32_t* uses, const int32_t* n_def,
              const int32_t* defs, const double* scalars, int n_scalars);
/* absolute sections (Table 1 use@/def@, Table 2 SetAbsoluteUse/Def, P:L171-173,
 * P:L188-191): entry e of device q uses/defines exactly the listed boxes
 * (half-open, ndim lb then ndim ub per box), instead of offset compositions.
 * n_use/n_def are [n_acc*P] box counts (entry-major), boxes concatenated in the same
 * order.  Kernels: NONE or STAMP. */
int orc_apply_abs(orc_t* w, int kernel, int part, int n_acc, const int32_t* arrays,
                  const int32_t* n_use, const int64_t* uses, const int32_t* n_def,
                  const int64_t* defs, const double* scalars, int n_scalars);
/* Trapezoid (Table 2 SetTrapezoidUse/Def): inclusive corners
 * (row,col) upper-left, upper-right, below-left, below-right; upper and lower rows
 * equal pairwise.  Row r of [top, bottom] spans columns [left(r), right(r)] with
 * left/right linearly interpolated and rounded half up: left(r) = ul_c +
 * floor(((r-top)*(bl_c-ul_c)*2 + h) / (2h)), h = bottom-top (h = 0: the top row).
 * Writes one box per row (rows with left > right are skipped); returns the count. */
int orc_trapezoid(const int64_t* corners, int64_t* boxes, int cap);
int orc_read(orc_t* w, int arr, int part, void* host);
/* Reduce (Table 2; "a device reduction is performed followed by an
 * MPI reduction"): coherence for LUSE_p = region_p, then every cell of every region,
 * device 0 first, row-major, folded sequentially in fp64 (int64 for integer dtypes,
 * returned as double).  op: 0 SUM, 1 PROD, 2 MAX, 3 MIN. */
#define ORC_SUM 0
#define ORC_PROD 1
#define ORC_MAX 2
#define ORC_MIN 3
int orc_reduce(orc_t* w, int arr, int part, int op, double* out);

/* messages of the last apply/read as (array, src, dst, linear index) quadruples,
 * sorted by (array, src, dst, index). */
int64_t orc_msg_count(const orc_t* w);
int64_t orc_msgs(const orc_t* w, int64_t* out, int64_t cap);

int orc_owner_map(const orc_t* w, int arr, int8_t* out);
int orc_valid_map(const orc_t* w, int arr, uint64_t* out);
int orc_replica(const orc_t* w, int arr, int dev, void* out);

/* standalone sampled GEMM (Listing 2): out[s] = alpha*sum_k A[i][k]B[k][j]
 * + beta*Cin[i][j] in fp64 over bf16 inputs (uint16 bit patterns), for the n
 * sampled (i, j) = (ii[s], jj[s]); Cin may be NULL when beta == 0 (fp64 C-in). */
void orc_gemm_sample(const uint16_t* A, const uint16_t* B, const double* Cin,
                     int64_t ni, int64_t nj, int64_t nk, double alpha, double beta,
                     const int64_t* ii, const int64_t* jj, int64_t n, double* out);

/* helpers exposed for pins */
uint64_t orc_splitmix64(uint64_t x);
uint16_t orc_f32_to_bf16(float f);
uint16_t orc_f64_to_bf16(double d);
#endif
