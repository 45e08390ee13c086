/*
 * hda_oracle.c — plain, slow, obviously-correct CPU oracle of the HDArray
 * def/use exchange path.  TEST INFRASTRUCTURE ONLY (see hda_oracle.h): only
 * tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may load it.
 *
 * Every function cites the passage of PAPER.md ("P:Lnnn") it follows, or the
 * DESIGN.md reading ("R<n>") where the paper is silent.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared (see oracle/build.py).
 */
#include "hda_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXP 64

typedef struct {
  int alive;
  int dtype, ndim;
  int64_t shape[3]; /* trailing unused dims are 1 */
  int64_t n;        /* number of cells */
  size_t es;        /* element size in bytes */
  int8_t* owner;    /* last writer, -1 = never written (sets empty at Create) */
  uint64_t* valid;  /* bit q set <=> device q holds the current value */
  unsigned char* rep[MAXP]; /* full-size replica per device, NULL in plan-only */
} oarr;

typedef struct {
  int ndim;
  int64_t domain[3];
  int64_t lb[MAXP][3], ub[MAXP][3]; /* per device work box, half-open (R1) */
} opart;

struct orc {
  int P, with_data;
  oarr* arrays;
  int n_arrays, cap_arrays;
  opart* parts;
  int n_parts, cap_parts;
  int64_t* msgs; /* quadruples (array, src, dst, linear index) */
  int64_t n_msgs, cap_msgs;
  char err[512];
};

static int fail(orc_t* w, int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(w->err, sizeof w->err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_error(const orc_t* w) { return w->err; }

static size_t elem_size(int dtype) {
  switch (dtype) {
    case ORC_F64: return 8;
    case ORC_F32: return 4;
    case ORC_BF16: return 2;
    case ORC_I32: return 4;
    case ORC_I64: return 8;
  }
  return 0;
}

/* ---------------- small numeric helpers ---------------- */

/* splitmix64 output function (Vigna's reference generator, one step from state x) */
uint64_t orc_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* IEEE round-to-nearest-even float -> bfloat16 */
uint16_t orc_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x40u); /* NaN */
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* IEEE round-to-nearest-even double -> bfloat16, in one rounding */
uint16_t orc_f64_to_bf16(double d) {
  if (isnan(d)) return 0x7FC0;
  uint16_t sign = signbit(d) ? 0x8000 : 0;
  double a = fabs(d);
  if (a < 0x1p-126) { /* bf16 subnormal range: spacing 2^-133 */
    double m = nearbyint(a * 0x1p133); /* exact scaling, RNE to integer */
    return (uint16_t)(sign | (uint16_t)m);
  }
  uint64_t u;
  memcpy(&u, &a, 8);
  /* keep 7 explicit mantissa bits: round at bit 45 of the double mantissa */
  uint64_t lsb = (u >> 45) & 1ULL;
  u += (1ULL << 44) - 1ULL + lsb;
  u &= ~((1ULL << 45) - 1ULL);
  double r;
  memcpy(&r, &u, 8);
  float f = (float)r; /* exact unless >= 2^128, then +inf */
  uint32_t fu;
  memcpy(&fu, &f, 4);
  return (uint16_t)(sign | (uint16_t)(fu >> 16));
}

/* ---------------- world, arrays ---------------- */

orc_t* orc_new(int P, int with_data) {
  if (P < 1 || P > MAXP) return NULL;
  orc_t* w = (orc_t*)calloc(1, sizeof(orc_t));
  if (!w) return NULL;
  w->P = P;
  w->with_data = with_data;
  return w;
}

static void free_array(orc_t* w, oarr* a) {
  free(a->owner);
  free(a->valid);
  for (int d = 0; d < w->P; d++) free(a->rep[d]);
  memset(a, 0, sizeof *a);
}

void orc_free(orc_t* w) {
  if (!w) return;
  for (int i = 0; i < w->n_arrays; i++) free_array(w, &w->arrays[i]);
  free(w->arrays);
  free(w->parts);
  free(w->msgs);
  free(w);
}

/* Table 2 Create: a buffer of the full user-array size on
 * every device; all sets empty => owner NONE, valid everywhere (R9). */
int orc_create(orc_t* w, int dtype, int ndim, const int64_t* shape, const void* init) {
  size_t es = elem_size(dtype);
  if (!es) return fail(w, ORC_EINVAL, "bad dtype %d", dtype);
  if (ndim < 1 || ndim > 3) return fail(w, ORC_EINVAL, "ndim %d", ndim);
  oarr a;
  memset(&a, 0, sizeof a);
  a.alive = 1;
  a.dtype = dtype;
  a.ndim = ndim;
  a.es = es;
  a.n = 1;
  for (int k = 0; k < 3; k++) {
    a.shape[k] = k < ndim ? shape[k] : 1;
    if (a.shape[k] < 1) return fail(w, ORC_EINVAL, "zero extent");
    a.n *= a.shape[k];
  }
  a.owner = (int8_t*)malloc((size_t)a.n);
  a.valid = (uint64_t*)malloc((size_t)a.n * sizeof(uint64_t));
  if (!a.owner || !a.valid) {
    free(a.owner);
    free(a.valid);
    return fail(w, ORC_ENOMEM, "oom");
  }
  uint64_t all = (w->P == 64) ? ~0ULL : ((1ULL << w->P) - 1ULL);
  for (int64_t c = 0; c < a.n; c++) {
    a.owner[c] = -1;
    a.valid[c] = all;
  }
  if (w->with_data) {
    for (int d = 0; d < w->P; d++) {
      a.rep[d] = (unsigned char*)calloc((size_t)a.n, es);
      if (!a.rep[d]) {
        free_array(w, &a);
        return fail(w, ORC_ENOMEM, "oom");
      }
      if (init) memcpy(a.rep[d], init, (size_t)a.n * es);
    }
  }
  if (w->n_arrays == w->cap_arrays) {
    int nc = w->cap_arrays ? 2 * w->cap_arrays : 8;
    oarr* na = (oarr*)realloc(w->arrays, (size_t)nc * sizeof(oarr));
    if (!na) {
      free_array(w, &a);
      return fail(w, ORC_ENOMEM, "oom");
    }
    w->arrays = na;
    w->cap_arrays = nc;
  }
  w->arrays[w->n_arrays] = a;
  return w->n_arrays++;
}

/* ---------------- partitions ---------------- */

/* even split of n items into k parts, part i: the first n%k parts get one more
 * ("evenly partitions"; remainder rule: reading R4) */
static void split(int64_t lo, int64_t n, int k, int i, int64_t* s, int64_t* e) {
  int64_t b = n / k, r = n % k;
  int64_t st = lo + (int64_t)i * b + (i < r ? i : r);
  *s = st;
  *e = st + b + (i < r ? 1 : 0);
}

static int add_part(orc_t* w, const opart* p) {
  if (w->n_parts == w->cap_parts) {
    int nc = w->cap_parts ? 2 * w->cap_parts : 8;
    opart* np = (opart*)realloc(w->parts, (size_t)nc * sizeof(opart));
    if (!np) return fail(w, ORC_ENOMEM, "oom");
    w->parts = np;
    w->cap_parts = nc;
  }
  w->parts[w->n_parts] = *p;
  return w->n_parts++;
}

/* Table 2 Partition: ROW splits dim 0, COL dim 1, BLOCK a
 * near-square pr x pc grid over dims 0-1 (pr >= pc, reading R5). */
int orc_partition(orc_t* w, int kind, int ndim, const int64_t* domain, const int64_t* lb,
                  const int64_t* ub) {
  if (ndim < 1 || ndim > 3) return fail(w, ORC_EINVAL, "ndim");
  if (kind != ORC_ROW && kind != ORC_COL && kind != ORC_BLOCK) return fail(w, ORC_EINVAL, "kind");
  if (kind != ORC_ROW && ndim < 2) return fail(w, ORC_EUNSUPPORTED, "COL/BLOCK on 1-D");
  for (int k = 0; k < ndim; k++) {
    if (domain[k] < 1) return fail(w, ORC_EINVAL, "domain");
    if (lb[k] > ub[k]) return fail(w, ORC_EINVAL, "lb > ub");
    if (lb[k] < 0 || ub[k] > domain[k]) return fail(w, ORC_ERANGE, "region outside domain");
  }
  opart p;
  memset(&p, 0, sizeof p);
  p.ndim = ndim;
  for (int k = 0; k < 3; k++) p.domain[k] = k < ndim ? domain[k] : 1;
  int pr = w->P, pc = 1;
  if (kind == ORC_BLOCK) { /* largest divisor of P not above sqrt(P) */
    for (int c = 1; c * c <= w->P; c++)
      if (w->P % c == 0) pc = c;
    pr = w->P / pc;
  }
  for (int d = 0; d < w->P; d++) {
    for (int k = 0; k < 3; k++) {
      p.lb[d][k] = k < ndim ? lb[k] : 0;
      p.ub[d][k] = k < ndim ? ub[k] : 1;
    }
    if (kind == ORC_ROW) {
      split(lb[0], ub[0] - lb[0], w->P, d, &p.lb[d][0], &p.ub[d][0]);
    } else if (kind == ORC_COL) {
      split(lb[1], ub[1] - lb[1], w->P, d, &p.lb[d][1], &p.ub[d][1]);
    } else {
      int ir = d / pc, ic = d % pc;
      split(lb[0], ub[0] - lb[0], pr, ir, &p.lb[d][0], &p.ub[d][0]);
      split(lb[1], ub[1] - lb[1], pc, ic, &p.lb[d][1], &p.ub[d][1]);
    }
  }
  return add_part(w, &p);
}

/* partition clause with explicit per-device regions (Table 1, Listing 1) */
int orc_partition_manual(orc_t* w, int ndim, const int64_t* domain, const int64_t* lbs,
                         const int64_t* ubs) {
  if (ndim < 1 || ndim > 3) return fail(w, ORC_EINVAL, "ndim");
  opart p;
  memset(&p, 0, sizeof p);
  p.ndim = ndim;
  for (int k = 0; k < 3; k++) {
    p.domain[k] = k < ndim ? domain[k] : 1;
    if (p.domain[k] < 1) return fail(w, ORC_EINVAL, "domain");
  }
  for (int d = 0; d < w->P; d++)
    for (int k = 0; k < 3; k++) {
      p.lb[d][k] = k < ndim ? lbs[d * ndim + k] : 0;
      p.ub[d][k] = k < ndim ? ubs[d * ndim + k] : 1;
      if (p.lb[d][k] > p.ub[d][k]) return fail(w, ORC_EINVAL, "lb > ub");
      if (p.lb[d][k] < 0 || p.ub[d][k] > p.domain[k]) return fail(w, ORC_ERANGE, "outside domain");
    }
  /* pairwise disjointness, checked cell by cell over the domain */
  int64_t n = p.domain[0] * p.domain[1] * p.domain[2];
  int8_t* who = (int8_t*)malloc((size_t)n);
  if (!who) return fail(w, ORC_ENOMEM, "oom");
  memset(who, -1, (size_t)n);
  for (int d = 0; d < w->P; d++)
    for (int64_t i = p.lb[d][0]; i < p.ub[d][0]; i++)
      for (int64_t j = p.lb[d][1]; j < p.ub[d][1]; j++)
        for (int64_t l = p.lb[d][2]; l < p.ub[d][2]; l++) {
          int64_t c = (i * p.domain[1] + j) * p.domain[2] + l;
          if (who[c] >= 0) {
            int other = who[c];
            free(who);
            return fail(w, ORC_EOVERLAP, "devices %d and %d overlap", other, d);
          }
          who[c] = (int8_t)d;
        }
  free(who);
  return add_part(w, &p);
}

int orc_region(const orc_t* w, int part, int dev, int64_t* lb, int64_t* ub) {
  if (part < 0 || part >= w->n_parts || dev < 0 || dev >= w->P) return ORC_EINVAL;
  const opart* p = &w->parts[part];
  for (int k = 0; k < p->ndim; k++) {
    lb[k] = p->lb[dev][k];
    ub[k] = p->ub[dev][k];
  }
  return ORC_OK;
}

static int box_empty(const int64_t* lb, const int64_t* ub) {
  return lb[0] >= ub[0] || lb[1] >= ub[1] || lb[2] >= ub[2];
}

/* ---------------- offset composition ---------------- */

/* P:L185-186 (offset clauses), P:L291 ("LUSE is updated by composing use offset ...
 * with partitioned work item regions"): the cells {w + d : w in W} for one offset
 * tuple d, where '*' stands for every index of that dimension of the array;
 * cells outside the array are dropped (reading R6).  W is a box, so the image of a
 * fixed offset is the shifted box; mark every cell of it in `mask`. */
static void mark_tuple(const oarr* a, const int64_t* wlb, const int64_t* wub,
                       const int32_t* d, unsigned char* mask, unsigned char val) {
  if (box_empty(wlb, wub)) return;
  int64_t lo[3], hi[3];
  for (int k = 0; k < 3; k++) {
    if (k >= a->ndim) {
      lo[k] = 0;
      hi[k] = 1;
    } else if (d[k] == ORC_STAR) {
      lo[k] = 0;
      hi[k] = a->shape[k];
    } else {
      lo[k] = wlb[k] + d[k];
      hi[k] = wub[k] + d[k];
      if (lo[k] < 0) lo[k] = 0;
      if (hi[k] > a->shape[k]) hi[k] = a->shape[k];
    }
    if (lo[k] >= hi[k]) return;
  }
  for (int64_t i = lo[0]; i < hi[0]; i++)
    for (int64_t j = lo[1]; j < hi[1]; j++)
      for (int64_t l = lo[2]; l < hi[2]; l++)
        mask[(i * a->shape[1] + j) * a->shape[2] + l] = val;
}

/* ---------------- messages (Eq. 1-2 as a plain definition) ---------------- */

static int push_msg(orc_t* w, int64_t arr, int64_t src, int64_t dst, int64_t c) {
  if (w->n_msgs == w->cap_msgs) {
    int64_t nc = w->cap_msgs ? 2 * w->cap_msgs : 1024;
    int64_t* nm = (int64_t*)realloc(w->msgs, (size_t)nc * 4 * sizeof(int64_t));
    if (!nm) return fail(w, ORC_ENOMEM, "oom");
    w->msgs = nm;
    w->cap_msgs = nc;
  }
  int64_t* m = &w->msgs[4 * w->n_msgs++];
  m[0] = arr;
  m[1] = src;
  m[2] = dst;
  m[3] = c;
  return ORC_OK;
}

static int cmp_quad(const void* x, const void* y) {
  const int64_t* a = (const int64_t*)x;
  const int64_t* b = (const int64_t*)y;
  for (int k = 0; k < 4; k++) {
    if (a[k] < b[k]) return -1;
    if (a[k] > b[k]) return 1;
  }
  return 0;
}

/* For device q and every cell c it uses (need[c] != 0): if the last writer of c is
 * another device and q does not hold the current value, the value flows from the
 * last writer to q (Eq. 1-2 P:L131-132 with sGDEF_{p,q} = cells p wrote and
 * has not sent to q).  The transfer copies raw bytes and marks q valid
 * (Eq. 3-4's "- SENDMSG/RECVMSG" terms). */
static int exchange_for(orc_t* w, int arr_id, int q, const unsigned char* need) {
  oarr* a = &w->arrays[arr_id];
  for (int64_t c = 0; c < a->n; c++) {
    if (!need[c]) continue;
    int o = a->owner[c];
    if (o < 0 || o == q) continue;
    if ((a->valid[c] >> q) & 1ULL) continue;
    int rc = push_msg(w, arr_id, o, q, c);
    if (rc) return rc;
    if (w->with_data) memcpy(a->rep[q] + (size_t)c * a->es, a->rep[o] + (size_t)c * a->es, a->es);
    a->valid[c] |= 1ULL << q;
  }
  return ORC_OK;
}

/* ---------------- kernels (evaluated naively on one device's replica) ---------------- */

typedef struct {
  orc_t* w;
  int q;
  int bad; /* set by the checked accessor */
} kctx;

static int64_t lin(const oarr* a, int64_t i, int64_t j, int64_t l) {
  return (i * a->shape[1] + j) * a->shape[2] + l;
}

/* checked accessor: a kernel on device q may only read a cell whose
 * current value q holds */
static const unsigned char* rd(kctx* k, const oarr* a, int64_t c) {
  int o = a->owner[c];
  if (!(o < 0 || o == k->q || ((a->valid[c] >> k->q) & 1ULL))) k->bad = 1;
  return a->rep[k->q] + (size_t)c * a->es;
}

static double rdf64(kctx* k, const oarr* a, int64_t c) {
  double v;
  memcpy(&v, rd(k, a, c), 8);
  return v;
}
static float rdf32(kctx* k, const oarr* a, int64_t c) {
  float v;
  memcpy(&v, rd(k, a, c), 4);
  return v;
}
static uint16_t rdbf16(kctx* k, const oarr* a, int64_t c) {
  uint16_t v;
  memcpy(&v, rd(k, a, c), 2);
  return v;
}
static void wrf64(kctx* k, oarr* a, int64_t c, double v) { memcpy(a->rep[k->q] + (size_t)c * 8, &v, 8); }
static void wrf32(kctx* k, oarr* a, int64_t c, float v) { memcpy(a->rep[k->q] + (size_t)c * 4, &v, 4); }
static void wrbf16(kctx* k, oarr* a, int64_t c, uint16_t v) { memcpy(a->rep[k->q] + (size_t)c * 2, &v, 2); }

/* Jacobi: A[i][j] = (B[i][j-1]+B[i][j+1]+B[i-1][j]+B[i+1][j]) / 4, summed left
 * to right as printed; "/4" evaluated as "*0.25" (exact, identical result). */
static void k_jacobi5(kctx* k, oarr* A, const oarr* B, const int64_t* lb, const int64_t* ub) {
  for (int64_t i = lb[0]; i < ub[0]; i++)
    for (int64_t j = lb[1]; j < ub[1]; j++) {
      if (B->dtype == ORC_F64) {
        double s = rdf64(k, B, lin(B, i, j - 1, 0)) + rdf64(k, B, lin(B, i, j + 1, 0));
        s = s + rdf64(k, B, lin(B, i - 1, j, 0));
        s = s + rdf64(k, B, lin(B, i + 1, j, 0));
        wrf64(k, A, lin(A, i, j, 0), s * 0.25);
      } else {
        float s = rdf32(k, B, lin(B, i, j - 1, 0)) + rdf32(k, B, lin(B, i, j + 1, 0));
        s = s + rdf32(k, B, lin(B, i - 1, j, 0));
        s = s + rdf32(k, B, lin(B, i + 1, j, 0));
        wrf32(k, A, lin(A, i, j, 0), s * 0.25f);
      }
    }
}

/* Convolution with eight neighbours; weights: reading R12:
 * e = ((W+E)+N)+S ; c = ((NW+NE)+SW)+SE ; Y = (4*e + c) / 20 */
static void k_stencil9(kctx* k, oarr* Y, const oarr* X, const int64_t* lb, const int64_t* ub) {
  for (int64_t i = lb[0]; i < ub[0]; i++)
    for (int64_t j = lb[1]; j < ub[1]; j++) {
      if (X->dtype == ORC_F64) {
        double e = rdf64(k, X, lin(X, i, j - 1, 0)) + rdf64(k, X, lin(X, i, j + 1, 0));
        e = e + rdf64(k, X, lin(X, i - 1, j, 0));
        e = e + rdf64(k, X, lin(X, i + 1, j, 0));
        double c = rdf64(k, X, lin(X, i - 1, j - 1, 0)) + rdf64(k, X, lin(X, i - 1, j + 1, 0));
        c = c + rdf64(k, X, lin(X, i + 1, j - 1, 0));
        c = c + rdf64(k, X, lin(X, i + 1, j + 1, 0));
        double t = 4.0 * e;
        t = t + c;
        wrf64(k, Y, lin(Y, i, j, 0), t / 20.0);
      } else {
        float e = rdf32(k, X, lin(X, i, j - 1, 0)) + rdf32(k, X, lin(X, i, j + 1, 0));
        e = e + rdf32(k, X, lin(X, i - 1, j, 0));
        e = e + rdf32(k, X, lin(X, i + 1, j, 0));
        float c = rdf32(k, X, lin(X, i - 1, j - 1, 0)) + rdf32(k, X, lin(X, i - 1, j + 1, 0));
        c = c + rdf32(k, X, lin(X, i + 1, j - 1, 0));
        c = c + rdf32(k, X, lin(X, i + 1, j + 1, 0));
        float t = 4.0f * e;
        t = t + c;
        wrf32(k, Y, lin(Y, i, j, 0), t / 20.0f);
      }
    }
}

/* 3-D analogue of the paper's Jacobi (reading R13): dims (z, y, x), x contiguous;
 * s = ((((x- + x+) + y-) + y+) + z-) + z+ ; Y = s / 6 */
static void k_stencil7(kctx* k, oarr* Y, const oarr* X, const int64_t* lb, const int64_t* ub) {
  for (int64_t z = lb[0]; z < ub[0]; z++)
    for (int64_t y = lb[1]; y < ub[1]; y++)
      for (int64_t x = lb[2]; x < ub[2]; x++) {
        if (X->dtype == ORC_F32) {
          float s = rdf32(k, X, lin(X, z, y, x - 1)) + rdf32(k, X, lin(X, z, y, x + 1));
          s = s + rdf32(k, X, lin(X, z, y - 1, x));
          s = s + rdf32(k, X, lin(X, z, y + 1, x));
          s = s + rdf32(k, X, lin(X, z - 1, y, x));
          s = s + rdf32(k, X, lin(X, z + 1, y, x));
          wrf32(k, Y, lin(Y, z, y, x), s / 6.0f);
        } else {
          double s = rdf64(k, X, lin(X, z, y, x - 1)) + rdf64(k, X, lin(X, z, y, x + 1));
          s = s + rdf64(k, X, lin(X, z, y - 1, x));
          s = s + rdf64(k, X, lin(X, z, y + 1, x));
          s = s + rdf64(k, X, lin(X, z - 1, y, x));
          s = s + rdf64(k, X, lin(X, z + 1, y, x));
          wrf64(k, Y, lin(Y, z, y, x), s / 6.0);
        }
      }
}

/* copy kernel of the Jacobi benchmark, "B[i][j]=A[i][j]": raw bytes */
static void k_copy(kctx* k, oarr* B, const oarr* A, const int64_t* lb, const int64_t* ub) {
  for (int64_t i = lb[0]; i < ub[0]; i++)
    for (int64_t j = lb[1]; j < ub[1]; j++)
      for (int64_t l = lb[2]; l < ub[2]; l++) {
        int64_t c = lin(A, i, j, l);
        memcpy(B->rep[k->q] + (size_t)c * B->es, rd(k, A, c), A->es);
      }
}

/* elementwise X = alpha * X in X's own arithmetic (repartition kernels, reading R16) */
static void k_scale(kctx* k, oarr* X, double alpha, const int64_t* lb, const int64_t* ub) {
  for (int64_t i = lb[0]; i < ub[0]; i++)
    for (int64_t j = lb[1]; j < ub[1]; j++)
      for (int64_t l = lb[2]; l < ub[2]; l++) {
        int64_t c = lin(X, i, j, l);
        if (X->dtype == ORC_F64) {
          wrf64(k, X, c, alpha * rdf64(k, X, c));
        } else if (X->dtype == ORC_F32) {
          wrf32(k, X, c, (float)alpha * rdf32(k, X, c));
        } else {
          float p = (float)alpha * bf16_to_f32(rdbf16(k, X, c));
          wrbf16(k, X, c, orc_f32_to_bf16(p));
        }
      }
}

/* GEMM, Listing 2: C[i][j] = beta*C[i][j] + alph * sum_k A[i][k]*B[k][j];
 * the sum is taken in fp64 (exact products of bf16 values, k ascending); C is read
 * only when beta != 0 (reading R15); the result is rounded once to C's dtype. */
static void k_gemm(kctx* k, oarr* C, const oarr* A, const oarr* B, double alpha, double beta,
                   const int64_t* lb, const int64_t* ub) {
  int64_t nk = A->shape[1];
  for (int64_t i = lb[0]; i < ub[0]; i++)
    for (int64_t j = lb[1]; j < ub[1]; j++) {
      double acc = 0.0;
      for (int64_t kk = 0; kk < nk; kk++) {
        double a = (double)bf16_to_f32(rdbf16(k, A, lin(A, i, kk, 0)));
        double b = (double)bf16_to_f32(rdbf16(k, B, lin(B, kk, j, 0)));
        acc = acc + a * b;
      }
      double r = alpha * acc;
      int64_t c = lin(C, i, j, 0);
      if (beta != 0.0) {
        double cin = C->dtype == ORC_F32 ? (double)rdf32(k, C, c) : (double)bf16_to_f32(rdbf16(k, C, c));
        r = r + beta * cin;
      }
      if (C->dtype == ORC_F32)
        wrf32(k, C, c, (float)r);
      else
        wrbf16(k, C, c, orc_f64_to_bf16(r));
    }
}

void orc_gemm_sample(const uint16_t* A, const uint16_t* B, const double* Cin, int64_t ni,
                     int64_t nj, int64_t nk, double alpha, double beta, const int64_t* ii,
                     const int64_t* jj, int64_t n, double* out) {
  (void)ni;
  for (int64_t s = 0; s < n; s++) {
    int64_t i = ii[s], j = jj[s];
    double acc = 0.0;
    for (int64_t kk = 0; kk < nk; kk++) {
      double a = (double)bf16_to_f32(A[i * nk + kk]);
      double b = (double)bf16_to_f32(B[kk * nj + j]);
      acc = acc + a * b;
    }
    double r = alpha * acc;
    if (beta != 0.0 && Cin) r = r + beta * Cin[i * nj + j];
    out[s] = r;
  }
}

/* test kernel: distinctive raw bits on every composed def cell (header, HDA_K_STAMP) */
static void k_stamp(kctx* k, oarr* X, uint64_t seed, const unsigned char* defmask) {
  for (int64_t c = 0; c < X->n; c++) {
    if (!defmask[c]) continue;
    uint64_t h = orc_splitmix64(seed * 0x9E3779B97F4A7C15ULL + (uint64_t)c);
    memcpy(X->rep[k->q] + (size_t)c * X->es, &h, X->es); /* little-endian low bytes */
  }
}

/* ---------------- apply (Table 2 ApplyKernel) ---------------- */

static int is_zero_tuple(const int32_t* d, int ndim) {
  for (int k = 0; k < ndim; k++)
    if (d[k] != 0) return 0;
  return 1;
}

/* declared tuple d covers required tuple r: per dim equal, or d is '*' */
static int covers(const int32_t* d, const int32_t* r, int ndim) {
  for (int k = 0; k < ndim; k++)
    if (!(d[k] == ORC_STAR || d[k] == r[k])) return 0;
  return 1;
}

static int declared(const int32_t* tuples, int n, const int32_t* r, int ndim) {
  for (int t = 0; t < n; t++)
    if (covers(tuples + t * ndim, r, ndim)) return 1;
  return 0;
}

static int nparams(int kernel) {
  switch (kernel) {
    case ORC_K_JACOBI5:
    case ORC_K_COPY:
    case ORC_K_STENCIL9:
    case ORC_K_STENCIL7_3D: return 2;
    case ORC_K_SCALE: return 1;
    case ORC_K_GEMM: return 3;
    case ORC_K_STAMP: /* [X, used...] */
    case ORC_K_NONE: return -1; /* any */
  }
  return -2;
}

int orc_apply(orc_t* w, int kernel, int part, int n_acc, const int32_t* arrays,
              const int32_t* n_use, const int32_t* uses, const int32_t* n_def,
              const int32_t* defs, const double* scalars, int n_scalars) {
  w->n_msgs = 0;
  int np = nparams(kernel);
  if (np == -2) return fail(w, ORC_EINVAL, "unknown kernel %d", kernel);
  if (np >= 0 && n_acc != np) return fail(w, ORC_EINVAL, "kernel takes %d params, got %d", np, n_acc);
  if (part < 0 || part >= w->n_parts) return fail(w, ORC_EINVAL, "unknown partition");
  const opart* pt = &w->parts[part];
  if (n_acc < 0 || n_acc > 16) return fail(w, ORC_EINVAL, "n_acc");

  /* locate each entry's tuples */
  const int32_t* ut[16];
  const int32_t* dt[16];
  oarr* A[16];
  {
    int64_t uo = 0, dof = 0;
    for (int e = 0; e < n_acc; e++) {
      if (arrays[e] < 0 || arrays[e] >= w->n_arrays || !w->arrays[arrays[e]].alive)
        return fail(w, ORC_EINVAL, "unknown array");
      A[e] = &w->arrays[arrays[e]];
      if (A[e]->ndim != pt->ndim) return fail(w, ORC_EINVAL, "array ndim != partition ndim");
      if (n_use[e] < 0 || n_def[e] < 0) return fail(w, ORC_EINVAL, "negative count");
      ut[e] = uses + uo;
      dt[e] = defs + dof;
      uo += (int64_t)n_use[e] * A[e]->ndim;
      dof += (int64_t)n_def[e] * A[e]->ndim;
    }
  }
  int nd = pt->ndim;
  int32_t zero[3] = {0, 0, 0};

  /* kernel-specific validation: footprint declared, defs exact, dtypes, bounds */
  if (kernel != ORC_K_NONE && kernel != ORC_K_STAMP) {
    /* parameter 0 is the defined one for all built-ins; it must be def (0,..,0) */
    if (!(n_def[0] == 1 && is_zero_tuple(dt[0], nd)))
      return fail(w, ORC_EINVAL, "built-in kernel needs exactly def (0,..,0) on param 0");
    for (int e = 1; e < n_acc; e++)
      if (n_def[e] != 0) return fail(w, ORC_EINVAL, "only param 0 may be defined");
  }
  if (kernel == ORC_K_STAMP) {
    if (n_acc < 1 || n_scalars < 1) return fail(w, ORC_EINVAL, "STAMP needs [X, ...] and a seed");
    for (int e = 1; e < n_acc; e++)
      if (n_def[e] != 0) return fail(w, ORC_EINVAL, "STAMP defines only param 0");
  }
  if (kernel == ORC_K_SCALE && n_scalars < 1) return fail(w, ORC_EINVAL, "SCALE needs alpha");
  if (kernel == ORC_K_GEMM && n_scalars < 2) return fail(w, ORC_EINVAL, "GEMM needs alpha, beta");
  int64_t fp[8][3];
  int nfp = 0;
  int64_t halo = 0;
  if (kernel == ORC_K_JACOBI5 || kernel == ORC_K_STENCIL9 || kernel == ORC_K_STENCIL7_3D) {
    oarr *dst = A[0], *src = A[1];
    if (kernel == ORC_K_STENCIL7_3D ? nd != 3 : nd != 2) return fail(w, ORC_EINVAL, "stencil ndim");
    if (dst->dtype != src->dtype) return fail(w, ORC_EINVAL, "dtype mismatch");
    if (src->dtype != ORC_F64 && src->dtype != ORC_F32) return fail(w, ORC_EUNSUPPORTED, "stencil dtype");
    for (int k = 0; k < 3; k++)
      if (dst->shape[k] != src->shape[k]) return fail(w, ORC_EINVAL, "shape mismatch");
    if (kernel == ORC_K_JACOBI5) {
      int64_t f[4][3] = {{0, -1, 0}, {0, 1, 0}, {-1, 0, 0}, {1, 0, 0}};
      memcpy(fp, f, sizeof f);
      nfp = 4;
    } else if (kernel == ORC_K_STENCIL9) {
      for (int a = -1; a <= 1; a++)
        for (int b = -1; b <= 1; b++)
          if (a || b) {
            fp[nfp][0] = a;
            fp[nfp][1] = b;
            fp[nfp][2] = 0;
            nfp++;
          }
    } else {
      int64_t f[6][3] = {{0, 0, -1}, {0, 0, 1}, {0, -1, 0}, {0, 1, 0}, {-1, 0, 0}, {1, 0, 0}};
      memcpy(fp, f, sizeof f);
      nfp = 6;
    }
    halo = 1;
    for (int f = 0; f < nfp; f++) {
      int32_t r[3] = {(int32_t)fp[f][0], (int32_t)fp[f][1], (int32_t)fp[f][2]};
      if (!declared(ut[1], n_use[1], r, nd)) return fail(w, ORC_EINVAL, "footprint offset not declared");
    }
  } else if (kernel == ORC_K_COPY) {
    if (A[0]->dtype != A[1]->dtype) return fail(w, ORC_EINVAL, "dtype mismatch");
    for (int k = 0; k < 3; k++)
      if (A[0]->shape[k] != A[1]->shape[k]) return fail(w, ORC_EINVAL, "shape mismatch");
    if (!declared(ut[1], n_use[1], zero, nd)) return fail(w, ORC_EINVAL, "use (0,..) not declared");
  } else if (kernel == ORC_K_SCALE) {
    if (A[0]->dtype != ORC_F64 && A[0]->dtype != ORC_F32 && A[0]->dtype != ORC_BF16)
      return fail(w, ORC_EUNSUPPORTED, "SCALE dtype");
    if (!declared(ut[0], n_use[0], zero, nd)) return fail(w, ORC_EINVAL, "use (0,..) not declared");
  } else if (kernel == ORC_K_GEMM) {
    oarr *C = A[0], *Aa = A[1], *B = A[2];
    if (nd != 2) return fail(w, ORC_EINVAL, "GEMM is 2-D");
    if (Aa->dtype != ORC_BF16 || B->dtype != ORC_BF16) return fail(w, ORC_EUNSUPPORTED, "A,B bf16");
    if (C->dtype != ORC_F32 && C->dtype != ORC_BF16) return fail(w, ORC_EUNSUPPORTED, "C f32/bf16");
    if (Aa->shape[0] != C->shape[0] || B->shape[1] != C->shape[1] || Aa->shape[1] != B->shape[0])
      return fail(w, ORC_EINVAL, "GEMM shapes");
    int32_t ra[2] = {0, ORC_STAR}, rb[2] = {ORC_STAR, 0};
    if (!declared(ut[1], n_use[1], ra, 2)) return fail(w, ORC_EINVAL, "use A (0,*) not declared");
    if (!declared(ut[2], n_use[2], rb, 2)) return fail(w, ORC_EINVAL, "use B (*,0) not declared");
    if (scalars[1] != 0.0 && !declared(ut[0], n_use[0], zero, 2))
      return fail(w, ORC_EINVAL, "use C (0,0) not declared with beta != 0");
    if (arrays[0] == arrays[1] || arrays[0] == arrays[2]) return fail(w, ORC_EINVAL, "C aliases A/B");
  }
  /* bounds: work (+ footprint halo) inside the defined / read arrays */
  if (kernel != ORC_K_NONE && kernel != ORC_K_STAMP) {
    for (int d = 0; d < w->P; d++) {
      if (box_empty(pt->lb[d], pt->ub[d])) continue;
      for (int k = 0; k < nd; k++) {
        if (pt->lb[d][k] - halo < 0 || pt->ub[d][k] + halo > A[0]->shape[k])
          return fail(w, ORC_ERANGE, "work + footprint outside the array");
      }
    }
  }
  /* an array used at a non-zero offset and defined in the same call (R15) */
  for (int e = 0; e < n_acc; e++)
    for (int f = 0; f < n_acc; f++) {
      if (arrays[e] != arrays[f] || n_def[f] == 0) continue;
      for (int t = 0; t < n_use[e]; t++)
        if (!is_zero_tuple(ut[e] + t * nd, nd))
          return fail(w, ORC_EINVAL, "array used at a non-zero offset and defined in one call");
    }
  /* ERACE: two devices define the same cell */
  unsigned char** defmask = (unsigned char**)calloc((size_t)n_acc, sizeof(unsigned char*));
  for (int e = 0; e < n_acc; e++) {
    if (n_def[e] == 0) continue;
    int64_t n = A[e]->n;
    int8_t* definer = (int8_t*)malloc((size_t)n);
    unsigned char* m = (unsigned char*)malloc((size_t)n);
    memset(definer, -1, (size_t)n);
    for (int d = 0; d < w->P; d++) {
      memset(m, 0, (size_t)n);
      for (int t = 0; t < n_def[e]; t++) mark_tuple(A[e], pt->lb[d], pt->ub[d], dt[e] + t * nd, m, 1);
      for (int64_t c = 0; c < n; c++) {
        if (!m[c]) continue;
        if (definer[c] >= 0 && definer[c] != d) {
          int other = definer[c];
          free(definer);
          free(m);
          for (int x = 0; x < n_acc; x++) free(defmask[x]);
          free(defmask);
          return fail(w, ORC_ERACE, "devices %d and %d define the same cell", other, d);
        }
        definer[c] = (int8_t)d;
      }
    }
    free(m);
    /* keep the definer map: defmask[e][c] = 1 + defining device */
    defmask[e] = (unsigned char*)definer;
  }

  int rc = ORC_OK;
  /* messages + exchange: per distinct used array, per device q, every cell of
   * LUSE_q = union over all entries naming this array of the composed use tuples */
  for (int e = 0; e < n_acc && rc == ORC_OK; e++) {
    int first = 1;
    for (int f = 0; f < e; f++)
      if (arrays[f] == arrays[e]) first = 0;
    if (!first) continue;
    oarr* a = A[e];
    unsigned char* need = (unsigned char*)malloc((size_t)a->n);
    for (int q = 0; q < w->P && rc == ORC_OK; q++) {
      memset(need, 0, (size_t)a->n);
      int any = 0;
      for (int f = e; f < n_acc; f++) {
        if (arrays[f] != arrays[e]) continue;
        for (int t = 0; t < n_use[f]; t++) {
          mark_tuple(a, pt->lb[q], pt->ub[q], ut[f] + t * nd, need, 1);
          any = 1;
        }
      }
      if (any) rc = exchange_for(w, arrays[e], q, need);
    }
    free(need);
  }

  /* kernel on every device, reading only that device's replica */
  if (rc == ORC_OK && w->with_data && kernel != ORC_K_NONE) {
    for (int q = 0; q < w->P && rc == ORC_OK; q++) {
      kctx k = {w, q, 0};
      const int64_t* lb = pt->lb[q];
      const int64_t* ub = pt->ub[q];
      if (kernel == ORC_K_STAMP) {
        unsigned char* m = (unsigned char*)calloc((size_t)A[0]->n, 1);
        const int8_t* definer = (const int8_t*)defmask[0];
        for (int64_t c = 0; c < A[0]->n; c++) m[c] = definer && definer[c] == q;
        k_stamp(&k, A[0], (uint64_t)scalars[0], m);
        free(m);
        continue;
      }
      if (box_empty(lb, ub)) continue;
      switch (kernel) {
        case ORC_K_JACOBI5: k_jacobi5(&k, A[0], A[1], lb, ub); break;
        case ORC_K_STENCIL9: k_stencil9(&k, A[0], A[1], lb, ub); break;
        case ORC_K_STENCIL7_3D: k_stencil7(&k, A[0], A[1], lb, ub); break;
        case ORC_K_COPY: k_copy(&k, A[0], A[1], lb, ub); break;
        case ORC_K_SCALE: k_scale(&k, A[0], scalars[0], lb, ub); break;
        case ORC_K_GEMM: k_gemm(&k, A[0], A[1], A[2], scalars[0], scalars[1], lb, ub); break;
      }
      if (k.bad) rc = fail(w, ORC_ESTALE, "device %d read a cell it does not hold", q);
    }
  }

  /* commit (Eq. 3-4 with last-writer semantics, reading R7): every defined cell is
   * now owned by its definer and valid only there */
  if (rc == ORC_OK) {
    for (int e = 0; e < n_acc; e++) {
      if (!defmask[e]) continue;
      const int8_t* definer = (const int8_t*)defmask[e];
      oarr* a = A[e];
      for (int64_t c = 0; c < a->n; c++)
        if (definer[c] >= 0) {
          a->owner[c] = definer[c];
          a->valid[c] = 1ULL << definer[c];
        }
    }
  }
  for (int e = 0; e < n_acc; e++) free(defmask[e]);
  free(defmask);
  if (w->n_msgs > 1) qsort(w->msgs, (size_t)w->n_msgs, 4 * sizeof(int64_t), cmp_quad);
  return rc;
}

/* ---------------- absolute sections + trapezoids ---------------- */

static int64_t floordiv(int64_t a, int64_t b) { /* b > 0 */
  int64_t q = a / b;
  if ((a % b) != 0 && a < 0) q--;
  return q;
}

int orc_trapezoid(const int64_t* k, int64_t* boxes, int cap) {
  const int64_t top = k[0], ul = k[1], ur = k[3], bottom = k[4], bl = k[5], br = k[7];
  const int64_t h = bottom - top;
  int n = 0;
  for (int64_t r = top; r <= bottom; r++) {
    int64_t left = ul, right = ur;
    if (h > 0) {
      left = ul + floordiv((r - top) * (bl - ul) * 2 + h, 2 * h);
      right = ur + floordiv((r - top) * (br - ur) * 2 + h, 2 * h);
    }
    if (left > right) continue;
    if (n < cap) {
      boxes[4 * n + 0] = r;
      boxes[4 * n + 1] = left;
      boxes[4 * n + 2] = r + 1;
      boxes[4 * n + 3] = right + 1;
    }
    n++;
  }
  return n;
}

/* mark the cells of explicit boxes (clipped rejected: out of bounds is ERANGE) */
static int mark_boxes(orc_t* w, const oarr* a, const int64_t* bx, int nb, unsigned char* mask) {
  int nd = a->ndim;
  for (int b = 0; b < nb; b++) {
    int64_t lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
    for (int k = 0; k < nd; k++) {
      lo[k] = bx[b * 2 * nd + k];
      hi[k] = bx[b * 2 * nd + nd + k];
      if (lo[k] < 0 || hi[k] > a->shape[k] || lo[k] > hi[k]) return fail(w, ORC_ERANGE, "absolute box outside");
    }
    for (int64_t i = lo[0]; i < hi[0]; i++)
      for (int64_t j = lo[1]; j < hi[1]; j++)
        for (int64_t l = lo[2]; l < hi[2]; l++) mask[lin(a, i, j, l)] = 1;
  }
  return ORC_OK;
}

int orc_apply_abs(orc_t* w, int kernel, int part, int n_acc, const int32_t* arrays, const int32_t* n_use,
                  const int64_t* uses, const int32_t* n_def, const int64_t* defs, const double* scalars,
                  int n_scalars) {
  w->n_msgs = 0;
  if (kernel != ORC_K_NONE && kernel != ORC_K_STAMP) return fail(w, ORC_EINVAL, "absolute sections: NONE/STAMP");
  if (part < 0 || part >= w->n_parts) return fail(w, ORC_EINVAL, "partition");
  if (n_acc < 1 || n_acc > 16) return fail(w, ORC_EINVAL, "n_acc");
  if (kernel == ORC_K_STAMP && n_scalars < 1) return fail(w, ORC_EINVAL, "STAMP needs seed");
  const int P = w->P;
  oarr* A[16];
  const int64_t* ub_[16][MAXP];
  const int64_t* db_[16][MAXP];
  {
    int64_t uo = 0, dof = 0;
    for (int e = 0; e < n_acc; e++) {
      if (arrays[e] < 0 || arrays[e] >= w->n_arrays || !w->arrays[arrays[e]].alive)
        return fail(w, ORC_EINVAL, "unknown array");
      A[e] = &w->arrays[arrays[e]];
      if (kernel == ORC_K_STAMP && e > 0)
        for (int q = 0; q < P; q++)
          if (n_def[e * P + q]) return fail(w, ORC_EINVAL, "STAMP defines only param 0");
      for (int q = 0; q < P; q++) {
        ub_[e][q] = uses + uo;
        db_[e][q] = defs + dof;
        uo += (int64_t)n_use[e * P + q] * 2 * A[e]->ndim;
        dof += (int64_t)n_def[e * P + q] * 2 * A[e]->ndim;
      }
    }
  }
  /* definer maps + race check */
  int8_t* definer[16] = {0};
  int rc = ORC_OK;
  unsigned char* m = NULL;
  for (int e = 0; e < n_acc && rc == ORC_OK; e++) {
    int any = 0;
    for (int q = 0; q < P; q++) any |= n_def[e * P + q] > 0;
    if (!any) continue;
    definer[e] = (int8_t*)malloc((size_t)A[e]->n);
    memset(definer[e], -1, (size_t)A[e]->n);
    m = (unsigned char*)realloc(m, (size_t)A[e]->n);
    for (int q = 0; q < P && rc == ORC_OK; q++) {
      memset(m, 0, (size_t)A[e]->n);
      rc = mark_boxes(w, A[e], db_[e][q], n_def[e * P + q], m);
      for (int64_t c = 0; c < A[e]->n && rc == ORC_OK; c++) {
        if (!m[c]) continue;
        if (definer[e][c] >= 0 && definer[e][c] != q)
          rc = fail(w, ORC_ERACE, "devices %d and %d define the same cell", definer[e][c], q);
        definer[e][c] = (int8_t)q;
      }
    }
  }
  /* validate use boxes before any state change */
  for (int e = 0; e < n_acc && rc == ORC_OK; e++) {
    unsigned char* u = (unsigned char*)calloc((size_t)A[e]->n, 1);
    for (int q = 0; q < P && rc == ORC_OK; q++) rc = mark_boxes(w, A[e], ub_[e][q], n_use[e * P + q], u);
    free(u);
  }
  /* messages + exchange (as in orc_apply) */
  for (int e = 0; e < n_acc && rc == ORC_OK; e++) {
    int first = 1;
    for (int f = 0; f < e; f++)
      if (arrays[f] == arrays[e]) first = 0;
    if (!first) continue;
    unsigned char* need = (unsigned char*)malloc((size_t)A[e]->n);
    for (int q = 0; q < P && rc == ORC_OK; q++) {
      memset(need, 0, (size_t)A[e]->n);
      for (int f = e; f < n_acc; f++)
        if (arrays[f] == arrays[e]) mark_boxes(w, A[e], ub_[f][q], n_use[f * P + q], need);
      rc = exchange_for(w, arrays[e], q, need);
    }
    free(need);
  }
  if (rc == ORC_OK && w->with_data && kernel == ORC_K_STAMP && definer[0]) {
    for (int q = 0; q < P; q++) {
      kctx k = {w, q, 0};
      unsigned char* dm = (unsigned char*)calloc((size_t)A[0]->n, 1);
      for (int64_t c = 0; c < A[0]->n; c++) dm[c] = definer[0][c] == q;
      k_stamp(&k, A[0], (uint64_t)scalars[0], dm);
      free(dm);
    }
  }
  if (rc == ORC_OK)
    for (int e = 0; e < n_acc; e++) {
      if (!definer[e]) continue;
      for (int64_t c = 0; c < A[e]->n; c++)
        if (definer[e][c] >= 0) {
          A[e]->owner[c] = definer[e][c];
          A[e]->valid[c] = 1ULL << definer[e][c];
        }
    }
  for (int e = 0; e < n_acc; e++) free(definer[e]);
  free(m);
  if (w->n_msgs > 1) qsort(w->msgs, (size_t)w->n_msgs, 4 * sizeof(int64_t), cmp_quad);
  return rc;
}

/* ---------------- Write / Read (Table 2) ---------------- */

/* Write: device p copies region_p from the user array; a definition by p (R8) */
int orc_write(orc_t* w, int arr, int part, const void* host) {
  w->n_msgs = 0;
  if (arr < 0 || arr >= w->n_arrays || !w->arrays[arr].alive) return fail(w, ORC_EINVAL, "array");
  if (part < 0 || part >= w->n_parts) return fail(w, ORC_EINVAL, "partition");
  oarr* a = &w->arrays[arr];
  const opart* pt = &w->parts[part];
  if (pt->ndim != a->ndim) return fail(w, ORC_EINVAL, "ndim");
  if (w->with_data && !host) return fail(w, ORC_EINVAL, "no host data");
  for (int d = 0; d < w->P; d++)
    for (int k = 0; k < a->ndim; k++)
      if (!box_empty(pt->lb[d], pt->ub[d]) && pt->ub[d][k] > a->shape[k])
        return fail(w, ORC_ERANGE, "region outside array");
  for (int d = 0; d < w->P; d++) {
    if (box_empty(pt->lb[d], pt->ub[d])) continue;
    for (int64_t i = pt->lb[d][0]; i < pt->ub[d][0]; i++)
      for (int64_t j = pt->lb[d][1]; j < pt->ub[d][1]; j++)
        for (int64_t l = pt->lb[d][2]; l < pt->ub[d][2]; l++) {
          int64_t c = lin(a, i, j, l);
          if (w->with_data)
            memcpy(a->rep[d] + (size_t)c * a->es, (const unsigned char*)host + (size_t)c * a->es, a->es);
          a->owner[c] = (int8_t)d;
          a->valid[c] = 1ULL << d;
        }
  }
  return ORC_OK;
}

/* Read: coherence for LUSE_p = region_p (Eq. 1-2, no definitions), then region_p of
 * device p's replica into the user array (R10) */
int orc_read(orc_t* w, int arr, int part, void* host) {
  w->n_msgs = 0;
  if (arr < 0 || arr >= w->n_arrays || !w->arrays[arr].alive) return fail(w, ORC_EINVAL, "array");
  if (part < 0 || part >= w->n_parts) return fail(w, ORC_EINVAL, "partition");
  oarr* a = &w->arrays[arr];
  const opart* pt = &w->parts[part];
  if (pt->ndim != a->ndim) return fail(w, ORC_EINVAL, "ndim");
  for (int d = 0; d < w->P; d++)
    for (int k = 0; k < a->ndim; k++)
      if (!box_empty(pt->lb[d], pt->ub[d]) && pt->ub[d][k] > a->shape[k])
        return fail(w, ORC_ERANGE, "region outside array");
  unsigned char* need = (unsigned char*)malloc((size_t)a->n);
  int32_t zero[3] = {0, 0, 0};
  int rc = ORC_OK;
  for (int q = 0; q < w->P && rc == ORC_OK; q++) {
    memset(need, 0, (size_t)a->n);
    mark_tuple(a, pt->lb[q], pt->ub[q], zero, need, 1);
    rc = exchange_for(w, arr, q, need);
    if (rc == ORC_OK && w->with_data && host)
      for (int64_t c = 0; c < a->n; c++)
        if (need[c])
          memcpy((unsigned char*)host + (size_t)c * a->es, a->rep[q] + (size_t)c * a->es, a->es);
  }
  free(need);
  if (w->n_msgs > 1) qsort(w->msgs, (size_t)w->n_msgs, 4 * sizeof(int64_t), cmp_quad);
  return rc;
}

/* ---------------- Reduce (Table 2) ---------------- */

static double cell_value(const oarr* a, int dev, int64_t c) {
  const unsigned char* p = a->rep[dev] + (size_t)c * a->es;
  switch (a->dtype) {
    case ORC_F64: {
      double v;
      memcpy(&v, p, 8);
      return v;
    }
    case ORC_F32: {
      float v;
      memcpy(&v, p, 4);
      return (double)v;
    }
    case ORC_BF16: {
      uint16_t v;
      memcpy(&v, p, 2);
      return (double)bf16_to_f32(v);
    }
    case ORC_I32: {
      int32_t v;
      memcpy(&v, p, 4);
      return (double)v;
    }
    default: {
      int64_t v;
      memcpy(&v, p, 8);
      return (double)v;
    }
  }
}

int orc_reduce(orc_t* w, int arr, int part, int op, double* out) {
  if (op < 0 || op > 3) return fail(w, ORC_EINVAL, "op");
  if (!w->with_data) return fail(w, ORC_EINVAL, "reduce needs data");
  int rc = orc_read(w, arr, part, NULL); /* coherence, exactly as a read */
  if (rc) return rc;
  const oarr* a = &w->arrays[arr];
  const opart* pt = &w->parts[part];
  int is_int = a->dtype == ORC_I32 || a->dtype == ORC_I64;
  double acc = op == ORC_SUM ? 0.0 : op == ORC_PROD ? 1.0 : op == ORC_MAX ? -INFINITY : INFINITY;
  int64_t iacc = op == ORC_PROD ? 1 : 0;
  int first = 1;
  for (int d = 0; d < w->P; d++) {
    if (box_empty(pt->lb[d], pt->ub[d])) continue;
    for (int64_t i = pt->lb[d][0]; i < pt->ub[d][0]; i++)
      for (int64_t j = pt->lb[d][1]; j < pt->ub[d][1]; j++)
        for (int64_t l = pt->lb[d][2]; l < pt->ub[d][2]; l++) {
          int64_t c = lin(a, i, j, l);
          if (is_int) {
            int64_t v;
            if (a->dtype == ORC_I32) {
              int32_t t;
              memcpy(&t, a->rep[d] + (size_t)c * 4, 4);
              v = t;
            } else {
              memcpy(&v, a->rep[d] + (size_t)c * 8, 8);
            }
            if (op == ORC_SUM) iacc += v;
            else if (op == ORC_PROD) iacc *= v;
            else if (first || (op == ORC_MAX ? v > iacc : v < iacc)) iacc = v;
          } else {
            double v = cell_value(a, d, c);
            if (op == ORC_SUM) acc = acc + v;
            else if (op == ORC_PROD) acc = acc * v;
            else if (op == ORC_MAX) acc = v > acc ? v : acc;
            else acc = v < acc ? v : acc;
          }
          first = 0;
        }
  }
  *out = is_int ? (double)iacc : acc;
  return ORC_OK;
}

/* ---------------- introspection ---------------- */

int64_t orc_msg_count(const orc_t* w) { return w->n_msgs; }

int64_t orc_msgs(const orc_t* w, int64_t* out, int64_t cap) {
  int64_t n = w->n_msgs < cap ? w->n_msgs : cap;
  memcpy(out, w->msgs, (size_t)n * 4 * sizeof(int64_t));
  return n;
}

int orc_owner_map(const orc_t* w, int arr, int8_t* out) {
  if (arr < 0 || arr >= w->n_arrays || !w->arrays[arr].alive) return ORC_EINVAL;
  memcpy(out, w->arrays[arr].owner, (size_t)w->arrays[arr].n);
  return ORC_OK;
}

int orc_valid_map(const orc_t* w, int arr, uint64_t* out) {
  if (arr < 0 || arr >= w->n_arrays || !w->arrays[arr].alive) return ORC_EINVAL;
  memcpy(out, w->arrays[arr].valid, (size_t)w->arrays[arr].n * sizeof(uint64_t));
  return ORC_OK;
}

int orc_replica(const orc_t* w, int arr, int dev, void* out) {
  if (arr < 0 || arr >= w->n_arrays || !w->arrays[arr].alive) return ORC_EINVAL;
  if (dev < 0 || dev >= w->P || !w->with_data) return ORC_EINVAL;
  const oarr* a = &w->arrays[arr];
  memcpy(out, a->rep[dev], (size_t)a->n * a->es);
  return ORC_OK;
}
