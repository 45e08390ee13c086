// tracker.cpp — compose / validate / plan / commit / cache (see tracker.hpp).
#include "tracker.hpp"

#include <algorithm>
#include <array>

#include "hdarray.h"

namespace hda {

// ---------------------------------------------------------------- arrays, partitions

int Tracker::add_array(int dtype, int ndim, const int64_t* shape, std::string& err) {
  if (!dtype_size(dtype)) {
    err = "unknown dtype";
    return HDA_EINVAL;
  }
  if (ndim < 1 || ndim > 3) {
    err = "ndim must be 1..3";
    return HDA_EINVAL;
  }
  TArray a;
  a.alive = true;
  a.dtype = dtype;
  a.ndim = ndim;
  a.es = dtype_size(dtype);
  for (int k = 0; k < ndim; k++) {
    if (shape[k] < 1) {
      err = "zero extent";
      return HDA_EINVAL;
    }
    a.shape[k] = shape[k];
  }
  int id = (int)arrays_.size();
  arrays_.push_back(a);
  states_.emplace_back();
  state_index_.emplace_back();
  ArrState s;  // all sets empty at Create
  s.own.assign(P_, Rects());
  s.stale.assign(P_, Rects());
  arrays_[id].state = intern(id, std::move(s));
  return id;
}

void Tracker::free_array(int id) {
  arrays_[id].alive = false;
  states_[id].clear();
  state_index_[id].clear();
  clear_cache();
}

void Tracker::clear_cache() {
  cache_.clear();
  specs_.clear();
}

// even split, first n%k parts one larger ("evenly", reading R4)
static void split(int64_t lo, int64_t n, int k, int i, int64_t* s, int64_t* e) {
  int64_t b = n / k, r = n % k;
  *s = lo + (int64_t)i * b + std::min<int64_t>(i, r);
  *e = *s + b + (i < r ? 1 : 0);
}

int Tracker::add_partition(int kind, int ndim, const int64_t* domain, const int64_t* lb,
                           const int64_t* ub, std::string& err) {
  if (ndim < 1 || ndim > 3) {
    err = "ndim must be 1..3";
    return HDA_EINVAL;
  }
  if (kind != HDA_ROW && kind != HDA_COL && kind != HDA_BLOCK) {
    err = "unknown partition kind";
    return HDA_EINVAL;
  }
  if (kind != HDA_ROW && ndim < 2) {
    err = "COL/BLOCK need >= 2 dimensions";
    return HDA_EUNSUPPORTED;
  }
  TPart p;
  p.ndim = ndim;
  for (int k = 0; k < ndim; k++) {
    if (domain[k] < 1) {
      err = "zero domain extent";
      return HDA_EINVAL;
    }
    if (lb[k] > ub[k]) {
      err = "region lb > ub";
      return HDA_EINVAL;
    }
    if (lb[k] < 0 || ub[k] > domain[k]) {
      err = "region outside the domain";
      return HDA_ERANGE;
    }
    p.domain[k] = domain[k];
  }
  // BLOCK: pr x pc grid, pc = largest divisor of P with pc*pc <= P (reading R5)
  int pr = P_, pc = 1;
  if (kind == HDA_BLOCK) {
    for (int c = 1; c * c <= P_; c++)
      if (P_ % c == 0) pc = c;
    pr = P_ / pc;
  }
  for (int d = 0; d < P_; d++) {
    Box b = unit_box();
    for (int k = 0; k < ndim; k++) {
      b.lb[k] = lb[k];
      b.ub[k] = ub[k];
    }
    if (kind == HDA_ROW) {
      split(lb[0], ub[0] - lb[0], P_, d, &b.lb[0], &b.ub[0]);
    } else if (kind == HDA_COL) {
      split(lb[1], ub[1] - lb[1], P_, d, &b.lb[1], &b.ub[1]);
    } else {
      split(lb[0], ub[0] - lb[0], pr, d / pc, &b.lb[0], &b.ub[0]);
      split(lb[1], ub[1] - lb[1], pc, d % pc, &b.lb[1], &b.ub[1]);
    }
    p.box.push_back(b);
  }
  parts_.push_back(p);
  return (int)parts_.size() - 1;
}

int Tracker::add_partition_manual(int ndim, const int64_t* domain, const int64_t* lbs,
                                  const int64_t* ubs, std::string& err) {
  if (ndim < 1 || ndim > 3) {
    err = "ndim must be 1..3";
    return HDA_EINVAL;
  }
  TPart p;
  p.ndim = ndim;
  for (int k = 0; k < ndim; k++) {
    if (domain[k] < 1) {
      err = "zero domain extent";
      return HDA_EINVAL;
    }
    p.domain[k] = domain[k];
  }
  for (int d = 0; d < P_; d++) {
    Box b = unit_box();
    for (int k = 0; k < ndim; k++) {
      b.lb[k] = lbs[d * ndim + k];
      b.ub[k] = ubs[d * ndim + k];
      if (b.lb[k] > b.ub[k]) {
        err = "region lb > ub";
        return HDA_EINVAL;
      }
      if (b.lb[k] < 0 || b.ub[k] > domain[k]) {
        err = "region outside the domain";
        return HDA_ERANGE;
      }
    }
    p.box.push_back(b);
  }
  for (int a = 0; a < P_; a++)
    for (int b = a + 1; b < P_; b++)
      if (!box_empty(box_and(p.box[a], p.box[b]))) {
        err = "manual partition regions of devices " + std::to_string(a) + " and " +
              std::to_string(b) + " overlap";
        return HDA_EOVERLAP;
      }
  parts_.push_back(p);
  return (int)parts_.size() - 1;
}

// ---------------------------------------------------------------- composition

// LUSE/LDEF = union over offset tuples of the work box shifted by
// the tuple ('*' = whole extent of the array's dimension), clamped to the array (R6).
Rects compose(const int32_t* tuples, int32_t n, int ndim, const Box& work, const int64_t* shape) {
  std::vector<Box> raw;
  if (box_empty(work)) return Rects();
  for (int32_t t = 0; t < n; t++) {
    const int32_t* d = tuples + (size_t)t * ndim;
    Box b = unit_box();
    bool empty = false;
    for (int k = 0; k < ndim; k++) {
      if (d[k] == STAR) {
        b.lb[k] = 0;
        b.ub[k] = shape[k];
      } else {
        b.lb[k] = std::max<int64_t>(work.lb[k] + d[k], 0);
        b.ub[k] = std::min<int64_t>(work.ub[k] + d[k], shape[k]);
      }
      if (b.lb[k] >= b.ub[k]) empty = true;
    }
    if (!empty) raw.push_back(b);
  }
  return canonicalize(raw);
}

// ---------------------------------------------------------------- validation

static bool zero_tuple(const int32_t* d, int nd) {
  for (int k = 0; k < nd; k++)
    if (d[k] != 0) return false;
  return true;
}

// declared tuple covers a required one: equal per dim, or declared '*'
static bool declared(const AccessIn& a, int nd, const int32_t* r) {
  for (int t = 0; t < a.n_use; t++) {
    const int32_t* d = a.use + (size_t)t * nd;
    bool ok = true;
    for (int k = 0; k < nd; k++)
      if (!(d[k] == STAR || d[k] == r[k])) ok = false;
    if (ok) return true;
  }
  return false;
}

static int nparams(int32_t kernel) {
  switch (kernel) {
    case KN_JACOBI5:
    case KN_COPY:
    case KN_STENCIL9:
    case KN_STENCIL7_3D: return 2;
    case KN_SCALE:
    case KN_READ:
    case KN_WRITE: return 1;
    case KN_GEMM: return 3;
    case KN_STAMP:  // [X, used...]
    case KN_NONE: return -1;
  }
  return -2;
}

// per-kernel minimum scalar count: checked on EVERY call, cache hit or not (the spec
// key does not hold the scalar values, so a cached spec says nothing about them)
static int check_scalars(int32_t kernel, int32_t n_scalars, std::string& err) {
  if ((kernel == KN_SCALE || kernel == KN_STAMP) && n_scalars < 1) {
    err = "kernel needs scalars[0]";
    return HDA_EINVAL;
  }
  if (kernel == KN_GEMM && n_scalars < 2) {
    err = "GEMM needs scalars {alpha, beta}";
    return HDA_EINVAL;
  }
  return HDA_OK;
}

int Tracker::validate_and_compose(int32_t kernel, int32_t part, const AccessIn* acc, int32_t n_acc,
                                  const double* scalars, int32_t n_scalars, CallInfo& ci,
                                  std::string& err) const {
  int np = nparams(kernel);
  if (np == -2) {
    err = "unknown kernel";
    return HDA_EINVAL;
  }
  if ((np >= 0 && n_acc != np) || n_acc < 0 || n_acc > 64) {
    err = "wrong number of kernel parameters";
    return HDA_EINVAL;
  }
  if (!part_ok(part)) {
    err = "unknown partition";
    return HDA_EINVAL;
  }
  const TPart& pt = parts_[part];
  const int nd = pt.ndim;
  for (int e = 0; e < n_acc; e++) {
    if (!array_ok(acc[e].array)) {
      err = "unknown array handle";
      return HDA_EINVAL;
    }
    if (arrays_[acc[e].array].ndim != nd) {
      err = "array rank differs from the partition rank";
      return HDA_EINVAL;
    }
    if (acc[e].n_use < 0 || acc[e].n_def < 0 || (acc[e].n_use && !acc[e].use) ||
        (acc[e].n_def && !acc[e].def)) {
      err = "bad offset list";
      return HDA_EINVAL;
    }
  }
  bool any_abs = false;
  for (int e = 0; e < n_acc; e++) any_abs |= acc[e].absolute();
  if (any_abs && kernel != KN_NONE && kernel != KN_STAMP) {
    err = "absolute sections are for kernels without a fixed footprint (NONE, STAMP)";
    return HDA_EINVAL;
  }
  const bool builtin = kernel > KN_NONE && kernel != KN_STAMP;
  if (builtin) {
    if (!(acc[0].n_def == 1 && zero_tuple(acc[0].def, nd))) {
      err = "built-in kernels define exactly parameter 0 at offset (0,..,0)";
      return HDA_EINVAL;
    }
    for (int e = 1; e < n_acc; e++)
      if (acc[e].n_def) {
        err = "only parameter 0 may be defined";
        return HDA_EINVAL;
      }
  }
  if (int rc = check_scalars(kernel, n_scalars, err)) return rc;
  if (kernel == KN_STAMP) {
    if (n_acc < 1) {
      err = "STAMP needs at least the stamped array";
      return HDA_EINVAL;
    }
    for (int e = 1; e < n_acc; e++) {
      bool d = acc[e].n_def != 0;
      if (acc[e].n_def_abs)
        for (int q = 0; q < P_; q++) d |= acc[e].n_def_abs[q] != 0;
      if (d) {
        err = "STAMP defines only parameter 0";
        return HDA_EINVAL;
      }
    }
  }
  const int32_t zero[3] = {0, 0, 0};
  int64_t halo = 0;
  if (kernel == KN_JACOBI5 || kernel == KN_STENCIL9 || kernel == KN_STENCIL7_3D) {
    const TArray &dst = arrays_[acc[0].array], &src = arrays_[acc[1].array];
    if (kernel == KN_STENCIL7_3D ? nd != 3 : nd != 2) {
      err = "stencil rank";
      return HDA_EINVAL;
    }
    if (dst.dtype != src.dtype) {
      err = "stencil dtypes differ";
      return HDA_EINVAL;
    }
    if (src.dtype != DT_F64 && src.dtype != DT_F32) {
      err = "stencils support f64/f32";
      return HDA_EUNSUPPORTED;
    }
    for (int k = 0; k < 3; k++)
      if (dst.shape[k] != src.shape[k]) {
        err = "stencil shapes differ";
        return HDA_EINVAL;
      }
    std::vector<std::array<int32_t, 3>> fp;
    if (kernel == KN_JACOBI5) {
      fp = {{0, -1, 0}, {0, 1, 0}, {-1, 0, 0}, {1, 0, 0}};
    } else if (kernel == KN_STENCIL9) {
      for (int a = -1; a <= 1; a++)
        for (int b = -1; b <= 1; b++)
          if (a || b) fp.push_back({a, b, 0});
    } else {
      fp = {{0, 0, -1}, {0, 0, 1}, {0, -1, 0}, {0, 1, 0}, {-1, 0, 0}, {1, 0, 0}};
    }
    for (auto& r : fp)
      if (!declared(acc[1], nd, r.data())) {
        err = "use offsets do not cover the kernel's footprint";
        return HDA_EINVAL;
      }
    halo = 1;
  } else if (kernel == KN_COPY) {
    const TArray &b = arrays_[acc[0].array], &a = arrays_[acc[1].array];
    if (a.dtype != b.dtype) {
      err = "copy dtypes differ";
      return HDA_EINVAL;
    }
    for (int k = 0; k < 3; k++)
      if (a.shape[k] != b.shape[k]) {
        err = "copy shapes differ";
        return HDA_EINVAL;
      }
    if (!declared(acc[1], nd, zero)) {
      err = "copy needs use (0,..,0) on the source";
      return HDA_EINVAL;
    }
  } else if (kernel == KN_SCALE) {
    int dt = arrays_[acc[0].array].dtype;
    if (dt != DT_F64 && dt != DT_F32 && dt != DT_BF16) {
      err = "scale supports f64/f32/bf16";
      return HDA_EUNSUPPORTED;
    }
    if (!declared(acc[0], nd, zero)) {
      err = "scale needs use (0,..,0)";
      return HDA_EINVAL;
    }
  } else if (kernel == KN_GEMM) {
    const TArray &C = arrays_[acc[0].array], &A = arrays_[acc[1].array], &B = arrays_[acc[2].array];
    if (nd != 2) {
      err = "GEMM is 2-D";
      return HDA_EINVAL;
    }
    if (A.dtype != DT_BF16 || B.dtype != DT_BF16 || (C.dtype != DT_F32 && C.dtype != DT_BF16)) {
      err = "GEMM needs bf16 A, B and f32/bf16 C";
      return HDA_EUNSUPPORTED;
    }
    if (A.shape[0] != C.shape[0] || B.shape[1] != C.shape[1] || A.shape[1] != B.shape[0]) {
      err = "GEMM shapes";
      return HDA_EINVAL;
    }
    const int32_t ra[2] = {0, STAR}, rb[2] = {STAR, 0};
    if (!declared(acc[1], 2, ra) || !declared(acc[2], 2, rb)) {
      err = "GEMM needs use A (0,*) and use B (*,0) (Listing 2)";
      return HDA_EINVAL;
    }
    if (scalars[1] != 0.0 && !declared(acc[0], 2, zero)) {
      err = "GEMM with beta != 0 needs use C (0,0)";
      return HDA_EINVAL;
    }
    if (acc[0].array == acc[1].array || acc[0].array == acc[2].array) {
      err = "GEMM C aliases A or B";
      return HDA_EINVAL;
    }
  }
  if (builtin) {  // work (+ halo) inside the arrays the kernel touches
    const TArray& a0 = arrays_[acc[0].array];
    for (int d = 0; d < P_; d++) {
      const Box& w = pt.box[d];
      if (box_empty(w)) continue;
      for (int k = 0; k < nd; k++)
        if (w.lb[k] - halo < 0 || w.ub[k] + halo > a0.shape[k]) {
          err = "work region (+ stencil footprint) leaves the array";
          return HDA_ERANGE;
        }
    }
  }
  if (kernel == KN_READ || kernel == KN_WRITE) {
    const TArray& a0 = arrays_[acc[0].array];
    for (int d = 0; d < P_; d++) {
      const Box& w = pt.box[d];
      if (box_empty(w)) continue;
      for (int k = 0; k < nd; k++)
        if (w.ub[k] > a0.shape[k]) {
          err = "partition region leaves the array";
          return HDA_ERANGE;
        }
    }
  }
  // used at a non-zero offset and defined in the same call (reading R15)
  for (int e = 0; e < n_acc; e++)
    for (int f = 0; f < n_acc; f++) {
      if (acc[e].absolute() || acc[f].absolute()) continue;
      if (acc[e].array != acc[f].array || !acc[f].n_def) continue;
      for (int t = 0; t < acc[e].n_use; t++)
        if (!zero_tuple(acc[e].use + (size_t)t * nd, nd)) {
          err = "array used at a non-zero offset and defined in the same call";
          return HDA_EINVAL;
        }
    }
  // compose LUSE/LDEF per distinct array
  ci.kernel = kernel;
  ci.part = part;
  ci.param_array.clear();
  for (int e = 0; e < n_acc; e++) {
    ci.param_array.push_back(acc[e].array);
    if (std::find(ci.arrays.begin(), ci.arrays.end(), acc[e].array) == ci.arrays.end())
      ci.arrays.push_back(acc[e].array);
  }
  size_t na = ci.arrays.size();
  ci.luse.assign(na, std::vector<Rects>(P_));
  ci.ldef.assign(na, std::vector<Rects>(P_));
  ci.used.assign(na, false);
  ci.defined.assign(na, false);
  for (size_t i = 0; i < na; i++) {
    int X = ci.arrays[i];
    const TArray& a = arrays_[X];
    for (int d = 0; d < P_; d++) {
      std::vector<Box> u, df;
      for (int e = 0; e < n_acc; e++) {
        if (acc[e].array != X) continue;
        if (acc[e].absolute()) {  // explicit per-device sections
          for (int pass = 0; pass < 2; pass++) {
            const int32_t* cnt = pass ? acc[e].n_def_abs : acc[e].n_use_abs;
            const int64_t* bx = pass ? acc[e].def_abs : acc[e].use_abs;
            if (!cnt) continue;
            int64_t off = 0;
            for (int q = 0; q < d; q++) off += (int64_t)cnt[q] * 2 * nd;
            for (int32_t b = 0; b < cnt[d]; b++) {
              Box bb = unit_box();
              for (int kk = 0; kk < nd; kk++) {
                bb.lb[kk] = bx[off + (int64_t)b * 2 * nd + kk];
                bb.ub[kk] = bx[off + (int64_t)b * 2 * nd + nd + kk];
                if (bb.lb[kk] < 0 || bb.ub[kk] > a.shape[kk] || bb.lb[kk] > bb.ub[kk]) {
                  err = "absolute section outside the array";
                  return HDA_ERANGE;
                }
              }
              (pass ? df : u).push_back(bb);
            }
          }
          continue;
        }
        Rects cu = compose(acc[e].use, acc[e].n_use, nd, pt.box[d], a.shape);
        Rects cd = compose(acc[e].def, acc[e].n_def, nd, pt.box[d], a.shape);
        u.insert(u.end(), cu.begin(), cu.end());
        df.insert(df.end(), cd.begin(), cd.end());
      }
      ci.luse[i][d] = canonicalize(u);
      ci.ldef[i][d] = canonicalize(df);
      if (!ci.luse[i][d].empty()) ci.used[i] = true;
      if (!ci.ldef[i][d].empty()) ci.defined[i] = true;
    }
    // two devices define the same cell
    for (int p = 0; p < P_; p++)
      for (int r = p + 1; r < P_; r++)
        if (intersects(ci.ldef[i][p], ci.ldef[i][r])) {
          err = "devices " + std::to_string(p) + " and " + std::to_string(r) +
                " define the same cells in one call";
          return HDA_ERACE;
        }
  }
  return HDA_OK;
}

// ---------------------------------------------------------------- states

int Tracker::intern(int array, ArrState&& s) {
  std::vector<int64_t> key;
  for (int d = 0; d < P_; d++) {
    append_rects(key, s.own[d]);
    append_rects(key, s.stale[d]);
  }
  auto& idx = state_index_[array];
  auto it = idx.find(key);
  if (it != idx.end()) return it->second;
  int id = (int)states_[array].size();
  states_[array].push_back(std::move(s));
  idx.emplace(std::move(key), id);
  return id;
}

void Tracker::owner_map(int id, int8_t* out) const {
  const TArray& a = arrays_[id];
  int64_t n = a.shape[0] * a.shape[1] * a.shape[2];
  std::fill(out, out + n, (int8_t)-1);
  const ArrState& s = state(id);
  for (int p = 0; p < P_; p++)
    for (const Box& b : s.own[p])
      for (int64_t i = b.lb[0]; i < b.ub[0]; i++)
        for (int64_t j = b.lb[1]; j < b.ub[1]; j++) {
          int64_t base = (i * a.shape[1] + j) * a.shape[2];
          std::fill(out + base + b.lb[2], out + base + b.ub[2], (int8_t)p);
        }
}

// ---------------------------------------------------------------- planning

static bool msg_less(const Msg& a, const Msg& b) {
  if (a.array != b.array) return a.array < b.array;
  if (a.src != b.src) return a.src < b.src;
  if (a.dst != b.dst) return a.dst < b.dst;
  for (int k = 0; k < 3; k++)
    if (a.box.lb[k] != b.box.lb[k]) return a.box.lb[k] < b.box.lb[k];
  return false;
}

void Tracker::compute(const CallInfo& ci, Transition& t) {
  t.info = &ci;
  t.msgs.clear();
  t.next.clear();
  t.bytes = 0;
  for (size_t i = 0; i < ci.arrays.size(); i++) {
    int X = ci.arrays[i];
    const TArray& a = arrays_[X];
    const ArrState& cur = states_[X][a.state];
    ArrState nx = cur;
    if (ci.used[i]) {
      // Eq. 1-2: M_{p->q} = LUSE_q ∩ stale_q ∩ own_p
      for (int q = 0; q < P_; q++) {
        const Rects& L = ci.luse[i][q];
        if (L.empty() || cur.stale[q].empty()) continue;
        Rects need = intersect(L, cur.stale[q]);
        if (need.empty()) continue;
        for (int p = 0; p < P_; p++) {
          if (p == q || cur.own[p].empty()) continue;
          Rects m = intersect(need, cur.own[p]);
          for (const Box& b : m) {
            t.msgs.push_back(Msg{X, p, q, b});
            t.bytes += box_volume(b) * (int64_t)a.es;
          }
        }
        // Eq. 3-4 "- RECVMSG": everything q uses is now current on q
        nx.stale[q] = subtract(cur.stale[q], L);
      }
    }
    if (ci.defined[i]) {
      // Eq. 3-4 "∪ LDEF", with last-writer semantics (reading R7)
      for (int p = 0; p < P_; p++) {
        const Rects& D = ci.ldef[i][p];
        if (D.empty()) continue;
        nx.own[p] = unite(nx.own[p], D);
        nx.stale[p] = subtract(nx.stale[p], D);
        for (int r = 0; r < P_; r++) {
          if (r == p) continue;
          nx.own[r] = subtract(nx.own[r], D);
          nx.stale[r] = unite(nx.stale[r], D);
        }
      }
    }
    t.next.push_back(intern(X, std::move(nx)));
  }
  std::sort(t.msgs.begin(), t.msgs.end(), msg_less);
  t.serial = ++serial_;
}

int Tracker::plan(int32_t kernel, int32_t part, const AccessIn* acc, int32_t n_acc,
                  const double* scalars, int32_t n_scalars, bool use_cache,
                  const Transition** out, bool* hit, std::string& err) {
  if (int rc = check_scalars(kernel, n_scalars, err)) return rc;
  // exact spec key
  std::vector<int64_t>& key = key_;
  key.clear();
  key.push_back(kernel);
  key.push_back(part);
  key.push_back(kernel == KN_GEMM && n_scalars >= 2 && scalars[1] != 0.0);
  key.push_back(n_acc);
  for (int e = 0; e < n_acc; e++) {
    key.push_back(acc[e].array);
    if (!array_ok(acc[e].array)) {
      err = "unknown array handle";
      return HDA_EINVAL;
    }
    int nd = arrays_[acc[e].array].ndim;
    key.push_back(acc[e].absolute() ? 1 : 0);
    if (acc[e].absolute()) {
      for (int pass = 0; pass < 2; pass++) {
        const int32_t* cnt = pass ? acc[e].n_def_abs : acc[e].n_use_abs;
        const int64_t* bx = pass ? acc[e].def_abs : acc[e].use_abs;
        int64_t off = 0;
        for (int q = 0; q < P_; q++) {
          int32_t n = cnt ? cnt[q] : 0;
          key.push_back(n);
          for (int64_t i = 0; i < (int64_t)n * 2 * nd; i++) key.push_back(bx[off + i]);
          off += (int64_t)n * 2 * nd;
        }
      }
      continue;
    }
    key.push_back(acc[e].n_use);
    for (int i = 0; i < acc[e].n_use * nd && acc[e].use; i++) key.push_back(acc[e].use[i]);
    key.push_back(acc[e].n_def);
    for (int i = 0; i < acc[e].n_def * nd && acc[e].def; i++) key.push_back(acc[e].def[i]);
  }
  const CallInfo* ci;
  auto sit = use_cache ? specs_.find(key) : specs_.end();
  if (sit != specs_.end()) {
    ci = sit->second.get();
  } else {
    auto nci = std::make_unique<CallInfo>();
    int rc = validate_and_compose(kernel, part, acc, n_acc, scalars, n_scalars, *nci, err);
    if (rc) return rc;
    ci = nci.get();
    if (use_cache)
      specs_[key] = std::move(nci);
    else
      scratch_ci_ = std::move(nci);
  }
  // transition key = spec key + state ids of the touched arrays
  for (int X : ci->arrays) key.push_back(arrays_[X].state);
  if (use_cache) {
    auto it = cache_.find(key);
    if (it != cache_.end()) {
      *out = it->second.get();
      *hit = true;
      return HDA_OK;
    }
    auto t = std::make_unique<Transition>();
    compute(*ci, *t);
    *out = t.get();
    cache_[key] = std::move(t);
  } else {
    scratch_ = std::make_unique<Transition>();
    compute(*ci, *scratch_);
    *out = scratch_.get();
  }
  *hit = false;
  return HDA_OK;
}

void Tracker::commit(const Transition* t) {
  const CallInfo& ci = *t->info;
  for (size_t i = 0; i < ci.arrays.size(); i++) arrays_[ci.arrays[i]].state = t->next[i];
}

}  // namespace hda
