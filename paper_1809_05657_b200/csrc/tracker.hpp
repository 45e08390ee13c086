// tracker.hpp — the def/use region tracker (host C++, no CUDA).
//
// Per array X and device p it keeps two canonical section sets:
//   own[p]   = cells whose last writer is p                 (the paper's sGDEF_{p,*} source side)
//   stale[p] = cells for which p does NOT hold the current value
// so that sGDEF_{p,q} = own[p] ∩ stale[q] and rGDEF_{q,p} is its mirror.
// A call k composes LUSE/LDEF from the kernel's offsets and the work partition
// (P:L185-186), plans the messages
//   M_{p->q}(X) = LUSE_q(X) ∩ own[p] ∩ stale[q]                      (Eq. 1-2)
// and commits with last-writer semantics (Eq. 3-4, corrected, reading R7):
//   stale[q] -= LUSE_q ; for each LDEF_p = D: own[p] ∪= D, own[r] -= D, stale[r] ∪= D (r≠p),
//   stale[p] -= D.
// States are interned per array (hash-consing of the canonical sets), so a call is a
// transition (call spec, state ids) -> (messages, next state ids) that is cached:
// the paper's history buffers and intersection cache, made exact.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "rect.hpp"

namespace hda {

constexpr int32_t STAR = INT32_MIN;

// kernel ids (mirror include/hdarray.h enum hda_kernel) + internal pseudo-kernels
enum : int32_t {
  KN_NONE = 0, KN_JACOBI5 = 1, KN_COPY = 2, KN_STENCIL9 = 3, KN_STENCIL7_3D = 4,
  KN_SCALE = 5, KN_GEMM = 6, KN_STAMP = 7, KN_COUNT = 8,
  KN_READ = -1,   // coherence-only call of hda_read (uses = region, no defs)
  KN_WRITE = -2   // hda_write (defs = region, no uses)
};

enum : int { DT_F64 = 0, DT_F32 = 1, DT_BF16 = 2, DT_I32 = 3, DT_I64 = 4 };

inline size_t dtype_size(int dt) {
  switch (dt) {
    case DT_F64: return 8;
    case DT_F32: return 4;
    case DT_BF16: return 2;
    case DT_I32: return 4;
    case DT_I64: return 8;
  }
  return 0;
}

struct TArray {
  bool alive = false;
  int dtype = 0, ndim = 0;
  int64_t shape[3] = {1, 1, 1};
  size_t es = 0;
  int state = 0;  // current interned state id
  Box full() const {
    Box b = unit_box();
    for (int k = 0; k < 3; k++) b.ub[k] = shape[k];
    return b;
  }
};

struct TPart {
  int ndim = 0;
  int64_t domain[3] = {1, 1, 1};
  std::vector<Box> box;  // one per device, possibly empty
};

struct Msg {
  int32_t array, src, dst;
  Box box;
};

struct AccessIn {  // one access-list entry, as passed through the C-ABI
  int32_t array;
  int32_t n_use;
  const int32_t* use;
  int32_t n_def;
  const int32_t* def;
  // absolute sections (Table 1 use@/def@): per-device box counts [P] and boxes
  // (lb[ndim], ub[ndim] each, device-major); when set, the offsets are ignored
  const int32_t* n_use_abs = nullptr;
  const int64_t* use_abs = nullptr;
  const int32_t* n_def_abs = nullptr;
  const int64_t* def_abs = nullptr;
  bool absolute() const { return n_use_abs != nullptr || n_def_abs != nullptr; }
};

// state-independent facts about a call spec, validated once
struct CallInfo {
  int32_t kernel = 0, part = 0;
  std::vector<int32_t> arrays;                  // distinct arrays, first-appearance order
  std::vector<std::vector<Rects>> luse, ldef;   // [distinct array][device]
  std::vector<bool> used, defined;              // per distinct array
  std::vector<int32_t> param_array;             // entry i -> array id
};

struct ArrState {
  std::vector<Rects> own, stale;
};

struct Transition {
  const CallInfo* info = nullptr;
  std::vector<Msg> msgs;          // canonical order: (array, src, dst, lb)
  std::vector<int32_t> next;      // per distinct array: next state id
  int64_t bytes = 0;
  uint64_t serial = 0;            // unique id (for runtime-side caches)
};

class Tracker {
 public:
  explicit Tracker(int P) : P_(P) {}
  int P() const { return P_; }

  int add_array(int dtype, int ndim, const int64_t* shape, std::string& err);
  void free_array(int id);
  int add_partition(int kind, int ndim, const int64_t* domain, const int64_t* lb,
                    const int64_t* ub, std::string& err);
  int add_partition_manual(int ndim, const int64_t* domain, const int64_t* lbs,
                           const int64_t* ubs, std::string& err);

  // Validate + compose (cached per spec) and plan (cached per spec+state).
  // Returns 0 or a negative HDA status; on success *out points to the transition
  // (owned by the cache, or by `scratch` when caching is disabled) and *hit says
  // whether it came from the cache.
  int plan(int32_t kernel, int32_t part, const AccessIn* acc, int32_t n_acc,
           const double* scalars, int32_t n_scalars, bool use_cache,
           const Transition** out, bool* hit, std::string& err);
  void commit(const Transition* t);
  void clear_cache();

  const TArray& array(int id) const { return arrays_[id]; }
  bool array_ok(int id) const { return id >= 0 && id < (int)arrays_.size() && arrays_[id].alive; }
  bool part_ok(int id) const { return id >= 0 && id < (int)parts_.size(); }
  const TPart& part(int id) const { return parts_[id]; }
  const ArrState& state(int id) const { return states_[id][arrays_[id].state]; }
  void owner_map(int id, int8_t* out) const;

 private:
  int P_;
  std::vector<TArray> arrays_;
  std::vector<TPart> parts_;
  std::vector<std::vector<ArrState>> states_;
  std::vector<std::unordered_map<std::vector<int64_t>, int, KeyHash>> state_index_;
  std::unordered_map<std::vector<int64_t>, std::unique_ptr<CallInfo>, KeyHash> specs_;
  std::unordered_map<std::vector<int64_t>, std::unique_ptr<Transition>, KeyHash> cache_;
  std::unique_ptr<Transition> scratch_;
  std::unique_ptr<CallInfo> scratch_ci_;
  uint64_t serial_ = 0;
  std::vector<int64_t> key_;  // reused buffer

  int intern(int array, ArrState&& s);
  int validate_and_compose(int32_t kernel, int32_t part, const AccessIn* acc, int32_t n_acc,
                           const double* scalars, int32_t n_scalars, CallInfo& ci,
                           std::string& err) const;
  void compute(const CallInfo& ci, Transition& t);
};

Rects compose(const int32_t* tuples, int32_t n, int ndim, const Box& work, const int64_t* shape);

}  // namespace hda
