// rect.hpp — section algebra of the def/use tracker (host C++, no CUDA).
//
// A section is a half-open box [lb, ub) in up to three dimensions ("[LB:UB]",
// reading R1).  A section SET is kept in a canonical form: the unique "band"
// decomposition — split dimension 0 at every box boundary, take the cross-section
// of each elementary slab (recursively canonical in the remaining dimensions), and
// merge adjacent slabs whose cross-sections are equal.  Two sets cover the same
// cells iff their canonical forms are identical, so equality is a linear scan and
// a state can be hashed (the paper keeps GDEF sorted for "simple and linear-time
// GDEF comparisons", and merges "adjacent or redundant sections",
// P:L504).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

namespace hda {

struct Box {
  int64_t lb[3];
  int64_t ub[3];
};

inline Box unit_box() {
  Box b;
  for (int k = 0; k < 3; k++) {
    b.lb[k] = 0;
    b.ub[k] = 1;
  }
  return b;
}

inline bool box_empty(const Box& b) {
  return b.lb[0] >= b.ub[0] || b.lb[1] >= b.ub[1] || b.lb[2] >= b.ub[2];
}

inline int64_t box_volume(const Box& b) {
  if (box_empty(b)) return 0;
  return (b.ub[0] - b.lb[0]) * (b.ub[1] - b.lb[1]) * (b.ub[2] - b.lb[2]);
}

inline bool box_eq(const Box& a, const Box& b) {
  for (int k = 0; k < 3; k++)
    if (a.lb[k] != b.lb[k] || a.ub[k] != b.ub[k]) return false;
  return true;
}

inline Box box_and(const Box& a, const Box& b) {
  Box r;
  for (int k = 0; k < 3; k++) {
    r.lb[k] = std::max(a.lb[k], b.lb[k]);
    r.ub[k] = std::min(a.ub[k], b.ub[k]);
  }
  return r;
}

using Rects = std::vector<Box>;  // canonical (see file comment) unless noted

inline int64_t volume(const Rects& s) {
  int64_t v = 0;
  for (const Box& b : s) v += box_volume(b);
  return v;
}

inline bool rects_eq(const Rects& a, const Rects& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); i++)
    if (!box_eq(a[i], b[i])) return false;
  return true;
}

namespace detail {
// canonical decomposition of the union of `in` over dimensions [d, 3); the dims
// below d of the returned boxes are [0,1).  `in` holds non-empty boxes.
inline Rects canon_from(const std::vector<Box>& in, int d) {
  Rects out;
  if (in.empty()) return out;
  if (d == 3) {
    out.push_back(unit_box());
    return out;
  }
  std::vector<int64_t> xs;
  xs.reserve(in.size() * 2);
  for (const Box& b : in) {
    xs.push_back(b.lb[d]);
    xs.push_back(b.ub[d]);
  }
  std::sort(xs.begin(), xs.end());
  xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
  Rects prev;
  bool have = false;
  int64_t lo_band = 0, hi_band = 0;
  auto flush = [&]() {
    if (!have) return;
    for (Box c : prev) {
      c.lb[d] = lo_band;
      c.ub[d] = hi_band;
      out.push_back(c);
    }
  };
  std::vector<Box> active;
  for (size_t i = 0; i + 1 < xs.size(); i++) {
    int64_t lo = xs[i], hi = xs[i + 1];
    active.clear();
    for (const Box& b : in)
      if (b.lb[d] <= lo && b.ub[d] >= hi) active.push_back(b);
    Rects cs = canon_from(active, d + 1);
    if (have && hi_band == lo && rects_eq(cs, prev)) {
      hi_band = hi;
      continue;
    }
    flush();
    prev.swap(cs);
    lo_band = lo;
    hi_band = hi;
    have = true;
  }
  flush();
  return out;
}

// a − b as up to 6 disjoint boxes
inline void box_minus(const Box& a, const Box& b, std::vector<Box>& out) {
  Box i = box_and(a, b);
  if (box_empty(i)) {
    out.push_back(a);
    return;
  }
  Box rest = a;
  for (int k = 0; k < 3; k++) {
    if (rest.lb[k] < i.lb[k]) {
      Box p = rest;
      p.ub[k] = i.lb[k];
      out.push_back(p);
      rest.lb[k] = i.lb[k];
    }
    if (i.ub[k] < rest.ub[k]) {
      Box p = rest;
      p.lb[k] = i.ub[k];
      out.push_back(p);
      rest.ub[k] = i.ub[k];
    }
  }
}
}  // namespace detail

// canonical form of an arbitrary list of boxes (empties, overlaps allowed)
inline Rects canonicalize(const std::vector<Box>& raw) {
  std::vector<Box> in;
  in.reserve(raw.size());
  for (const Box& b : raw)
    if (!box_empty(b)) in.push_back(b);
  return detail::canon_from(in, 0);
}

inline Rects unite(const Rects& a, const Rects& b) {
  if (a.empty()) return b;
  if (b.empty()) return a;
  std::vector<Box> all(a);
  all.insert(all.end(), b.begin(), b.end());
  return canonicalize(all);
}

inline Rects intersect(const Rects& a, const Rects& b) {
  std::vector<Box> out;
  for (const Box& x : a)
    for (const Box& y : b) {
      Box i = box_and(x, y);
      if (!box_empty(i)) out.push_back(i);
    }
  return canonicalize(out);
}

inline bool intersects(const Rects& a, const Rects& b) {
  for (const Box& x : a)
    for (const Box& y : b)
      if (!box_empty(box_and(x, y))) return true;
  return false;
}

inline Rects subtract(const Rects& a, const Rects& b) {
  if (a.empty() || b.empty()) return a;
  std::vector<Box> cur(a), nxt;
  for (const Box& y : b) {
    nxt.clear();
    for (const Box& x : cur) detail::box_minus(x, y, nxt);
    cur.swap(nxt);
  }
  return canonicalize(cur);
}

// serialize (for hashing / exact keys)
inline void append_rects(std::vector<int64_t>& key, const Rects& s) {
  key.push_back((int64_t)s.size());
  for (const Box& b : s)
    for (int k = 0; k < 3; k++) {
      key.push_back(b.lb[k]);
      key.push_back(b.ub[k]);
    }
}

struct KeyHash {
  size_t operator()(const std::vector<int64_t>& v) const {
    uint64_t h = 0x9E3779B97F4A7C15ULL ^ v.size();
    for (int64_t x : v) {
      h ^= (uint64_t)x + 0x9E3779B97F4A7C15ULL + (h << 6) + (h >> 2);
      h *= 0xBF58476D1CE4E5B9ULL;
    }
    return (size_t)(h ^ (h >> 31));
  }
};

}  // namespace hda
