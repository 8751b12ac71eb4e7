// common.hpp -- internal types of libaxe (host side).
//
// The product path: layouts -> storage composition -> joint digit
// refinement (App. B Alg. 1; split/fuse P:1016-1034) -> kernel
// parameter tables -> CUDA kernels (kernels.cu).  Nothing here is shared with
// oracle/ (the independent CPU checker).
#pragma once

#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>
#include <utility>
#include <algorithm>
#include <vector>

#include "axe.h"

namespace axe {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...) __attribute__((format(printf, 1, 2)));
const char *last_error();

#define AXE_FAIL(code, ...)          \
  do {                               \
    ::axe::set_error(__VA_ARGS__);   \
    return (code);                   \
  } while (0)

#define AXE_TRY(expr)                \
  do {                               \
    axe_status _st = (expr);         \
    if (_st != AXE_OK) return _st;   \
  } while (0)

// ---------------------------------------------------------------- axes
// Axis names are interned process-wide; ids are small, stable integers.
int intern_axis(const char *name);  // -1 if the name is not an identifier
const char *axis_name(int id);
bool valid_axis_name(const char *name);
int axis_m();      // id of "m"
int axis_gpuid();  // id of "gpuid"

// ---------------------------------------------------------------- layouts
struct Iter {
  int64_t e;  // extent >= 1
  int64_t s;  // stride != 0
  int a;      // axis id
};

// An Axe layout L = (D, R, O) (Def. Layout).
struct Layout {
  std::vector<Iter> D;                       // ordered, outermost first
  std::vector<Iter> R;                       // multiset
  std::vector<std::pair<int, int64_t>> O;    // nonzero components, first-appearance order
  std::vector<int> axes;                     // axes in first-appearance order over D, R, O
  int64_t ED = 1, ER = 1;

  int64_t offset(int a) const {
    for (auto &p : O)
      if (p.first == a) return p.second;
    return 0;
  }
  bool names_axis(int a) const {
    for (int x : axes)
      if (x == a) return true;
    return false;
  }
};

// Validate and build (computes E_D, E_R, axes; checks int64 overflow of the
// extent products and of every axis's coordinate range).
axe_status make_layout(std::vector<Iter> D, std::vector<Iter> R, std::vector<std::pair<int, int64_t>> O,
                       Layout *out);
// f_L(x): E_R rows over L.axes (App. Def. Induced map).
void eval_layout(const Layout &L, int64_t x, int64_t *rows);
// Signed closed-form bounds of an axis (Lemma span-closed, reading R1).
void axis_bounds(const Layout &L, int a, int64_t *mn, int64_t *mx);
// Canonical form, App. A.1.
Layout canonicalize(const Layout &L, bool *gap_ok);
// D0/D1 on an iter list.
std::vector<Iter> normalize_shard(const std::vector<Iter> &D);

// ---------------------------------------------------------------- storage
struct SDigit {
  int a;
  int64_t ext, div;
  int64_t mult;  // element-index multiplier prod_{j>k} ext_j
};
struct Storage {
  std::vector<SDigit> d;  // outermost first
  int swz_b = 0, swz_m = 0, swz_s = 0;
  int64_t cells = 1;
  bool binds(int a) const {
    for (auto &x : d)
      if (x.a == a) return true;
    return false;
  }
  // [0, top) bound of an axis (outermost digit: ext * div)
  int64_t top(int a) const {
    for (auto &x : d)
      if (x.a == a) return x.ext * x.div;
    return 0;
  }
};
axe_status make_storage(const axe_storage *st, Storage *out);
std::string storage_key(const Storage &s);
std::string layout_key(const Layout &L);

// A layout composed with its storage: every iter is now a stride on the
// buffer's element index ("memory components").
struct LinIter {
  int64_t e;
  int64_t s;        // element-index stride (may be negative); rank stride when dev
  int dev = 0;      // 1: a piece on the device axis (gpuid), kept unsplit
};
struct Linear {
  std::vector<LinIter> D;  // outermost first
  std::vector<LinIter> R;
  int64_t base = 0;        // element index of f_D(0) + O (the r = 0 representative)
  int64_t dev_base = 0;    // device-axis component of O
};
// Returns false (no error) when the composition is not affine in the digits;
// the caller then uses the generic kernel.  dev_axis: the device axis, whose
// iters are emitted as dev pieces (only when keep_dev) or dropped.
bool compose_linear(const Layout &L, const Storage &st, int dev_axis, Linear *out, bool keep_dev = false);

// Joint digit of a copy: one extent, a source and a destination stride.
struct Joint {
  int64_t e;
  int64_t ss, ds;
  int sdev = 0, ddev = 0;  // stride is on the device axis (redistribute)
};
// Refine two linear shard lists over the same domain into one joint digit list
// (innermost-first gcd/divisibility pairing; Alg. 1 generalised, R21).
bool joint_refine(const std::vector<LinIter> &src, const std::vector<LinIter> &dst, std::vector<Joint> *out);
// When the two digit systems do not nest (joint_refine fails), the innermost part still refines: pair
// from the fastest digit as joint_refine does, and at the first pair whose extents do not divide each
// other split off their gcd g as one more joint digit (both digits are multiples of g, so an aligned run
// of g consecutive x stays inside both).  What is left -- the outer index x / G over the two
// remaining lists -- has two independent decodings (src_rest, dst_rest, outermost first; the same
// product).  The inner list is empty when even the fastest pair shares no factor (gcd 1).
bool joint_refine_partial(const std::vector<LinIter> &src, const std::vector<LinIter> &dst, std::vector<Joint> *inner,
                          std::vector<LinIter> *src_rest, std::vector<LinIter> *dst_rest);

// Order digits by |dst stride| (outermost first) and fuse neighbours that are
// contiguous on both sides (Cor. fuse): fewer digits to decode.
inline void sort_fuse_outer(std::vector<Joint> &v) {
  std::stable_sort(v.begin(), v.end(), [](const Joint &a, const Joint &b) {
    int64_t x = a.ds < 0 ? -a.ds : a.ds, y = b.ds < 0 ? -b.ds : b.ds;
    return x > y;
  });
  std::vector<Joint> f;
  for (auto &j : v) {
    if (!f.empty() && f.back().ss == j.e * j.ss && f.back().ds == j.e * j.ds && f.back().sdev == j.sdev &&
        f.back().ddev == j.ddev) {
      f.back() = Joint{f.back().e * j.e, j.ss, j.ds, j.sdev, j.ddev};
    } else {
      f.push_back(j);
    }
  }
  v.swap(f);
}

inline int64_t ilog2_floor(uint64_t v) {
  int64_t r = -1;
  while (v) {
    v >>= 1;
    r++;
  }
  return r;
}

}  // namespace axe
