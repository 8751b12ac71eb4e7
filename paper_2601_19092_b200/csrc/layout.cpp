// layout.cpp -- Axe layout core (host): creation/validation, evaluation,
// closed-form bounds, canonicalisation, storage descriptors, composition of a
// layout with its storage, and joint refinement of two layouts.
//
// Citations: P:<line> = /root/reference/PAPER.md.
#include <algorithm>
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <unordered_map>

#include "common.hpp"

namespace axe {

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}
const char *last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- axes
namespace {
std::mutex g_axis_mu;
std::vector<std::unique_ptr<std::string>> g_axis_names;
std::unordered_map<std::string, int> g_axis_ids;
}  // namespace

bool valid_axis_name(const char *a) {
  if (!a || !a[0]) return false;
  auto alpha = [](char c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_'; };
  if (!alpha(a[0])) return false;
  for (const char *p = a + 1; *p; p++)
    if (!alpha(*p) && !(*p >= '0' && *p <= '9')) return false;
  return strlen(a) < 64;
}

int intern_axis(const char *name) {
  if (!valid_axis_name(name)) return -1;
  std::lock_guard<std::mutex> lk(g_axis_mu);
  auto it = g_axis_ids.find(name);
  if (it != g_axis_ids.end()) return it->second;
  int id = (int)g_axis_names.size();
  g_axis_names.emplace_back(new std::string(name));
  g_axis_ids.emplace(*g_axis_names.back(), id);
  return id;
}

const char *axis_name(int id) {
  std::lock_guard<std::mutex> lk(g_axis_mu);
  return (id >= 0 && id < (int)g_axis_names.size()) ? g_axis_names[id]->c_str() : "?";
}

int axis_m() {
  static int id = intern_axis("m");
  return id;
}
int axis_gpuid() {
  static int id = intern_axis("gpuid");
  return id;
}

// ---------------------------------------------------------------- layouts
axe_status make_layout(std::vector<Iter> D, std::vector<Iter> R, std::vector<std::pair<int, int64_t>> O,
                       Layout *out) {
  // Def. Iter: e > 0, s != 0; Def. Layout: n_D >= 1.
  if (D.empty()) AXE_FAIL(AXE_ERR_INVALID_ARG, "layout needs at least one shard iter (n_D >= 1, P:237)");
  Layout L;
  auto add_axis = [&](int a) {
    if (std::find(L.axes.begin(), L.axes.end(), a) == L.axes.end()) L.axes.push_back(a);
  };
  for (auto *lst : {&D, &R})
    for (auto &it : *lst) {
      if (it.e < 1) AXE_FAIL(AXE_ERR_INVALID_ARG, "iter extent %lld < 1 (Def. Iter, P:233)", (long long)it.e);
      if (it.s == 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "iter stride 0 (Def. Iter requires s != 0, P:233)");
      if (it.a < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad axis name");
      add_axis(it.a);
    }
  for (auto &it : D)
    if (__builtin_mul_overflow(L.ED, it.e, &L.ED)) AXE_FAIL(AXE_ERR_OVERFLOW, "E_D overflows int64");
  for (auto &it : R)
    if (__builtin_mul_overflow(L.ER, it.e, &L.ER)) AXE_FAIL(AXE_ERR_OVERFLOW, "E_R overflows int64");
  // merge repeated offset axes, drop zeros (sparse Z^A)
  for (auto &p : O) {
    if (p.first < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad offset axis name");
    bool found = false;
    for (auto &q : L.O)
      if (q.first == p.first) {
        if (__builtin_add_overflow(q.second, p.second, &q.second)) AXE_FAIL(AXE_ERR_OVERFLOW, "offset overflow");
        found = true;
      }
    if (!found) L.O.push_back(p);
  }
  L.O.erase(std::remove_if(L.O.begin(), L.O.end(), [](auto &p) { return p.second == 0; }), L.O.end());
  for (auto &p : O) add_axis(p.first);
  // every coordinate must be representable: |O_a| + sum (e-1)|s| fits int64
  for (int a : L.axes) {
    int64_t acc = L.offset(a);
    acc = acc < 0 ? -acc : acc;
    for (auto *lst : {&D, &R})
      for (auto &it : *lst) {
        if (it.a != a) continue;
        int64_t t, as = it.s < 0 ? -it.s : it.s;
        if (__builtin_mul_overflow(it.e - 1, as, &t) || __builtin_add_overflow(acc, t, &acc))
          AXE_FAIL(AXE_ERR_OVERFLOW, "coordinate range of axis %s overflows int64", axis_name(a));
      }
  }
  L.D = std::move(D);
  L.R = std::move(R);
  *out = std::move(L);
  return AXE_OK;
}

void eval_layout(const Layout &L, int64_t x, int64_t *rows) {
  const int na = (int)L.axes.size();
  auto slot = [&](int a) {
    for (int i = 0; i < na; i++)
      if (L.axes[i] == a) return i;
    return -1;
  };
  std::vector<int64_t> base(na, 0);
  int64_t rem = x;  // lexicographic unflattening, last iter fastest
  for (int i = (int)L.D.size() - 1; i >= 0; i--) {
    int64_t d = rem % L.D[i].e;
    rem /= L.D[i].e;
    base[slot(L.D[i].a)] += d * L.D[i].s;
  }
  for (auto &p : L.O) base[slot(p.first)] += p.second;
  for (int64_t r = 0; r < L.ER; r++) {
    int64_t *row = rows + r * na;
    for (int i = 0; i < na; i++) row[i] = base[i];
    int64_t rr = r;
    for (int t = (int)L.R.size() - 1; t >= 0; t--) {
      int64_t d = rr % L.R[t].e;
      rr /= L.R[t].e;
      row[slot(L.R[t].a)] += d * L.R[t].s;
    }
  }
}

void axis_bounds(const Layout &L, int a, int64_t *mn, int64_t *mx) {
  // Lemma span-closed, signed: digits are independent, so the
  // extremes are attained digit by digit.
  int64_t lo = L.offset(a), hi = lo;
  for (auto *lst : {&L.D, &L.R})
    for (auto &it : *lst)
      if (it.a == a) {
        int64_t t = (it.e - 1) * it.s;
        if (t < 0) lo += t;
        else hi += t;
      }
  *mn = lo;
  *mx = hi;
}

std::vector<Iter> normalize_shard(const std::vector<Iter> &D) {
  // D0: drop unit extents; D1: merge (e_i, s_i, a), (e_{i+1}, s_{i+1}, a) when
  // s_i = e_{i+1} s_{i+1} (App. A.1).  One left-to-right pass with a
  // stack reaches the fixpoint because merging never enables an earlier merge
  // that was not already checked against the merged iter.
  std::vector<Iter> out;
  for (auto it : D) {
    if (it.e == 1) continue;
    out.push_back(it);
    while (out.size() >= 2) {
      Iter &p = out[out.size() - 2], &q = out.back();
      if (p.a == q.a && p.s == q.e * q.s) {
        Iter m{p.e * q.e, q.s, q.a};
        out.pop_back();
        out.back() = m;
      } else {
        break;
      }
    }
  }
  if (out.empty()) out.push_back(Iter{1, 1, axis_m()});
  return out;
}

Layout canonicalize(const Layout &L, bool *gap_ok) {
  Layout C;
  std::vector<Iter> D = normalize_shard(L.D);
  std::vector<std::pair<int, int64_t>> O = L.O;
  auto addO = [&](int a, int64_t v) {
    for (auto &p : O)
      if (p.first == a) {
        p.second += v;
        return;
      }
    O.push_back({a, v});
  };
  std::vector<Iter> R;
  for (auto it : L.R) {
    if (it.e == 1) continue;                  // C0
    if (it.s < 0) {                           // C1: O += (e-1) s, s <- -s
      addO(it.a, (it.e - 1) * it.s);
      it.s = -it.s;
    }
    R.push_back(it);
  }
  // C2: absorb (E2, q s) into (E1, s) when 1 <= q <= E1 (reading R9), same axis.
  bool changed = true;
  while (changed) {
    changed = false;
    for (size_t i = 0; i < R.size() && !changed; i++)
      for (size_t j = 0; j < R.size() && !changed; j++) {
        if (i == j || R[i].a != R[j].a || R[j].s % R[i].s != 0) continue;
        int64_t q = R[j].s / R[i].s;
        if (q < 1 || q > R[i].e) continue;
        if (q == 1 && j < i) continue;        // equal strides: merge the later into the earlier
        R[i].e = R[i].e + q * (R[j].e - 1);
        R.erase(R.begin() + j);
        changed = true;
      }
  }
  std::sort(R.begin(), R.end(), [](const Iter &x, const Iter &y) {
    int c = strcmp(axis_name(x.a), axis_name(y.a));
    return c != 0 ? c < 0 : x.s < y.s;
  });
  // gap condition GC: sigma_{k+1} > E_k sigma_k per axis
  bool gc = true;
  for (size_t i = 0; i + 1 < R.size(); i++)
    if (R[i].a == R[i + 1].a && !(R[i + 1].s > R[i].e * R[i].s)) gc = false;
  if (gap_ok) *gap_ok = gc;
  make_layout(D, R, O, &C);
  // keep the axis order of the input where possible
  std::vector<int> ax;
  for (int a : L.axes)
    if (C.names_axis(a)) ax.push_back(a);
  for (int a : C.axes)
    if (std::find(ax.begin(), ax.end(), a) == ax.end()) ax.push_back(a);
  C.axes = ax;
  return C;
}

std::string layout_key(const Layout &L) {
  std::string k;
  char b[96];
  for (auto &i : L.D) {
    snprintf(b, sizeof b, "(%lld,%lld,%d)", (long long)i.e, (long long)i.s, i.a);
    k += b;
  }
  k += "|";
  for (auto &i : L.R) {
    snprintf(b, sizeof b, "(%lld,%lld,%d)", (long long)i.e, (long long)i.s, i.a);
    k += b;
  }
  k += "|";
  for (auto &p : L.O) {
    snprintf(b, sizeof b, "%d:%lld,", p.first, (long long)p.second);
    k += b;
  }
  return k;
}

// ---------------------------------------------------------------- storage
axe_status make_storage(const axe_storage *st, Storage *out) {
  if (!st || st->n < 1 || !st->digits) AXE_FAIL(AXE_ERR_INVALID_ARG, "storage needs >= 1 digit");
  Storage S;
  for (int k = 0; k < st->n; k++) {
    const axe_storage_digit &g = st->digits[k];
    int a = intern_axis(g.axis ? g.axis : "m");
    if (a < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad storage axis name");
    if (g.extent < 1 || g.divisor < 1) AXE_FAIL(AXE_ERR_INVALID_ARG, "storage digit extent/divisor < 1");
    S.d.push_back(SDigit{a, g.extent, g.divisor, 0});
  }
  for (int k = (int)S.d.size() - 1; k >= 0; k--) {
    S.d[k].mult = S.cells;
    if (__builtin_mul_overflow(S.cells, S.d[k].ext, &S.cells)) AXE_FAIL(AXE_ERR_OVERFLOW, "storage size overflow");
  }
  // chain condition per axis (R17): div_k = ext_k' * div_k' for the next inner digit k'
  for (size_t k = 0; k < S.d.size(); k++) {
    int next = -1;
    for (size_t j = k + 1; j < S.d.size(); j++)
      if (S.d[j].a == S.d[k].a) {
        next = (int)j;
        break;
      }
    if (next < 0 ? S.d[k].div != 1 : S.d[k].div != S.d[next].ext * S.d[next].div)
      AXE_FAIL(AXE_ERR_INVALID_ARG, "storage digits of axis %s do not form a divisor chain", axis_name(S.d[k].a));
  }
  S.swz_b = st->swz_bits;
  S.swz_m = st->swz_base;
  S.swz_s = st->swz_shift;
  if (S.swz_b < 0 || S.swz_m < 0 || S.swz_s < 0 || S.swz_b + S.swz_m + S.swz_s > 40 ||
      (S.swz_b > 0 && S.swz_s < S.swz_b))
    AXE_FAIL(AXE_ERR_INVALID_ARG, "bad swizzle (B=%d, M=%d, S=%d)", S.swz_b, S.swz_m, S.swz_s);
  *out = std::move(S);
  return AXE_OK;
}

std::string storage_key(const Storage &s) {
  std::string k;
  char b[96];
  for (auto &d : s.d) {
    snprintf(b, sizeof b, "[%d,%lld,%lld]", d.a, (long long)d.ext, (long long)d.div);
    k += b;
  }
  snprintf(b, sizeof b, "sw%d.%d.%d", s.swz_b, s.swz_m, s.swz_s);
  return k + b;
}

// ---------------------------------------------------------------- composition
// Compose L with its storage into element-index strides.  Each iter (e, s, a)
// is split (Lemma split) so every piece lands in one storage
// digit of axis a; the result is exact iff, per storage digit, the offset's
// digit plus every piece's contribution stays inside [0, ext) (no carries).
bool compose_linear(const Layout &L, const Storage &st, int skip_axis, Linear *out, bool keep_dev) {
  Linear lin;
  struct Piece {
    int64_t e, t;  // extent, coefficient in storage-digit units
    int k;         // storage digit
  };
  // per storage digit: [lo, hi] range of contributions
  std::vector<int64_t> lo(st.d.size(), 0), hi(st.d.size(), 0);
  auto split = [&](const Iter &it, std::vector<Piece> &inner_first) -> bool {
    int64_t cur_e = it.e, u = it.s < 0 ? -it.s : it.s, sg = it.s < 0 ? -1 : 1;
    while (cur_e > 1) {
      int k = -1;
      for (size_t j = 0; j < st.d.size(); j++)
        if (st.d[j].a == it.a && st.d[j].div <= u && u / st.d[j].ext < st.d[j].div) {
          k = (int)j;
          break;
        }
      if (k < 0) return false;
      const SDigit &g = st.d[k];
      if (u % g.div) return false;
      int64_t cap = g.div * g.ext;
      if ((cur_e - 1) <= (cap - 1) / u) {  // (cur_e-1) * u < cap
        inner_first.push_back(Piece{cur_e, sg * (u / g.div), k});
        break;
      }
      if (cap % u) return false;
      int64_t gsz = cap / u;
      if (gsz <= 1 || cur_e % gsz) return false;
      inner_first.push_back(Piece{gsz, sg * (u / g.div), k});
      cur_e /= gsz;
      u = cap;
    }
    return true;
  };
  auto emit = [&](const std::vector<Iter> &src, std::vector<LinIter> &dst) -> bool {
    for (auto &it : src) {
      if (it.e == 1) continue;
      if (it.a == skip_axis) {
        if (keep_dev) dst.push_back(LinIter{it.e, it.s, 1});
        continue;
      }
      if (!st.binds(it.a)) return false;
      std::vector<Piece> pcs;
      if (!split(it, pcs)) return false;
      for (auto p = pcs.rbegin(); p != pcs.rend(); ++p) {
        int64_t t = (p->e - 1) * p->t;
        if (t < 0) lo[p->k] += t;
        else hi[p->k] += t;
        dst.push_back(LinIter{p->e, p->t * st.d[p->k].mult});
      }
    }
    return true;
  };
  if (!emit(L.D, lin.D) || !emit(L.R, lin.R)) return false;
  // offset digits and the carry-free check
  for (size_t k = 0; k < st.d.size(); k++) {
    const SDigit &g = st.d[k];
    int64_t o = L.offset(g.a);
    if (g.a == skip_axis) continue;
    if (o < 0) return false;
    int64_t ok = (o / g.div) % g.ext;
    bool outermost = true;
    for (size_t j = 0; j < k; j++)
      if (st.d[j].a == g.a) outermost = false;
    if (outermost && o / g.div >= g.ext) return false;
    if (ok + lo[k] < 0 || ok + hi[k] >= g.ext) return false;
    lin.base += ok * g.mult;
  }
  for (auto &p : L.O)
    if (p.first != skip_axis && !st.binds(p.first)) return false;
  if (skip_axis >= 0) lin.dev_base = L.offset(skip_axis);
  *out = std::move(lin);
  return true;
}

// ---------------------------------------------------------------- joint refinement
static std::vector<LinIter> normalize_lin(const std::vector<LinIter> &D) {
  std::vector<LinIter> out;
  for (auto it : D) {
    if (it.e == 1) continue;
    out.push_back(it);
    while (out.size() >= 2) {
      LinIter &p = out[out.size() - 2], &q = out.back();
      if (p.dev == q.dev && p.s == q.e * q.s) {
        LinIter m{p.e * q.e, q.s, q.dev};
        out.pop_back();
        out.back() = m;
      } else {
        break;
      }
    }
  }
  return out;
}

bool joint_refine(const std::vector<LinIter> &src_in, const std::vector<LinIter> &dst_in, std::vector<Joint> *out) {
  // Both lists unflatten the same x lexicographically (last fastest).
  // Pair them from the fastest digit: if one extent divides the other, split
  // the larger (Lemma split) and emit a joint digit.  If neither
  // divides the other the two digit systems are not nested and no common
  // refinement exists (Alg. 1 fails with gcd = 1 in the same situation).
  std::vector<LinIter> a = normalize_lin(src_in), b = normalize_lin(dst_in);
  std::vector<Joint> J;
  while (!a.empty() && !b.empty()) {
    LinIter &x = a.back(), &y = b.back();
    if (x.e == y.e) {
      J.push_back(Joint{x.e, x.s, y.s, x.dev, y.dev});
      a.pop_back();
      b.pop_back();
    } else if (x.e % y.e == 0) {
      J.push_back(Joint{y.e, x.s, y.s, x.dev, y.dev});
      x = LinIter{x.e / y.e, x.s * y.e, x.dev};
      b.pop_back();
    } else if (y.e % x.e == 0) {
      J.push_back(Joint{x.e, x.s, y.s, x.dev, y.dev});
      y = LinIter{y.e / x.e, y.s * x.e, y.dev};
      a.pop_back();
    } else {
      return false;
    }
  }
  if (!a.empty() || !b.empty()) return false;
  std::reverse(J.begin(), J.end());
  // joint D1: fuse neighbours that are contiguous on both sides (Cor. fuse)
  std::vector<Joint> F;
  for (auto &j : J) {
    F.push_back(j);
    while (F.size() >= 2) {
      Joint &p = F[F.size() - 2], &q = F.back();
      if (p.sdev == q.sdev && p.ddev == q.ddev && p.ss == q.e * q.ss && p.ds == q.e * q.ds) {
        Joint m{p.e * q.e, q.ss, q.ds, q.sdev, q.ddev};
        F.pop_back();
        F.back() = m;
      } else {
        break;
      }
    }
  }
  if (F.empty()) F.push_back(Joint{1, 1, 1});
  *out = std::move(F);
  return true;
}

bool joint_refine_partial(const std::vector<LinIter> &src_in, const std::vector<LinIter> &dst_in,
                          std::vector<Joint> *inner, std::vector<LinIter> *src_rest, std::vector<LinIter> *dst_rest) {
  std::vector<LinIter> a = normalize_lin(src_in), b = normalize_lin(dst_in);
  std::vector<Joint> J;
  while (!a.empty() && !b.empty()) {
    LinIter &x = a.back(), &y = b.back();
    if (x.e == y.e) {
      J.push_back(Joint{x.e, x.s, y.s, x.dev, y.dev});
      a.pop_back();
      b.pop_back();
    } else if (x.e % y.e == 0) {
      J.push_back(Joint{y.e, x.s, y.s, x.dev, y.dev});
      x = LinIter{x.e / y.e, x.s * y.e, x.dev};
      b.pop_back();
    } else if (y.e % x.e == 0) {
      J.push_back(Joint{x.e, x.s, y.s, x.dev, y.dev});
      y = LinIter{y.e / x.e, y.s * x.e, y.dev};
      a.pop_back();
    } else {
      const int64_t g = std::gcd(x.e, y.e);
      if (g > 1) {
        J.push_back(Joint{g, x.s, y.s, x.dev, y.dev});
        x = LinIter{x.e / g, x.s * g, x.dev};
        y = LinIter{y.e / g, y.s * g, y.dev};
      }
      break;
    }
  }
  std::reverse(J.begin(), J.end());
  std::vector<Joint> F;  // joint D1 (Cor. fuse)
  for (auto &j : J) {
    F.push_back(j);
    while (F.size() >= 2) {
      Joint &p = F[F.size() - 2], &q = F.back();
      if (p.sdev == q.sdev && p.ddev == q.ddev && p.ss == q.e * q.ss && p.ds == q.e * q.ds) {
        Joint m{p.e * q.e, q.ss, q.ds, q.sdev, q.ddev};
        F.pop_back();
        F.back() = m;
      } else {
        break;
      }
    }
  }
  *inner = std::move(F);
  *src_rest = a;
  *dst_rest = b;
  return true;
}

}  // namespace axe
