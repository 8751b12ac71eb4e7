// text.cpp -- the textual / structured surface of layouts:
// parse and format the paper's matrix notation "(e0,e1):(s0@a0,s1@a1) +
// [(r):(t@b)] + o@c" (Figures 2 and 5; the axis m is the default),
// JSON rendering, and canonical equivalence (§3.3 "Canonicalize ... verify if
// they represent the same induced function"; App. A uniqueness under the gap
// condition).
#include <algorithm>
#include <cctype>
#include <cstring>
#include <map>
#include <set>
#include <string>

#include "handles.hpp"

namespace axe {
namespace {

struct Parser {
  const char *s;
  size_t i = 0;
  std::string err;
  size_t err_pos = 0;

  void ws() {
    while (s[i] && isspace((unsigned char)s[i])) i++;
  }
  bool fail(const char *m) {
    if (err.empty()) {
      err = m;
      err_pos = i;
    }
    return false;
  }
  bool eat(char c) {
    ws();
    if (s[i] == c) {
      i++;
      return true;
    }
    return false;
  }
  bool expect(char c) {
    if (eat(c)) return true;
    char m[48];
    snprintf(m, sizeof m, "expected '%c'", c);
    return fail(m);
  }
  bool integer(int64_t *v) {
    ws();
    size_t j = i;
    bool neg = false;
    if (s[j] == '-' || s[j] == '+') neg = s[j++] == '-';
    if (!isdigit((unsigned char)s[j])) return fail("expected an integer");
    __int128 x = 0;
    while (isdigit((unsigned char)s[j])) {
      x = x * 10 + (s[j++] - '0');
      if (x > (__int128)INT64_MAX) return fail("integer out of int64 range");
    }
    i = j;
    *v = (int64_t)(neg ? -x : x);
    return true;
  }
  bool axis(int *a) {
    ws();
    size_t j = i;
    if (!(isalpha((unsigned char)s[j]) || s[j] == '_')) return fail("expected an axis name");
    while (isalnum((unsigned char)s[j]) || s[j] == '_') j++;
    std::string name(s + i, j - i);
    *a = intern_axis(name.c_str());
    if (*a < 0) return fail("bad axis name");
    i = j;
    return true;
  }
  // "(" INT ("," INT)* "):(" stride ("," stride)* ")"
  bool iters(std::vector<Iter> *out) {
    std::vector<int64_t> ext;
    if (!expect('(')) return false;
    do {
      int64_t e;
      if (!integer(&e)) return false;
      ext.push_back(e);
    } while (eat(','));
    if (!expect(')') || !expect(':') || !expect('(')) return false;
    size_t k = 0;
    do {
      int64_t st;
      int a = axis_m();
      if (!integer(&st)) return false;
      if (eat('@') && !axis(&a)) return false;
      if (k >= ext.size()) return fail("more strides than extents");
      out->push_back(Iter{ext[k], st, a});
      k++;
    } while (eat(','));
    if (k != ext.size()) return fail("fewer strides than extents");
    return expect(')');
  }
};

std::string fmt_iters(const std::vector<Iter> &v) {
  std::string a = "(", b = "(";
  for (size_t k = 0; k < v.size(); k++) {
    a += (k ? "," : "") + std::to_string(v[k].e);
    b += (k ? "," : "") + std::to_string(v[k].s);
    if (v[k].a != axis_m()) b += std::string("@") + axis_name(v[k].a);
  }
  return a + "):" + b + ")";
}

std::string format_layout(const Layout &L) {
  std::string s = fmt_iters(L.D);
  if (!L.R.empty()) s += " + [" + fmt_iters(L.R) + "]";
  for (auto &o : L.O) s += " + " + std::to_string(o.second) + "@" + axis_name(o.first);
  return s;
}

std::string json_iters(const std::vector<Iter> &v) {
  std::string s = "[";
  for (size_t k = 0; k < v.size(); k++)
    s += (k ? "," : "") + std::string("[") + std::to_string(v[k].e) + "," + std::to_string(v[k].s) + ",\"" +
         axis_name(v[k].a) + "\"]";
  return s + "]";
}

axe_status put(const std::string &s, char *buf, int capacity) {
  if (!buf) AXE_FAIL(AXE_ERR_INVALID_ARG, "buf is NULL");
  if ((int64_t)s.size() + 1 > capacity) AXE_FAIL(AXE_ERR_CAPACITY, "need %d bytes", (int)s.size() + 1);
  memcpy(buf, s.c_str(), s.size() + 1);
  return AXE_OK;
}

// replica iters per axis sorted by (stride, extent): R is a multiset (App. A Theorem proof)
std::map<int, std::vector<std::pair<int64_t, int64_t>>> replica_key(const Layout &L) {
  std::map<int, std::vector<std::pair<int64_t, int64_t>>> m;
  for (auto &r : L.R) m[r.a].push_back({r.s, r.e});
  for (auto &kv : m) std::sort(kv.second.begin(), kv.second.end());
  return m;
}

std::map<int, int64_t> offset_key(const Layout &L) {
  std::map<int, int64_t> m;
  for (auto &o : L.O)
    if (o.second) m[o.first] += o.second;
  return m;
}

}  // namespace
}  // namespace axe

using namespace axe;

extern "C" {

axe_status axe_layout_parse(const char *text, axe_layout **out, int *error_pos) {
  if (!text || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (error_pos) *error_pos = -1;
  Parser p{text};
  std::vector<Iter> D, R;
  std::vector<std::pair<int, int64_t>> O;
  bool ok = p.iters(&D);
  bool seen_replica = false;
  while (ok && p.eat('+')) {
    p.ws();
    if (p.s[p.i] == '[') {
      if (seen_replica || !O.empty()) {
        ok = p.fail("the replica term comes once, before the offsets");
        break;
      }
      p.i++;
      ok = p.iters(&R) && p.expect(']');
      seen_replica = true;
    } else {
      int64_t v;
      int a;
      ok = p.integer(&v) && p.expect('@') && p.axis(&a);
      if (ok) O.push_back({a, v});
    }
  }
  if (ok) {
    p.ws();
    if (p.s[p.i]) ok = p.fail("trailing characters");
  }
  if (!ok) {
    if (error_pos) *error_pos = (int)p.err_pos;
    AXE_FAIL(AXE_ERR_INVALID_ARG, "parse error at %zu: %s", p.err_pos, p.err.c_str());
  }
  auto *h = new axe_layout;
  axe_status st = make_layout(std::move(D), std::move(R), std::move(O), &h->L);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *out = h;
  return AXE_OK;
}

axe_status axe_layout_format(const axe_layout *layout, char *buf, int capacity) {
  if (!layout) AXE_FAIL(AXE_ERR_INVALID_ARG, "layout is NULL");
  return put(format_layout(layout->L), buf, capacity);
}

axe_status axe_layout_to_json(const axe_layout *layout, char *buf, int capacity) {
  if (!layout) AXE_FAIL(AXE_ERR_INVALID_ARG, "layout is NULL");
  const Layout &L = layout->L;
  std::string s = "{\"schema_version\":1,\"shard\":" + json_iters(L.D) + ",\"replica\":" + json_iters(L.R) +
                  ",\"offset\":{";
  for (size_t k = 0; k < L.O.size(); k++)
    s += (k ? ",\"" : "\"") + std::string(axis_name(L.O[k].first)) + "\":" + std::to_string(L.O[k].second);
  s += "},\"E_D\":" + std::to_string(L.ED) + ",\"E_R\":" + std::to_string(L.ER) + ",\"text\":\"" + format_layout(L) +
       "\"}";
  return put(s, buf, capacity);
}

axe_status axe_layout_equivalent(const axe_layout *a, const axe_layout *b, int64_t threshold, int *result) {
  if (!a || !b || !result) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  if (threshold < 0) threshold = 65536;
  *result = 0;
  if (a->L.ED != b->L.ED) return AXE_OK;  // different logical domains
  bool ga = true, gb = true;
  const Layout ca = canonicalize(a->L, &ga), cb = canonicalize(b->L, &gb);
  if (ga && gb) {  // canonical forms are unique under GC (App. A): compare structurally
    bool same = ca.D.size() == cb.D.size();
    for (size_t k = 0; same && k < ca.D.size(); k++)
      same = ca.D[k].e == cb.D[k].e && ca.D[k].s == cb.D[k].s && ca.D[k].a == cb.D[k].a;
    same = same && replica_key(ca) == replica_key(cb) && offset_key(ca) == offset_key(cb);
    *result = same ? 1 : 0;
    return AXE_OK;
  }
  // no uniqueness guarantee: compare the induced maps pointwise as sets, if small enough
  if (a->L.ED * std::max(a->L.ER, b->L.ER) > threshold) {
    *result = -1;
    return AXE_OK;
  }
  std::set<int> axes(a->L.axes.begin(), a->L.axes.end());
  axes.insert(b->L.axes.begin(), b->L.axes.end());
  auto image = [&](const Layout &L, int64_t x) {
    std::vector<int64_t> rows(L.ER * L.axes.size());
    eval_layout(L, x, rows.data());
    std::set<std::vector<int64_t>> img;
    for (int64_t r = 0; r < L.ER; r++) {
      std::vector<int64_t> c;
      for (int ax : axes) {
        int64_t v = 0;
        for (size_t i = 0; i < L.axes.size(); i++)
          if (L.axes[i] == ax) v = rows[r * L.axes.size() + i];
        c.push_back(v);
      }
      img.insert(c);
    }
    return img;
  };
  for (int64_t x = 0; x < a->L.ED; x++)
    if (image(a->L, x) != image(b->L, x)) return AXE_OK;
  *result = 1;
  return AXE_OK;
}

}  // extern "C"
