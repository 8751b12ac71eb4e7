// plan.cpp -- copy planning: validation, storage composition, joint digits,
// kernel selection and parameter-table emission.
#include "plan.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <set>
#include <mutex>
#include <thread>
#include <unordered_map>

namespace axe {

axe_status check_side(const Layout &L, const Storage &st, int skip_axis, const char *which) {
  if (skip_axis < 0 && L.names_axis(axis_gpuid()))
    AXE_FAIL(AXE_ERR_UNSUPPORTED_AXIS, "%s layout names the device axis gpuid; use axe_redistribute", which);
  for (int a : L.axes) {
    if (a == skip_axis) continue;
    int64_t mn, mx;
    axis_bounds(L, a, &mn, &mx);
    if (!st.binds(a)) {
      if (mn != 0 || mx != 0)
        AXE_FAIL(AXE_ERR_UNSUPPORTED_AXIS, "%s layout uses axis %s, which its storage does not bind", which,
                 axis_name(a));
      continue;
    }
    int64_t top = st.top(a);
    if (mn < 0 || mx >= top)
      AXE_FAIL(AXE_ERR_BOUNDS, "%s layout reaches %s in [%lld, %lld], outside the storage box [0, %lld)", which,
               axis_name(a), (long long)mn, (long long)mx, (long long)top);
  }
  if (st.swz_b > 0) {
    // the swizzle permutes bytes inside 2^(B+M+S)-byte blocks; the buffer must hold whole blocks
    (void)0;
  }
  return AXE_OK;
}

// Destination injectivity (reading R6): different x never share a cell.
axe_status check_injective(const Layout &dst, const Storage &st, int skip_axis) {
  Linear lin;
  if (skip_axis < 0 && compose_linear(dst, st, skip_axis, &lin)) {
    // fast sufficient test: sorted by |s|, each stride exceeds the reach of all
    // smaller digits (cumulative separation, Lemma cum.)
    std::vector<LinIter> all = lin.D;
    all.insert(all.end(), lin.R.begin(), lin.R.end());
    std::sort(all.begin(), all.end(), [](const LinIter &a, const LinIter &b) {
      return (a.s < 0 ? -a.s : a.s) < (b.s < 0 ? -b.s : b.s);
    });
    bool ok = true;
    int64_t reach = 0;
    for (auto &it : all) {
      int64_t u = it.s < 0 ? -it.s : it.s;
      if (u <= reach) {
        ok = false;
        break;
      }
      reach += (it.e - 1) * u;
    }
    if (ok) return AXE_OK;
    // exact: enumerate every (x, r) on the element index (odometer), bitmap of cells
    int64_t work = dst.ED * dst.ER;
    if (work > (int64_t(1) << 28) || st.cells > (int64_t(1) << 34))
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "cannot verify destination injectivity (E_D*E_R = %lld too large)",
               (long long)work);
    std::vector<uint64_t> seen((size_t)(st.cells / 64 + 1), 0);
    std::vector<int64_t> reps{0};
    for (auto &r : lin.R) {
      std::vector<int64_t> nx;
      for (int64_t base : reps)
        for (int64_t d = 0; d < r.e; d++) nx.push_back(base + d * r.s);
      reps.swap(nx);
    }
    std::sort(reps.begin(), reps.end());
    reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
    std::vector<int64_t> dig(lin.D.size(), 0);
    int64_t off = lin.base;
    for (int64_t x = 0; x < dst.ED; x++) {
      for (int64_t r : reps) {
        int64_t c = off + r;
        uint64_t m = uint64_t(1) << (c & 63);
        if (seen[c >> 6] & m)
          AXE_FAIL(AXE_ERR_NONINJECTIVE, "destination layout writes element %lld twice (x = %lld)", (long long)c,
                   (long long)x);
        seen[c >> 6] |= m;
      }
      for (int k = (int)lin.D.size() - 1; k >= 0; k--) {  // odometer step
        off += lin.D[k].s;
        if (++dig[k] < lin.D[k].e) break;
        off -= lin.D[k].e * lin.D[k].s;
        dig[k] = 0;
      }
    }
    return AXE_OK;
  }
  // non-affine composition: evaluate every (x, r) on the host
  int64_t work = dst.ED * dst.ER;
  if (work > (int64_t(1) << 24))
    AXE_FAIL(AXE_ERR_UNSUPPORTED, "cannot verify destination injectivity of a non-affine layout (E_D*E_R = %lld)",
             (long long)work);
  const int na = (int)dst.axes.size();
  std::vector<int64_t> rows((size_t)(dst.ER * na));
  std::vector<uint64_t> seen((size_t)(st.cells / 64 + 1), 0);
  std::vector<int> slot(st.d.size(), -1);
  for (size_t k = 0; k < st.d.size(); k++)
    for (int i = 0; i < na; i++)
      if (dst.axes[i] == st.d[k].a) slot[k] = i;
  for (int64_t x = 0; x < dst.ED; x++) {
    eval_layout(dst, x, rows.data());
    std::vector<int64_t> cells;
    for (int64_t r = 0; r < dst.ER; r++) {
      int64_t idx = 0;
      for (size_t k = 0; k < st.d.size(); k++) {
        int64_t v = slot[k] >= 0 ? rows[r * na + slot[k]] : 0;
        idx = idx * st.d[k].ext + (v / st.d[k].div) % st.d[k].ext;
      }
      cells.push_back(idx);
    }
    std::sort(cells.begin(), cells.end());
    cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
    for (int64_t c : cells) {
      uint64_t m = uint64_t(1) << (c & 63);
      if (seen[c >> 6] & m)
        AXE_FAIL(AXE_ERR_NONINJECTIVE, "destination layout writes element %lld twice (x = %lld)", (long long)c,
                 (long long)x);
      seen[c >> 6] |= m;
    }
  }
  return AXE_OK;
}

Swz make_swz(const Storage &st) {
  Swz s;
  s.shift = (uint32_t)(st.swz_m + st.swz_s);
  s.mask = st.swz_b > 0 ? (uint32_t)((1u << st.swz_b) - 1) : 0u;
  s.base = (uint32_t)st.swz_m;
  return s;
}

axe_status build_k0_side(const Layout &L, const Storage &st, int skip_axis, K0Side *S) {
  memset(S, 0, sizeof(*S));
  std::vector<int> ax;
  for (int a : L.axes)
    if (a != skip_axis) ax.push_back(a);
  if ((int)ax.size() > K0_MAXAX) AXE_FAIL(AXE_ERR_UNSUPPORTED, "generic kernel supports <= %d axes", K0_MAXAX);
  auto slot = [&](int a) {
    for (size_t i = 0; i < ax.size(); i++)
      if (ax[i] == a) return (int)i;
    return -1;
  };
  S->nax = (int)ax.size();
  for (auto &it : L.D) {
    if (it.a == skip_axis) continue;
    if (S->nD == K0_MAXI) AXE_FAIL(AXE_ERR_UNSUPPORTED, "generic kernel supports <= %d shard iters", K0_MAXI);
    S->e[S->nD] = it.e;
    S->s[S->nD] = it.s;
    S->ax[S->nD] = (int8_t)slot(it.a);
    S->nD++;
  }
  // skipped-axis iters still take part in the unflattening: keep them with stride 0 on a dummy slot
  if (skip_axis >= 0) {
    S->nD = 0;
    for (auto &it : L.D) {
      if (S->nD == K0_MAXI) AXE_FAIL(AXE_ERR_UNSUPPORTED, "generic kernel supports <= %d shard iters", K0_MAXI);
      bool sk = it.a == skip_axis;
      S->e[S->nD] = it.e;
      S->s[S->nD] = sk ? 0 : it.s;
      S->ax[S->nD] = (int8_t)(sk ? 0 : slot(it.a));
      S->nD++;
    }
  }
  for (auto &it : L.R) {
    if (S->nR == K0_MAXI) AXE_FAIL(AXE_ERR_UNSUPPORTED, "generic kernel supports <= %d replica iters", K0_MAXI);
    bool sk = it.a == skip_axis;
    S->re[S->nR] = it.e;
    S->rs[S->nR] = sk ? 0 : it.s;
    S->rax[S->nR] = (int8_t)(sk ? 0 : slot(it.a));
    S->nR++;
  }
  for (auto &p : L.O)
    if (p.first != skip_axis) S->off[slot(p.first)] = p.second;
  if ((int)st.d.size() > K0_MAXSD) AXE_FAIL(AXE_ERR_UNSUPPORTED, "generic kernel supports <= %d storage digits", K0_MAXSD);
  S->nsd = (int)st.d.size();
  for (size_t k = 0; k < st.d.size(); k++) {
    S->sax[k] = (int8_t)slot(st.d[k].a);
    S->sext[k] = st.d[k].ext;
    S->sdiv[k] = st.d[k].div;
  }
  S->sw = make_swz(st);
  return AXE_OK;
}

std::string joint_json(const std::vector<Joint> &J) {
  std::string s = "[";
  char b[96];
  for (size_t i = 0; i < J.size(); i++) {
    snprintf(b, sizeof b, "%s[%lld,%lld,%lld]", i ? "," : "", (long long)J[i].e, (long long)J[i].ss,
             (long long)J[i].ds);
    s += b;
  }
  return s + "]";
}

static int64_t env_int(const char *name, int64_t dflt) {
  const char *e = getenv(name);
  return (e && *e) ? atoll(e) : dflt;
}

int64_t grid_cap(int64_t per_sm) {
  if (env_int("AXE_ONESHOT", 0)) return (int64_t(1) << 31) - 1;
  return (int64_t)num_sms() * per_sm;
}

// The in-order schedule (unit_range in kernels.cuh): `chunk` consecutive units per CTA and a grid that
// covers them all; 0 keeps the persistent grid.  AXE_CHUNK overrides the schedule's default.
uint32_t unit_chunk(int64_t dflt) { return (uint32_t)std::max<int64_t>(0, env_int("AXE_CHUNK", dflt)); }

unsigned chunk_grid(int64_t units, uint32_t chunk, unsigned persistent) {
  if (!chunk) return persistent;
  return (unsigned)std::max<int64_t>(1, (units + chunk - 1) / chunk);
}

static int env_kernel() {
  const char *e = getenv("AXE_FORCE_KERNEL");
  if (!e || !*e) return AXE_KERNEL_AUTO;
  if (!strcmp(e, "generic")) return AXE_KERNEL_GENERIC;
  if (!strcmp(e, "vector")) return AXE_KERNEL_VECTOR;
  if (!strcmp(e, "tma")) return AXE_KERNEL_TMA;
  if (!strcmp(e, "tile")) return AXE_KERNEL_TILE;
  if (!strcmp(e, "register")) return AXE_KERNEL_REGISTER;
  if (!strcmp(e, "shuffle")) return AXE_KERNEL_SHUFFLE;
  if (!strcmp(e, "transpose")) return AXE_KERNEL_TRANSPOSE;
  if (!strcmp(e, "lowered")) return AXE_KERNEL_LOWERED;
  if (!strcmp(e, "dual")) return AXE_KERNEL_DUAL;
  return AXE_KERNEL_AUTO;
}

static bool divides_all(int64_t v, const std::vector<int64_t> &xs) {
  for (int64_t x : xs)
    if (x % v) return false;
  return true;
}

// K1: vector digit + joint digits -> parameter block.  Returns false if K1 cannot run the problem.
static bool build_k1(const std::vector<Joint> &J0, const Linear &ls, const Linear &ld, const Storage &sst,
                     const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why) {
  // destination replica offsets (elements), deduplicated (set semantics)
  std::vector<int64_t> reps{0};
  for (auto &r : ld.R) {
    std::vector<int64_t> nx;
    for (int64_t b : reps)
      for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
    reps.swap(nx);
    if (reps.size() > 4096) break;
  }
  std::sort(reps.begin(), reps.end());
  reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
  if ((int)reps.size() > K1_MAXREP) {
    *why = "too many destination replicas for the vector kernel";
    return false;
  }
  std::vector<Joint> J = J0;
  // vector width V (elements): a power of two with V*es <= 16 dividing the shared
  // innermost stride-1 run, every other stride, both bases and every replica offset
  int64_t V = 1;
  const Joint &in = J.back();
  if (in.ss == 1 && in.ds == 1) {
    std::vector<int64_t> all{ls.base, ld.base};
    for (size_t k = 0; k + 1 < J.size(); k++) {
      all.push_back(J[k].ss);
      all.push_back(J[k].ds);
    }
    for (int64_t r : reps) all.push_back(r);
    int64_t cap = std::min<int64_t>(16, max_align) / es;
    if (sst.swz_b > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(1) << sst.swz_m) / es));
    if (dstst.swz_b > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(1) << dstst.swz_m) / es));
    for (int64_t v = 2; v <= cap; v *= 2)
      if (in.e % v == 0 && divides_all(v, all)) V = v;
  }
  if (V > 1) {
    Joint last = J.back();
    J.pop_back();
    if (last.e / V > 1) J.push_back(Joint{last.e / V, V, V});
  }
  // kernel order: the traversal order of a copy is free (every digit is an
  // independent loop), so consecutive threads walk the destination-contiguous
  // digits first -- every warp writes whole 128-byte lines.
  std::vector<Joint> D;  // inner (fastest) first
  for (auto &j : J)
    if (j.e > 1) D.push_back(j);
  std::stable_sort(D.begin(), D.end(), [](const Joint &a, const Joint &b) {
    int64_t x = a.ds < 0 ? -a.ds : a.ds, y = b.ds < 0 ? -b.ds : b.ds;
    if (x != y) return x < y;
    return (a.ss < 0 ? -a.ss : a.ss) < (b.ss < 0 ? -b.ss : b.ss);
  });
  if (D.empty()) D.push_back(Joint{1, 0, 0});
  int64_t total = 1;
  for (auto &j : D) total *= j.e;
  if (total >= (int64_t(1) << 31)) {  // 32-bit grid-stride index: base + step must not wrap
    *why = "2^31 or more vectors";
    return false;
  }
  K1Params &k = P->k1;
  memset(&k, 0, sizeof(k));
  k.total = (uint32_t)total;
  k.sbase = ls.base * es;
  k.dbase = ld.base * es;
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  k.ssw = make_swz(sst);
  k.dsw = make_swz(dstst);
  P->covers_all = (int64_t)reps.size() * total * V == dstst.cells;
  // distinct 32-byte sectors (source, destination) touched by the first nv vectors of order D
  auto sectors = [&](const std::vector<Joint> &order, int64_t nv) {
    std::set<int64_t> ssec, dsec;
    for (int64_t i = 0; i < nv; i++) {
      int64_t rem = i, so = 0, dof = 0;
      for (auto &j : order) {
        int64_t d = rem % j.e;
        rem /= j.e;
        so += d * j.ss;
        dof += d * j.ds;
      }
      for (int64_t b = so * es; b < so * es + (int64_t)(V * es); b += 32) ssec.insert(b >> 5);
      for (int64_t b = dof * es; b < dof * es + (int64_t)(V * es); b += 32) dsec.insert(b >> 5);
    }
    return std::make_pair((int64_t)ssec.size(), (int64_t)dsec.size());
  };
  {
    // sector efficiency of one CTA's worth of vectors (kernel order, dst-contiguous first): a
    // schedule whose source reads scatter over many 32-byte sectors is better staged through smem
    const int64_t nv = std::min<int64_t>(total, 1024);
    auto sd = sectors(D, nv);
    const double useful = (double)nv * V * es;
    P->k1_sector_eff = std::min(useful / (32.0 * sd.first), useful / (32.0 * sd.second));
  }
  if (env_int("AXE_K1_WARP_ORDER", 1) && total >= env_int("AXE_K1_WARP_VECTORS", 32)) {
    // warp-level order: the 32 vectors one warp moves at once are chosen greedily, one prime
    // factor of a digit at a time, to touch the fewest 32-byte sectors on both sides (ties keep
    // the destination-contiguous order); the rest stays destination-stride sorted. Any order of
    // the independent digits is the same copy, so this only changes the schedule.
    const int64_t wv = env_int("AXE_K1_WARP_VECTORS", 32);
    std::vector<Joint> rem = D, pre;
    int64_t pv = 1;
    while (pv < wv) {
      int bi = -1;
      int64_t bc = 0, bf = 0;
      for (size_t i = 0; i < rem.size(); i++) {
        int64_t e = rem[i].e, f = 2;
        if (e <= 1) continue;
        while (e % f) f++;
        if (pv * f > wv) continue;
        std::vector<Joint> t = pre;
        t.push_back(Joint{f, rem[i].ss, rem[i].ds});
        auto sd = sectors(t, pv * f);
        int64_t c = sd.first + sd.second;
        if (bi < 0 || c < bc) bi = (int)i, bc = c, bf = f;
      }
      if (bi < 0) break;
      pre.push_back(Joint{bf, rem[bi].ss, rem[bi].ds});
      rem[bi] = Joint{rem[bi].e / bf, rem[bi].ss * bf, rem[bi].ds * bf};
      pv *= bf;
    }
    std::vector<Joint> nd;
    for (auto &j : pre) nd.push_back(j);
    for (auto &j : rem)
      if (j.e > 1) nd.push_back(j);
    // fuse neighbours that continue one another (inner-first)
    std::vector<Joint> fz;
    for (auto &j : nd) {
      if (!fz.empty() && fz.back().ss * fz.back().e == j.ss && fz.back().ds * fz.back().e == j.ds)
        fz.back().e *= j.e;
      else
        fz.push_back(j);
    }
    auto a = sectors(D, wv), b = sectors(fz, wv);
    if (b.first + b.second < a.first + a.second) D = fz;
  }
  P->vb = (int)(V * es);
  P->align = std::max(P->vb, es);
  const int u = k1_unroll(P->vb);

  // tiled form: a digit boundary at tile_v = 256 * u vectors (split by gcd, Lemma split)
  std::vector<Joint> inner, outer;
  int64_t tile_v = 256LL * u;
  bool tiled = total >= tile_v && total % tile_v == 0;
  if (tiled) {
    int64_t prefix = 1;
    size_t k2 = 0;
    std::vector<Joint> rest = D;
    while (prefix < tile_v && k2 < rest.size()) {
      int64_t need = tile_v / prefix;
      Joint j = rest[k2];
      int64_t g = std::gcd(j.e, need);
      if (g == j.e) {
        inner.push_back(j);
        prefix *= j.e;
        k2++;
      } else if (g > 1) {
        inner.push_back(Joint{g, j.ss, j.ds});
        rest[k2] = Joint{j.e / g, j.ss * g, j.ds * g};
        prefix *= g;
      } else {
        break;
      }
    }
    if (prefix != tile_v) tiled = false;
    for (; tiled && k2 < rest.size(); k2++) outer.push_back(rest[k2]);
    if (tiled) {
      // fill() below expects inner-first order: fuse outermost-first, then reverse
      sort_fuse_outer(outer);
      std::reverse(outer.begin(), outer.end());
    }
    if ((int)inner.size() > K1_MAXD || (int)outer.size() > K1_MAXD) tiled = false;
  }
  auto fill = [&](const std::vector<Joint> &inner_first, FastDiv *fd, int64_t *a, int64_t *b) {
    int n = (int)inner_first.size();
    for (int i = 0; i < n; i++) {  // parameter blocks are outermost first
      const Joint &j = inner_first[n - 1 - i];
      fd[i] = make_fastdiv((uint32_t)j.e);
      a[i] = j.ss * es;
      b[i] = j.ds * es;
    }
    return n;
  };
  std::string mode;
  if (tiled) {
    k.tile_v = (uint32_t)tile_v;
    k.ntiles = (uint32_t)(total / tile_v);
    k.nin = fill(inner, k.ifd, k.iss, k.ids);
    k.nout = fill(outer, k.ofd, k.oss, k.ods);
    // the swizzle commutes with adding a tile base that is a whole number of swizzle blocks
    auto whole = [&](const Swz &sw, int64_t base, const std::vector<int64_t> &extra, bool src) {
      if (!sw.mask) return 1;
      int64_t blk = int64_t(1) << (sw.shift + ilog2_floor(sw.mask + 1));
      if (base % blk) return 0;
      for (auto &j : outer)
        if ((src ? j.ss : j.ds) * es % blk) return 0;
      for (int64_t r : extra)
        if (r % blk) return 0;
      return 1;
    };
    std::vector<int64_t> rb;
    for (int64_t r : reps) rb.push_back(r * es);
    k.pre_s = whole(k.ssw, k.sbase, {}, true);
    k.pre_d = whole(k.dsw, k.dbase, rb, false);
    int64_t cap = grid_cap(8);
    P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(k.ntiles, cap));
    // in-order schedule, 2 tiles (32 KiB) per CTA, whenever the tiles outnumber the persistent grid
    // (16 KiB-run gathers, profiles/r02_sweep_front.log: 32 MiB 12.0 us vs 12.8, 256 MiB 82.1 vs 88.1)
    k.chunk = unit_chunk(k.ntiles > (int64_t)P->blocks ? 2 : 0);
    P->blocks = chunk_grid(k.ntiles, k.chunk, P->blocks);
    mode = "tiled";
  } else {
    if ((int)D.size() > K1_MAXD) {
      *why = "too many joint digits for the vector kernel";
      return false;
    }
    k.nd = fill(D, k.fd, k.ss, k.ds);
    int64_t blocks = (total + 256LL * u - 1) / (256LL * u);
    int64_t cap = grid_cap(8);
    P->blocks = (unsigned)std::max<int64_t>(1, std::min(blocks, cap));
    k.chunk = unit_chunk(0);
    P->blocks = chunk_grid(blocks, k.chunk, P->blocks);
    mode = "decode";
  }
  char b[320];
  snprintf(b, sizeof b,
           "{\"kernel\":\"vector\",\"mode\":\"%s\",\"vec_bytes\":%d,\"vectors\":%lld,\"replicas\":%d,\"blocks\":%u,"
           "\"tile_vectors\":%u,\"chunk\":%u,\"pre_swizzle\":[%d,%d],\"digits\":",
           mode.c_str(), P->vb, (long long)total, k.nrep, P->blocks, k.tile_v, k.chunk, k.pre_s, k.pre_d);
  P->desc = std::string(b) + joint_json(D) + ",\"joint\":" + joint_json(J0) + "}";
  return true;
}

// K1-TMA: boxes of (rows x row bytes) contiguous on the "bulk" side
// and a strided 2-D box (plus up to 3 outer dims) on the "tensor" side.
// mode 0: tensor side = source (TMA load), bulk side = destination;
// mode 1: tensor side = destination (TMA store), bulk side = source.
static bool build_tma(const std::vector<Joint> &J0, const Linear &ls, const Linear &ld, const Storage &sst,
                      const Storage &dstst, int es, int mode, CopyPlan *P, std::string *why) {
  const Storage &tst = mode == 0 ? sst : dstst;
  const Storage &bst = mode == 0 ? dstst : sst;
  const Linear &lt = mode == 0 ? ls : ld;
  const Linear &lb = mode == 0 ? ld : ls;
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  if (tst.swz_b) return fail("tma: the tensor-map side is swizzled in global memory");
  int span = 0;
  if (bst.swz_b) {
    if (bst.swz_m != 4 || bst.swz_s != 3 || bst.swz_b > 3) return fail("tma: swizzle is not a TMA mode");
    span = 16 << bst.swz_b;
  }
  if (mode == 1 && !ld.R.empty()) return fail("tma: destination replicas need the bulk-store mode");
  std::vector<int64_t> reps{0};
  for (auto &r : ld.R) {
    std::vector<int64_t> nx;
    for (int64_t b : reps)
      for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
    reps.swap(nx);
  }
  std::sort(reps.begin(), reps.end());
  reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
  if ((int)reps.size() > K1_MAXREP) return fail("tma: too many replicas");
  struct TB {
    int64_t e, t, b;
  };
  std::vector<TB> d;
  for (auto &j : J0)
    if (j.e > 1) d.push_back(TB{j.e, mode == 0 ? j.ss : j.ds, mode == 0 ? j.ds : j.ss});
  for (auto &x : d)
    if (x.t <= 0 || x.b <= 0) return fail("tma: negative strides");
  std::stable_sort(d.begin(), d.end(), [](const TB &a, const TB &b) { return a.b < b.b; });
  if (d.size() < 2 || d[0].t != 1 || d[0].b != 1) return fail("tma: no shared contiguous run");
  const int64_t e0 = d[0].e;
  int64_t R = 0;
  if (span) {
    if (span % es || e0 % (span / es)) return fail("tma: run does not fill the swizzle span");
    R = span / es;
  } else {
    for (int64_t r = e0; r >= 1; r--)
      if (e0 % r == 0 && r * es <= 256 && (r * es) % 16 == 0) {
        R = r;
        break;
      }
    if (!R) return fail("tma: no 16-byte-multiple row length");
  }
  if (e0 > R) {
    d[0] = TB{R, 1, 1};
    d.insert(d.begin() + 1, TB{e0 / R, R, R});
  }
  if (d[1].b != R) return fail("tma: rows of a box are not contiguous on the bulk side");
  const int64_t E1 = d[1].e, t1 = d[1].t;
  if ((t1 * es) % 16) return fail("tma: row stride not a multiple of 16 bytes");
  const int64_t row_bytes = R * es;
  int64_t B1 = 0;
  for (int64_t b = std::min<int64_t>(E1, 256); b >= 1; b--)
    if (E1 % b == 0 && b * row_bytes <= 16384 && (!span || b % 8 == 0)) {
      B1 = b;
      break;
    }
  if (!B1) return fail("tma: no legal box height");
  int64_t box_bytes = B1 * row_bytes;
  const int64_t blk = span ? span * 8 : 16;  // the bulk-side box base must be a whole swizzle block
  TmaParams &k = P->tma;
  memset(&k, 0, sizeof(k));
  std::vector<std::array<int64_t, 4>> digs;  // extent, cdim, cmul, bulk stride (bytes), outermost last
  if (E1 / B1 > 1) digs.push_back({E1 / B1, 1, B1, B1 * d[1].b * es});
  int dim = 2;
  P->tm_dims[0] = (uint64_t)row_bytes;
  P->tm_box[0] = (uint32_t)row_bytes;
  P->tm_dims[1] = (uint64_t)E1;
  P->tm_strides[0] = (uint64_t)(t1 * es);
  P->tm_box[1] = (uint32_t)B1;
  for (size_t i = 2; i < d.size(); i++) {
    if (dim > 4) return fail("tma: more than 5 tensor dimensions");
    if ((d[i].t * es) % 16) return fail("tma: outer stride not a multiple of 16 bytes");
    P->tm_dims[dim] = (uint64_t)d[i].e;
    P->tm_strides[dim - 1] = (uint64_t)(d[i].t * es);
    P->tm_box[dim] = 1;
    if (d[i].e > 1) digs.push_back({d[i].e, dim, 1, d[i].b * es});
    dim++;
  }
  for (int i = dim; i < 5; i++) P->tm_strides[i - 1] = P->tm_strides[dim - 2 > 0 ? dim - 2 : 0];
  if ((int)digs.size() > TMA_MAXD) return fail("tma: too many box digits");
  int64_t nboxes = 1;
  for (auto &g : digs) {
    nboxes *= g[0];
    if (g[3] % blk) return fail("tma: box bases are not whole swizzle blocks");
  }
  if (nboxes >= (int64_t(1) << 31)) return fail("tma: too many boxes");
  if ((lb.base * es) % blk || (lt.base * es) % 16) return fail("tma: misaligned base offset");
  for (int64_t r : reps)
    if ((r * es) % blk) return fail("tma: replica offsets are not whole swizzle blocks");
  k.nboxes = (uint32_t)nboxes;
  k.nd = (int)digs.size();
  for (int i = 0; i < k.nd; i++) {  // params are outermost first; digs is innermost first
    auto &g = digs[digs.size() - 1 - i];
    k.fd[i] = make_fastdiv((uint32_t)g[0]);
    k.cdim[i] = (int32_t)g[1];
    k.cmul[i] = (int32_t)g[2];
    k.bstride[i] = g[3];
  }
  k.bbase = lb.base * es;
  k.box_bytes = (uint32_t)box_bytes;
  {
    const int64_t al = span ? 1024 : 128;
    k.slot_bytes = (uint32_t)((box_bytes + al - 1) / al * al);
  }
  k.mode = mode;
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  // 16 KiB of boxes per CTA (2 x 8 KiB for config 2) and 8 CTAs per SM: measured on B200 at
  // 1 GiB 174 us against 190 us with 3 stages or 10-12 CTAs/SM, unchanged at 64 MiB (10.1 us)
  int64_t stage_bytes = env_int("AXE_TMA_STAGE_BYTES", 16384);
  int stages = (int)std::max<int64_t>(2, std::min<int64_t>(16, stage_bytes / k.slot_bytes));
  k.stages = stages;
  P->tm_swizzle = span;
  P->tm_base = lt.base * es;
  P->tm_cache = std::make_shared<TmaCache>();
  int per_sm = (int)std::max<int64_t>(1, std::min<int64_t>(16, (220 * 1024) / (int64_t)tma_smem_bytes(k)));
  per_sm = (int)std::min<int64_t>(per_sm, env_int("AXE_TMA_PER_SM", 8));
  P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nboxes, grid_cap(per_sm)));
  // in-order schedule, 2 boxes per CTA (256-byte-run gathers, profiles/r02_sweep_front.log: 32 MiB
  // 12.8 us vs 14.5, 256 MiB 82.4 vs 96.1)
  k.chunk = unit_chunk(nboxes > (int64_t)P->blocks ? 2 : 0);
  P->blocks = chunk_grid(nboxes, k.chunk, P->blocks);
  if (k.chunk && env_int("AXE_TMA_CHUNK_RING", 1)) k.stages = (int)std::min<int64_t>(k.stages, k.chunk);
  P->align = 16;
  P->covers_all = (int64_t)reps.size() * nboxes * box_bytes == dstst.cells * es;
  char b[320];
  snprintf(b, sizeof b,
           "{\"kernel\":\"tma\",\"mode\":\"%s\",\"box\":[%lld,%lld],\"box_bytes\":%lld,\"boxes\":%lld,\"stages\":%d,"
           "\"blocks\":%u,\"chunk\":%u,\"swizzle\":%d,\"replicas\":%d,\"joint\":",
           mode == 0 ? "tensor-load/bulk-store" : "bulk-load/tensor-store", (long long)B1, (long long)row_bytes,
           (long long)box_bytes, (long long)nboxes, stages, P->blocks, k.chunk, span, k.nrep);
  // the encoded tensor map (byte elements): dims / byte strides innermost first, box
  std::string tm = ",\"tensor_map\":{\"dims\":[";
  for (int i = 0; i < 5; i++) tm += (i ? "," : "") + std::to_string(P->tm_dims[i]);
  tm += "],\"strides\":[1";
  for (int i = 0; i < 4; i++) tm += "," + std::to_string(P->tm_strides[i]);
  tm += "],\"box\":[";
  for (int i = 0; i < 5; i++) tm += (i ? "," : "") + std::to_string(P->tm_box[i]);
  tm += "],\"base\":" + std::to_string(P->tm_base) + "}";
  P->desc = std::string(b) + joint_json(J0) + tm + "}";
  return true;
}

// K1-TMA mode 2: a run contiguous on BOTH sides (the innermost joint digit with unit strides,
// >= 1 KiB) moves as whole boxes: cp.async.bulk global->smem, cp.async.bulk smem->global per
// destination replica.  No tensor map; the box-index digits give both byte offsets.
static bool build_bulk(const std::vector<Joint> &J0, const Linear &ls, const Linear &ld, const Storage &sst,
                       const Storage &dstst, int es, int64_t min_run_bytes, CopyPlan *P, std::string *why) {
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  if (sst.swz_b || dstst.swz_b) return fail("bulk: swizzled storage");
  std::vector<Joint> J;
  for (auto &j : J0)
    if (j.e > 1) J.push_back(j);
  if (J.empty() || J.back().ss != 1 || J.back().ds != 1) return fail("bulk: no run contiguous on both sides");
  const int64_t run = J.back().e;
  if (run * es < min_run_bytes) return fail("bulk: contiguous run too short");
  // box: the largest divisor of the run with <= 16 KiB and a multiple of 16 bytes
  int64_t be = 0;
  for (int64_t d = 1; d * d <= run; d++)
    if (run % d == 0)
      for (int64_t c : {d, run / d})
        if (c * es <= env_int("AXE_TMA_BULK_BOX", 16384) && (c * es) % 16 == 0 && c > be) be = c;
  if (be * es < 1024) return fail("bulk: no box of 1-16 KiB divides the run");
  std::vector<int64_t> reps{0};
  for (auto &r : ld.R) {
    std::vector<int64_t> nx;
    for (int64_t b : reps)
      for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
    reps.swap(nx);
    if (reps.size() > 4096) break;
  }
  std::sort(reps.begin(), reps.end());
  reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
  if ((int)reps.size() > K1_MAXREP) return fail("bulk: too many replicas");
  std::vector<Joint> D(J.begin(), J.end() - 1);
  if (run / be > 1) D.push_back(Joint{run / be, be, be});
  // box order: destination order, fused where contiguous on both sides
  std::stable_sort(D.begin(), D.end(), [](const Joint &a, const Joint &b) { return std::llabs(a.ds) > std::llabs(b.ds); });
  sort_fuse_outer(D);
  if ((int)D.size() > TMA_MAXD) return fail("bulk: too many box digits");
  int64_t nboxes = 1;
  for (auto &j : D) nboxes *= j.e;
  if (nboxes >= (int64_t(1) << 31)) return fail("bulk: too many boxes");
  auto a16 = [&](int64_t v) { return (v * es) % 16 == 0; };
  if (!a16(ls.base) || !a16(ld.base)) return fail("bulk: bases not 16-byte aligned");
  for (auto &j : D)
    if (!a16(j.ss) || !a16(j.ds)) return fail("bulk: strides not 16-byte aligned");
  for (int64_t r : reps)
    if (!a16(r)) return fail("bulk: replica offsets not 16-byte aligned");
  TmaParams &k = P->tma;
  memset(&k, 0, sizeof(k));
  k.nboxes = (uint32_t)nboxes;
  k.nd = (int)D.size();
  for (int i = 0; i < k.nd; i++) {
    k.fd[i] = make_fastdiv((uint32_t)D[i].e);
    k.cdim[i] = -1;
    k.bstride[i] = D[i].ds * es;
    k.sstride[i] = D[i].ss * es;
  }
  k.bbase = ld.base * es;
  k.sbase = ls.base * es;
  k.box_bytes = (uint32_t)(be * es);
  k.slot_bytes = (uint32_t)((k.box_bytes + 127) / 128 * 128);
  k.mode = 2;
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  // ring per CTA and CTAs per SM by size (identity copies, profiles/r02_bulk_ring_sweep.log): up to 64 MiB
  // a side, 96 KiB rings x 2 CTAs/SM (32 MiB: 10.6 us vs 13.1 with 16 KiB x 4: the whole copy is in flight
  // at once); up to 256 MiB, 64 KiB x 3 (128 MiB: 44.5 vs 46.2); beyond, 16 KiB x 4 (512 MiB: 171 vs 176 --
  // long copies stream, and deep rings only delay the first stores)
  const int64_t bytes = nboxes * be * es;
  const int64_t ring_def = bytes <= (int64_t(64) << 20) ? 98304 : bytes <= (int64_t(256) << 20) ? 65536 : 16384;
  const int64_t per_def = bytes <= (int64_t(64) << 20) ? 2 : bytes <= (int64_t(256) << 20) ? 3 : 4;
  const int64_t stage_bytes = env_int("AXE_TMA_STAGE_BYTES", ring_def);
  k.stages = (int)std::max<int64_t>(2, std::min<int64_t>(16, stage_bytes / k.slot_bytes));
  P->tm_swizzle = 0;
  P->tm_cache.reset();
  int per_sm = (int)std::max<int64_t>(1, std::min<int64_t>(16, (220 * 1024) / (int64_t)tma_smem_bytes(k)));
  per_sm = (int)std::min<int64_t>(per_sm, env_int("AXE_TMA_BULK_PER_SM", per_def));
  P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nboxes, grid_cap(per_sm)));
  // beyond 64 MiB, the in-order schedule with 2 boxes per CTA (identity 256 MiB: 77.6 us vs 89.5;
  // up to 64 MiB the persistent ring keeps the whole copy in flight and wins: 11.1 us vs 14.3)
  k.chunk = unit_chunk(bytes > (int64_t(64) << 20) && nboxes > (int64_t)P->blocks ? 2 : 0);
  P->blocks = chunk_grid(nboxes, k.chunk, P->blocks);
  // in-order schedule: a ring of the CTA's own boxes only (every box in flight at once, no refill), so the
  // shared memory admits more CTAs per SM
  if (k.chunk && env_int("AXE_TMA_CHUNK_RING", 1)) k.stages = (int)std::min<int64_t>(k.stages, k.chunk);
  P->align = 16;
  P->covers_all = (int64_t)reps.size() * nboxes * be == dstst.cells;
  char b[320];
  snprintf(b, sizeof b,
           "{\"kernel\":\"tma\",\"mode\":\"bulk-load/bulk-store\",\"box_bytes\":%lld,\"boxes\":%lld,\"stages\":%d,"
           "\"blocks\":%u,\"chunk\":%u,\"replicas\":%d,\"joint\":",
           (long long)(be * es), (long long)nboxes, k.stages, P->blocks, k.chunk, k.nrep);
  P->desc = std::string(b) + joint_json(J0) + "}";
  return true;
}

static axe_status plan_copy_core(const PlanRequest &rq, CopyPlan *out);

axe_status plan_copy(const PlanRequest &rq, CopyPlan *out) {
  AXE_TRY(plan_copy_core(rq, out));
  if (!rq.no_chunk && rq.skip_axis < 0 && out->linear) {
    Linear ls, ld;
    std::vector<Joint> J;
    if (compose_linear(*rq.src, *rq.sst, -1, &ls) && compose_linear(*rq.dst, *rq.dstst, -1, &ld) &&
        joint_refine(ls.D, ld.D, &J))
      plan_chunks(rq, J, ls, ld, out);  // best effort: no chunking on failure
    if (out->n_chunks && !out->desc.empty() && out->desc.back() == '}')
      out->desc.insert(out->desc.size() - 1, ",\"host_chunks\":" + std::to_string(out->n_chunks));
  }
  return AXE_OK;
}

HostPipe::~HostPipe() {
  for (auto e : ev)
    if (e) cudaEventDestroy(e);
  for (auto s : {h2d, comp, d2h})
    if (s) cudaStreamDestroy(s);
}

// A joint digit that spans both whole buffers (src stride * extent = src cells,
// dst stride * extent = dst cells) cuts the copy into independent slabs.
axe_status plan_chunks(const PlanRequest &rq, const std::vector<Joint> &J, const Linear &ls, const Linear &ld,
                       CopyPlan *P) {
  if (ls.base || ld.base || !ld.R.empty()) return AXE_OK;
  const int64_t sc = rq.sst->cells, dc = rq.dstst->cells, es = rq.es;
  int best = -1;
  for (size_t i = 0; i < J.size(); i++)
    if (J[i].ss > 0 && J[i].ds > 0 && J[i].ss * J[i].e == sc && J[i].ds * J[i].e == dc && J[i].e > 1) best = (int)i;
  if (best < 0) return AXE_OK;
  const Joint cj = J[best];
  // up to AXE_HOST_CHUNKS (8, measured best of 4..32) slabs of >= 1 MiB, each a whole number of swizzle blocks on both sides
  int n = 1;
  const int64_t max_ch = rq.host_slabs > 0 ? rq.host_slabs : env_int("AXE_HOST_CHUNKS", 8);
  for (int c = 2; c <= 32; c++) {
    if (cj.e % c) continue;
    int64_t sb = sc / c * es, db = dc / c * es;
    if (sb < (1 << 20)) break;
    auto whole = [&](const Storage *st, int64_t bytes) {
      return !st->swz_b || bytes % (int64_t(1) << (st->swz_b + st->swz_m + st->swz_s)) == 0;
    };
    if (whole(rq.sst, sb) && whole(rq.dstst, db) && sb % 16 == 0 && db % 16 == 0) n = c;
    if (n >= max_ch) break;
  }
  if (n < 2) return AXE_OK;
  std::vector<Iter> sD, dD;
  for (size_t i = 0; i < J.size(); i++) {
    int64_t e = (int)i == best ? J[i].e / n : J[i].e;
    sD.push_back(Iter{e, J[i].ss, axis_m()});
    dD.push_back(Iter{e, J[i].ds, axis_m()});
  }
  Layout sL, dL;
  AXE_TRY(make_layout(sD, {}, {}, &sL));
  AXE_TRY(make_layout(dD, {}, {}, &dL));
  Storage sst, dst;
  sst.d.push_back(SDigit{axis_m(), sc / n, 1, 1});
  sst.cells = sc / n;
  sst.swz_b = rq.sst->swz_b, sst.swz_m = rq.sst->swz_m, sst.swz_s = rq.sst->swz_s;
  dst.d.push_back(SDigit{axis_m(), dc / n, 1, 1});
  dst.cells = dc / n;
  dst.swz_b = rq.dstst->swz_b, dst.swz_m = rq.dstst->swz_m, dst.swz_s = rq.dstst->swz_s;
  auto sub = std::make_shared<CopyPlan>();
  PlanRequest r2{&sL, &dL, &sst, &dst, rq.es, rq.kernel, rq.max_align, -1};
  r2.no_chunk = 1;
  if (plan_copy_core(r2, sub.get()) != AXE_OK) return AXE_OK;
  P->chunk = sub;
  P->n_chunks = n;
  P->pipe = std::make_shared<HostPipe>();
  return AXE_OK;
}

axe_status run_copy_host(const CopyPlan &P, const void *host_src, void *host_dst, void *dev_src, void *dev_dst,
                         cudaStream_t st) {
  cudaError_t e = cudaSuccess;
#define CU(x)                                                                              \
  do {                                                                                     \
    e = (x);                                                                               \
    if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e));     \
  } while (0)
  if (!P.chunk) {
    CU(cudaMemcpyAsync(dev_src, host_src, (size_t)P.src_bytes, cudaMemcpyHostToDevice, st));
    // cells outside the destination image keep their contents (reading R7): stage them too
    if (!P.covers_all) CU(cudaMemcpyAsync(dev_dst, host_dst, (size_t)P.dst_bytes, cudaMemcpyHostToDevice, st));
    AXE_TRY(run_copy(P, dev_src, dev_dst, st));
    CU(cudaMemcpyAsync(host_dst, dev_dst, (size_t)P.dst_bytes, cudaMemcpyDeviceToHost, st));
    return AXE_OK;
  }
  HostPipe &H = *P.pipe;
  std::lock_guard<std::mutex> lk(H.mu);
  int dev = 0;
  CU(cudaGetDevice(&dev));
  if (H.device != dev) {
    for (auto ev : H.ev)
      if (ev) cudaEventDestroy(ev);
    H.ev.clear();
    for (cudaStream_t *s : {&H.h2d, &H.comp, &H.d2h}) {
      if (*s) cudaStreamDestroy(*s);
      CU(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
    }
    H.ev.assign(3 * P.n_chunks + 2, nullptr);
    for (auto &ev : H.ev) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    H.device = dev;
  }
  const int n = P.n_chunks;
  const int64_t sb = P.src_bytes / n, db = P.dst_bytes / n;
  cudaEvent_t fork = H.ev[3 * n], join = H.ev[3 * n + 1];
  CU(cudaEventRecord(fork, st));
  for (cudaStream_t s : {H.h2d, H.comp, H.d2h}) CU(cudaStreamWaitEvent(s, fork, 0));
  stream_forget(H.comp);
  for (int c = 0; c < n; c++) {
    const uint8_t *hs = (const uint8_t *)host_src + c * sb;
    uint8_t *hd = (uint8_t *)host_dst + c * db;
    uint8_t *ds = (uint8_t *)dev_src + c * sb, *dd = (uint8_t *)dev_dst + c * db;
    CU(cudaMemcpyAsync(ds, hs, (size_t)sb, cudaMemcpyHostToDevice, H.h2d));
    if (!P.covers_all) CU(cudaMemcpyAsync(dd, hd, (size_t)db, cudaMemcpyHostToDevice, H.h2d));
    CU(cudaEventRecord(H.ev[3 * c], H.h2d));
    CU(cudaStreamWaitEvent(H.comp, H.ev[3 * c], 0));
    stream_forget(H.comp);
    AXE_TRY(run_copy(*P.chunk, ds, dd, H.comp));
    CU(cudaEventRecord(H.ev[3 * c + 1], H.comp));
    CU(cudaStreamWaitEvent(H.d2h, H.ev[3 * c + 1], 0));
    CU(cudaMemcpyAsync(hd, dd, (size_t)db, cudaMemcpyDeviceToHost, H.d2h));
  }
  CU(cudaEventRecord(join, H.d2h));
  CU(cudaStreamWaitEvent(st, join, 0));
#undef CU
  return AXE_OK;
}

static axe_status plan_copy_core(const PlanRequest &rq, CopyPlan *out) {
  const Layout &S = *rq.src, &D = *rq.dst;
  int es = rq.es;
  if (es != 1 && es != 2 && es != 4 && es != 8 && es != 16)
    AXE_FAIL(AXE_ERR_ALIGNMENT, "elem_size %d not in {1,2,4,8,16}", es);
  if (S.ED != D.ED) AXE_FAIL(AXE_ERR_SIZE_MISMATCH, "E_D(src) = %lld != E_D(dst) = %lld", (long long)S.ED, (long long)D.ED);
  AXE_TRY(check_side(S, *rq.sst, rq.skip_axis, "source"));
  AXE_TRY(check_side(D, *rq.dstst, rq.skip_axis, "destination"));
  for (const Storage *st : {rq.sst, rq.dstst})
    if (st->swz_b > 0 && (st->cells * es) % (int64_t(1) << (st->swz_b + st->swz_m + st->swz_s)))
      AXE_FAIL(AXE_ERR_BOUNDS, "swizzled storage of %lld bytes is not a whole number of %d-byte swizzle blocks",
               (long long)(st->cells * es), 1 << (st->swz_b + st->swz_m + st->swz_s));
  AXE_TRY(check_injective(D, *rq.dstst, rq.skip_axis));

  CopyPlan P;
  P.es = es;
  P.src_bytes = rq.sst->cells * es;
  P.dst_bytes = rq.dstst->cells * es;
  P.align = es;
  int kernel = rq.kernel == AXE_KERNEL_AUTO ? env_kernel() : rq.kernel;
  if (kernel == 6) AXE_FAIL(AXE_ERR_UNSUPPORTED, "kernel 6 (K2T) was retired: K7 / K2 run these transposes");
  if (kernel < AXE_KERNEL_AUTO || kernel > AXE_KERNEL_DUAL) AXE_FAIL(AXE_ERR_INVALID_ARG, "unknown kernel %d", kernel);

  Linear ls, ld;
  bool lin = compose_linear(S, *rq.sst, rq.skip_axis, &ls) && compose_linear(D, *rq.dstst, rq.skip_axis, &ld);
  std::vector<Joint> J;
  bool joint = lin && joint_refine(ls.D, ld.D, &J);
  P.linear = joint;
  if (joint) P.joint = J;

  std::string why = lin ? (joint ? "" : "digit systems are not nested (no joint refinement)")
                        : "storage composition is not affine";
  if (kernel == AXE_KERNEL_LOWERED) {
    std::string wl = joint ? "" : why;
    if (joint && rq.max_align >= 16 && build_lowered(J, ls, ld, *rq.sst, *rq.dstst, es, &P, &wl)) {
      P.kernel = KK_LOWERED;
      *out = std::move(P);
      return AXE_OK;
    }
    AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced lowered schedule cannot run these layouts: %s",
             rq.max_align < 16 ? "needs 16-byte aligned buffers" : wl.c_str());
  }
  // AUTO and unswizzled storage on both sides: K1-TMA only for a copy that is one contiguous run (a
  // bulk copy: 32 MiB 10.9 us vs K1's 11.8); strided runs go to K1 (4 KiB runs 12.4 vs 14.0 at 32 MiB,
  // 81.5 vs 85.1 at 256 MiB; 128-256-byte runs within 2%; profiles/r02_segment_probe.log)
  bool tma_auto_ok = true;
  if (kernel == AXE_KERNEL_AUTO && !rq.sst->swz_b && !rq.dstst->swz_b && env_int("AXE_TMA_STRIDED_AUTO", 0) == 0) {
    int nz = 0;
    for (auto &j : J) nz += j.e > 1;
    tma_auto_ok = nz <= 1;
  }
  if (joint && rq.max_align >= 16 && (kernel == AXE_KERNEL_TMA || (kernel == AXE_KERNEL_AUTO && tma_auto_ok))) {
    std::string w0, w1, w2;
    // AUTO takes a TMA plan only with boxes of >= 4 KiB: 1 KiB boxes measured 35 us against K1's 21 us
    // on a 64 MiB copy of 1 KiB rows (tools/perf_configs.py rows_1k); forced TMA takes any box
    const int64_t min_box = kernel == AXE_KERNEL_TMA ? 0 : env_int("AXE_TMA_MIN_BOX", 4096);
    const int64_t min_run = kernel == AXE_KERNEL_TMA ? 1024 : std::max<int64_t>(min_box, 1024);
    auto big = [&](bool ok) { return ok && (int64_t)P.tma.box_bytes >= min_box; };
    if (kernel == AXE_KERNEL_AUTO && env_int("AXE_LOWERED_AUTO", 1) &&
        (big(build_tma(J, ls, ld, *rq.sst, *rq.dstst, es, 0, &P, &w0)) ||
         big(build_tma(J, ls, ld, *rq.sst, *rq.dstst, es, 1, &P, &w1)))) {
      // the paper's own lowering (slice -> tile_of the swizzle atom -> tensor map) when it
      // reaches boxes as large as the joint-digit box: config 2 10.01 us vs 10.15 (64 MiB), 16384^2
      // 180.4 vs 177.5 us; reversed (TMA stores) 10.31 vs 10.46 us
      CopyPlan L = P;
      std::string wl;
      if (build_lowered(J, ls, ld, *rq.sst, *rq.dstst, es, &L, &wl) && lowered_box_bytes(L) >= P.tma.box_bytes) {
        L.kernel = KK_LOWERED;
        *out = std::move(L);
        return AXE_OK;
      }
    }
    if (big(build_tma(J, ls, ld, *rq.sst, *rq.dstst, es, 0, &P, &w0)) ||
        big(build_tma(J, ls, ld, *rq.sst, *rq.dstst, es, 1, &P, &w1)) ||
        big(build_bulk(J, ls, ld, *rq.sst, *rq.dstst, es, min_run, &P, &w2))) {
      P.kernel = KK_TMA;
      *out = std::move(P);
      return AXE_OK;
    }
    if (kernel == AXE_KERNEL_TMA)
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced TMA kernel cannot run these layouts: %s / %s / %s", w0.c_str(), w1.c_str(),
               w2.c_str());
  }
  if (joint && (kernel == AXE_KERNEL_AUTO || kernel == AXE_KERNEL_REGISTER)) {
    std::string w3;
    if (build_k3(J, ls, ld, *rq.sst, *rq.dstst, es, rq.max_align, &P, &w3)) {
      P.kernel = KK_REGISTER;
      // AUTO: the same permute with bulk-copied 16 KiB boxes and movmatrix in shared memory (config 3b:
      // 1373 us vs 1423 us for the register kernel); a forced "register" keeps the register kernel
      std::string w4;
      if (kernel == AXE_KERNEL_AUTO && env_int("AXE_K3_TMA", 1) && build_k3_bulk(&P, &w4)) P.kernel = KK_TMA;
      *out = std::move(P);
      return AXE_OK;
    }
    if (kernel == AXE_KERNEL_REGISTER)
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced register kernel cannot run these layouts: %s", w3.c_str());
  }
  if (joint && (kernel == AXE_KERNEL_AUTO || kernel == AXE_KERNEL_SHUFFLE)) {
    std::string w6;
    if (build_k6(J, ls, ld, *rq.sst, *rq.dstst, es, rq.max_align, &P, &w6)) {
      P.kernel = KK_SHUFFLE;
      *out = std::move(P);
      return AXE_OK;
    }
    if (kernel == AXE_KERNEL_SHUFFLE)
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced shuffle kernel cannot run these layouts: %s", w6.c_str());
  }
  if (joint && (kernel == AXE_KERNEL_AUTO || kernel == AXE_KERNEL_TRANSPOSE) && env_int("AXE_K7", 1)) {
    std::string w7, w9;
    if (build_k7(J, ls, ld, *rq.sst, *rq.dstst, es, rq.max_align, &P, &w7, kernel == AXE_KERNEL_TRANSPOSE)) {
      P.kernel = KK_TRANSPOSE;
      *out = std::move(P);
      return AXE_OK;
    }
    // forced: K9, the same 2-D transpose with ragged extents or pitches that are not whole 16-byte
    // vectors (AUTO tries it after K2, below)
    if (kernel == AXE_KERNEL_TRANSPOSE && build_k9(J, ls, ld, *rq.sst, *rq.dstst, es, &P, &w9)) {
      P.kernel = KK_RAGGED;
      *out = std::move(P);
      return AXE_OK;
    }
    if (kernel == AXE_KERNEL_TRANSPOSE)
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced transpose kernel cannot run these layouts: %s / %s", w7.c_str(),
               w9.c_str());
  }
  if (joint && kernel == AXE_KERNEL_TILE) {
    if (build_k2(J, ls, ld, *rq.sst, *rq.dstst, es, rq.max_align, &P, &why)) {
      P.kernel = KK_TILE;
      *out = std::move(P);
      return AXE_OK;
    }
    AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced tile kernel cannot run these layouts: %s", why.c_str());
  }
  if (kernel == AXE_KERNEL_AUTO || kernel == AXE_KERNEL_VECTOR || kernel == AXE_KERNEL_TMA) {
    if (joint && build_k1(J, ls, ld, *rq.sst, *rq.dstst, es, rq.max_align, &P, &why)) {
      P.kernel = KK_VECTOR;
      // vectors of <= 4 bytes (or scattered sectors): stage through shared memory instead (K2), which
      // moves 16-byte vectors on both sides (config 3a: K1 4-byte 1583 us, K2 1547 us on B200)
      if (kernel == AXE_KERNEL_AUTO && P.vb < 16 && (P.vb <= 4 || P.k1_sector_eff < 0.5)) {
        CopyPlan T = P;
        std::string w2, w9;
        if (build_k2(J, ls, ld, *rq.sst, *rq.dstst, es, rq.max_align, &T, &w2)) {
          T.kernel = KK_TILE;
          *out = std::move(T);
          return AXE_OK;
        }
        // no legal K2 tile (prime-ish extents, rows at any alignment): a 2-D transpose goes to K9
        // (4095 x 4097 bf16: 33.9 us vs K1's 78.4 with 2-byte vectors)
        CopyPlan R = P;
        if (env_int("AXE_K9", 1) && build_k9(J, ls, ld, *rq.sst, *rq.dstst, es, &R, &w9)) {
          R.kernel = KK_RAGGED;
          *out = std::move(R);
          return AXE_OK;
        }
      }
      *out = std::move(P);
      return AXE_OK;
    }
    if (kernel != AXE_KERNEL_AUTO)
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced kernel cannot run these layouts: %s", why.c_str());
  }
  // K8: the digit systems do not nest -- the shared innermost run still vectorises, the outer index is
  // decoded once per side (measured against K0 in profiles/r02_k8_dual.json)
  if (lin && !joint && (kernel == AXE_KERNEL_AUTO || kernel == AXE_KERNEL_DUAL)) {
    std::string w8;
    if (build_k8(ls, ld, *rq.sst, *rq.dstst, es, rq.max_align, &P, &w8)) {
      P.kernel = KK_DUAL;
      *out = std::move(P);
      return AXE_OK;
    }
    if (kernel == AXE_KERNEL_DUAL) AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced dual kernel cannot run these layouts: %s", w8.c_str());
  }
  if (kernel == AXE_KERNEL_DUAL) AXE_FAIL(AXE_ERR_UNSUPPORTED, "forced dual kernel: %s", why.c_str());
  // K0 generic
  memset(&P.k0, 0, sizeof(P.k0));
  AXE_TRY(build_k0_side(S, *rq.sst, rq.skip_axis, &P.k0.src));
  AXE_TRY(build_k0_side(D, *rq.dstst, rq.skip_axis, &P.k0.dst));
  P.k0.src.nR = 0;  // the source is read at its representative (reading R4)
  P.k0.ED = D.ED;
  P.k0.ER = D.ER;
  P.k0.es = es;
  P.kernel = KK_GENERIC;
  char b[256];
  snprintf(b, sizeof b, "{\"kernel\":\"generic\",\"elements\":%lld,\"replicas\":%lld,\"reason\":\"%s\"}",
           (long long)D.ED, (long long)D.ER, why.c_str());
  P.desc = b;
  *out = std::move(P);
  return AXE_OK;
}

// Programmatic-dependent-launch bookkeeping.  A kernel launched without
// griddepcontrol.wait may run concurrently with every libaxe kernel still in
// flight on its stream -- not only the previous one: when the previous kernel
// itself skipped the wait, it can be running beside ITS predecessor, and so on
// (measured: a read of a 1 GiB copy's output two launches later saw stale data
// when only the immediate predecessor was checked, tools/pdl_chain_probe.py).
// A kernel that does wait sees every earlier kernel complete (completion is
// transitive: a PDL secondary completes only after its primary; the same probe
// shows no stale read once the reader waits).  So each stream keeps the byte
// ranges of the kernels launched since its last waiting kernel (that one
// included); a new kernel skips the wait only when it neither reads nor writes
// what any of them writes and does not write what any of them reads.  Work the
// library did not launch (NCCL, memcpy) resets the window (stream_forget): the
// next kernel waits.  Windows are capped at 64 kernels.
namespace {
struct Ranges {
  uintptr_t s0, s1, d0, d1;
};
// A window belongs to one stream of one device: the handles 0 (legacy default stream) and
// cudaStreamPerThread name a different stream on every device, and the per-thread stream a different
// one on every host thread.
struct WinKey {
  cudaStream_t st;
  int dev;
  uint64_t tid;
  bool operator==(const WinKey &o) const { return st == o.st && dev == o.dev && tid == o.tid; }
};
struct WinKeyHash {
  size_t operator()(const WinKey &k) const {
    return std::hash<uintptr_t>()((uintptr_t)k.st) ^ (std::hash<uint64_t>()(k.tid) * 31) ^ ((size_t)k.dev << 20);
  }
};
std::mutex g_dep_mu;
std::unordered_map<WinKey, std::vector<Ranges>, WinKeyHash> g_win;

WinKey win_key(cudaStream_t st) {
  WinKey k{st, 0, 0};
  cudaGetDevice(&k.dev);
  if (st == cudaStreamPerThread) k.tid = (uint64_t)std::hash<std::thread::id>()(std::this_thread::get_id());
  return k;
}
}  // namespace

// Skipping griddepcontrol.wait across calls is opt-in (AXE_PDL_OVERLAP=1): the window sees only libaxe
// kernels, and a foreign kernel on the stream that triggers its dependents early (several libraries
// do) would be invisible to it.  By default every kernel waits (dep = 1): PDL then only overlaps the
// next kernel's launch and prologue with the previous kernel's tail.
bool pdl_overlap_enabled() {
  static const int on = [] {
    const char *e = getenv("AXE_PDL_OVERLAP");
    return (e && *e == '1') ? 1 : 0;
  }();
  return on != 0;
}

int stream_dependency(cudaStream_t st, uintptr_t s0, uintptr_t s1, uintptr_t d0, uintptr_t d1) {
  if (!pdl_overlap_enabled()) return 1;
  // only kernels moving <= 256 MiB overlap their predecessors: for them ramp-up and tail are a
  // visible share of the run, while two interleaved full-GPU 1 GiB copies contend (191 us vs 175 us
  // serialised)
  static const uintptr_t max_bytes = (uintptr_t)env_int("AXE_PDL_MAX_OVERLAP_BYTES", int64_t(256) << 20);
  auto hit = [](uintptr_t a0, uintptr_t a1, uintptr_t b0, uintptr_t b1) { return a0 < b1 && b0 < a1; };
  const WinKey key = win_key(st);
  std::lock_guard<std::mutex> lk(g_dep_mu);
  int dep = 1;
  auto it = g_win.find(key);
  if ((s1 - s0) + (d1 - d0) <= max_bytes && it != g_win.end() && !it->second.empty() && it->second.size() < 64) {
    dep = 0;
    for (const Ranges &L : it->second)
      if (hit(d0, d1, L.d0, L.d1) || hit(d0, d1, L.s0, L.s1) || hit(s0, s1, L.d0, L.d1)) {
        dep = 1;
        break;
      }
  }
  if (g_win.size() > 256) g_win.clear();
  std::vector<Ranges> &w = g_win[key];
  if (dep) w.clear();  // waiting: every earlier kernel is complete when this one proceeds
  w.push_back(Ranges{s0, s1, d0, d1});
  return dep;
}

// The plan's CUtensorMap for a given pointer (encoded once per pointer, small per-plan cache).
static axe_status tensor_map_for(const CopyPlan &p, const void *tptr, std::array<uint64_t, 16> *map) {
  {
    std::lock_guard<std::mutex> lk(p.tm_cache->mu);
    for (auto &m : p.tm_cache->maps)
      if (m.first == tptr) {
        *map = m.second;
        return AXE_OK;
      }
  }
  int r = encode_tensor_map(map->data(), (uint8_t *)tptr + p.tm_base, p.tm_dims, p.tm_strides, p.tm_box, p.tm_swizzle);
  if (r != 0) AXE_FAIL(AXE_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", r);
  std::lock_guard<std::mutex> lk(p.tm_cache->mu);
  if (p.tm_cache->maps.size() >= 32) p.tm_cache->maps.erase(p.tm_cache->maps.begin());
  p.tm_cache->maps.push_back({tptr, *map});
  return AXE_OK;
}

// Work the library does not launch itself (NCCL, memcpy) was enqueued on st:
// the next libaxe kernel there must wait (full dependency).
void stream_forget(cudaStream_t st) {
  if (!pdl_overlap_enabled()) return;
  const WinKey key = win_key(st);
  std::lock_guard<std::mutex> lk(g_dep_mu);
  g_win.erase(key);
}

axe_status run_copy(const CopyPlan &p, const void *src, void *dst, cudaStream_t st) {
  uintptr_t s = (uintptr_t)src, d = (uintptr_t)dst;
  if (!src || !dst) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL buffer");
  if (s % p.align || d % p.align)
    AXE_FAIL(AXE_ERR_ALIGNMENT, "buffers must be %d-byte aligned for this plan", p.align);
  if (s < d + p.dst_bytes && d < s + p.src_bytes) AXE_FAIL(AXE_ERR_ALIAS, "source and destination buffers overlap");
  const int dep = stream_dependency(st, s, s + p.src_bytes, d, d + p.dst_bytes);
  cudaError_t e = cudaSuccess;
  switch (p.kernel) {
    case KK_VECTOR: {
      K1Params k = p.k1;
      k.dep = dep;
      e = launch_k1(k, p.vb, p.blocks, src, dst, st);
      break;
    }
    case KK_RAGGED: {
      K9Params k = p.k9;
      k.dep = dep;
      e = launch_k9(k, p.es, src, dst, st);
      break;
    }
    case KK_DUAL: {
      K8Params k = p.k8;
      k.dep = dep;
      e = k.bulk ? launch_k8_bulk(k, src, dst, st) : launch_k8(k, p.vb, src, dst, st);
      break;
    }
    case KK_GENERIC: {
      K0Params k = p.k0;
      k.dep = dep;
      e = launch_k0(k, src, dst, st);
      break;
    }
    case KK_REGISTER: {
      K3Params k = p.k3;
      k.dep = dep;
      e = launch_k3(k, p.blocks, src, dst, st);
      break;
    }
    case KK_LOWERED:
      return run_lowered(p, src, dst, st, dep);
    case KK_TRANSPOSE: {
      K7Params k = p.k7;
      k.dep = dep;
      e = launch_k7(k, p.es, p.blocks, src, dst, st);
      break;
    }
    case KK_SHUFFLE: {
      K6Params k = p.k6;
      k.dep = dep;
      e = launch_k6(k, p.blocks, src, dst, st);
      break;
    }
    case KK_TILE: {
      K2Params k = p.k2;
      k.dep = dep;
      e = launch_k2(k, p.k2_vs, p.k2_vd, p.k2_gb, p.blocks, src, dst, st);
      break;
    }
    case KK_TMA: {
      const void *tptr = p.tma.mode == 0 ? src : (const void *)dst;
      std::array<uint64_t, 16> map{};
      if (p.tma.mode != 2) AXE_TRY(tensor_map_for(p, tptr, &map));  // mode 2 has no tensor map
      TmaParams k = p.tma;
      k.dep = dep;
      e = launch_tma(map.data(), k, p.blocks, src, dst, st);
      break;
    }
    default: AXE_FAIL(AXE_ERR_UNSUPPORTED, "unknown kernel");
  }
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
  return AXE_OK;
}

}  // namespace axe
