// plan_k2.cpp -- planner of the K2 shared-memory staged tile kernel.
//
// From the joint digits (element strides) it chooses: the granule (the run
// shared by both sides), a source-contiguous chain and a destination-
// contiguous chain whose union is the tile, the per-thread/per-iteration
// offset tables, and -- by simulating the bank conflicts of one warp's
// shared-memory accesses -- the XOR swizzle of the staged tile ("swizzles
// chosen from the layouts", BASELINE north star; SW-style XOR of 16-byte
// chunks as in the TMA atoms of P:527).
#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <set>

#include "plan.hpp"

#include <cstdlib>

namespace axe {

Swz make_swz(const Storage &st);
int num_sms();

namespace {

struct Dig {
  int64_t e, ss, ds;
};

// chain prefix cut: how much of each digit a contiguous run of `len` elements
// (granule included) takes; returns false if the cut falls inside a digit at a
// non-divisor.
bool cut_chain(const std::vector<int> &chain, const std::vector<Dig> &D, int64_t G, int64_t len,
               std::vector<int64_t> &incl) {
  if (len % G) return false;
  int64_t rem = len / G;
  for (int i : chain) {
    if (rem <= 1) break;
    if (rem >= D[i].e) {
      if (rem % D[i].e) return false;
      incl[i] = D[i].e;
      rem /= D[i].e;
    } else {
      if (D[i].e % rem) return false;
      incl[i] = rem;
      rem = 1;
    }
  }
  return rem == 1;
}

// element offsets of index idx over digit pieces (outermost first: e, stride)
int64_t offset_of(const std::vector<std::pair<int64_t, int64_t>> &digs, int64_t idx) {
  int64_t o = 0;
  for (int k = (int)digs.size() - 1; k >= 0; k--) {
    o += (idx % digs[k].first) * digs[k].second;
    idx /= digs[k].first;
  }
  return o;
}

uint32_t swz_host(const Swz &s, uint32_t b) { return b ^ (((b >> s.shift) & s.mask) << s.base); }

// shared-memory wavefronts of one warp instruction (32 threads, width bytes each)
int wavefronts(const uint32_t *addr, int width) {
  int phases = width == 16 ? 4 : width == 8 ? 2 : 1;
  int per = 32 / phases, total = 0;
  for (int ph = 0; ph < phases; ph++) {
    std::map<int, std::set<uint32_t>> banks;
    for (int t = ph * per; t < (ph + 1) * per; t++)
      for (uint32_t b = addr[t] & ~3u; b < addr[t] + (uint32_t)width; b += 4) banks[(b / 4) % 32].insert(b / 4);
    int wf = 1;
    for (auto &kv : banks) wf = std::max(wf, (int)kv.second.size());
    total += wf;
  }
  return total;
}

}  // namespace

bool build_k2(const std::vector<Joint> &J, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why) {
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  if (max_align < 16) return fail("tile: needs 16-byte aligned buffers");
  for (auto &j : J)
    if (j.ss <= 0 || j.ds <= 0) return fail("tile: negative strides");
  std::vector<int64_t> reps{0};
  for (auto &r : ld.R) {
    std::vector<int64_t> nx;
    for (int64_t b : reps)
      for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
    reps.swap(nx);
  }
  std::sort(reps.begin(), reps.end());
  reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
  if ((int)reps.size() > K1_MAXREP) return fail("tile: too many replicas");

  // granule: the innermost run shared by both sides, as in K1's vector digit
  std::vector<Dig> D;
  int64_t G = 1;
  {
    std::vector<int64_t> all{ls.base, ld.base};
    for (auto &j : J)
      if (!(j.ss == 1 && j.ds == 1)) {
        all.push_back(j.ss);
        all.push_back(j.ds);
      }
    for (int64_t r : reps) all.push_back(r);
    int64_t run = 1;
    for (auto &j : J)
      if (j.ss == 1 && j.ds == 1) run = j.e;
    for (int64_t g = 2; g * es <= 16; g *= 2) {
      bool ok = run % g == 0;
      for (int64_t a : all) ok = ok && a % g == 0;
      if (ok) G = g;
    }
    for (auto &j : J) {
      if (j.ss == 1 && j.ds == 1) {
        if (j.e / G > 1) D.push_back(Dig{j.e / G, G, G});
      } else if (j.e > 1) {
        D.push_back(Dig{j.e, j.ss, j.ds});
      }
    }
  }
  if (sst.swz_b && (int64_t(1) << sst.swz_m) < G * es) return fail("tile: source swizzle finer than the granule");
  if (dstst.swz_b && (int64_t(1) << dstst.swz_m) < 16) return fail("tile: destination swizzle finer than 16 bytes");
  const int n = (int)D.size();
  std::vector<int> sch, dch;  // contiguous chains, fastest first
  {
    std::vector<int> o(n);
    std::iota(o.begin(), o.end(), 0);
    std::sort(o.begin(), o.end(), [&](int a, int b) { return D[a].ss < D[b].ss; });
    int64_t exp = G;
    for (int i : o) {
      if (D[i].ss != exp) break;
      sch.push_back(i);
      exp *= D[i].e;
    }
    std::sort(o.begin(), o.end(), [&](int a, int b) { return D[a].ds < D[b].ds; });
    exp = G;
    for (int i : o) {
      if (D[i].ds != exp) break;
      dch.push_back(i);
      exp *= D[i].e;
    }
  }
  auto chain_lens = [&](const std::vector<int> &ch) {
    std::vector<int64_t> L{G};
    int64_t p = G;
    for (int i : ch) {
      for (int64_t f = 2; f < D[i].e; f *= 2)
        if (D[i].e % f == 0) L.push_back(p * f);
      p *= D[i].e;
      L.push_back(p);
    }
    return L;
  };
  int64_t budget = 32768 / es;  // tile elements (32 KiB)
  if (const char *ev = getenv("AXE_K2_TILE_BYTES")) budget = std::max<int64_t>(1024, atoll(ev)) / es;  // tuning knob
  const int NT = K2_NT;
  struct Choice {
    int64_t Ls, Ld, TE, Vs, Vd;
    std::vector<int64_t> incl;
    int score;
  } best{0, 0, 0, 0, 0, {}, -1};
  for (int64_t Ls : chain_lens(sch))
    for (int64_t Ld : chain_lens(dch)) {
      std::vector<int64_t> is(n, 1), id(n, 1), inc(n, 1);
      if (!cut_chain(sch, D, G, Ls, is) || !cut_chain(dch, D, G, Ld, id)) continue;
      int64_t TE = G;
      bool ok = true;
      for (int i = 0; i < n; i++) {
        int64_t l = std::lcm(is[i], id[i]);
        if (D[i].e % l) ok = false;
        inc[i] = l;
        TE *= l;
      }
      if (!ok || TE > budget) continue;
      int64_t Vs = 1, Vd = 1;
      while (Vs * 2 * es <= 16 && Ls % (Vs * 2) == 0) Vs *= 2;
      while (Vd * 2 * es <= 16 && Ld % (Vd * 2) == 0) Vd *= 2;
      if (Vs * es < 4 || Vd * es < 4) continue;
      if (TE % (Vs * NT) || TE % (Vd * NT)) continue;
      if (TE / (Vs * NT) > 8 || TE / (Vd * NT) > K2_MAXJ || Vd / G > K2_MAXK) continue;
      static const int64_t run_cap = [] {
        const char *e = getenv("AXE_K2_RUN_CAP");  // tuning knob: run bytes worth rewarding
        return (e && *e) ? (int64_t)atoll(e) : (int64_t)256;
      }();
      int score = (int)(std::min<int64_t>(Ls * es, run_cap) + std::min<int64_t>(Ld * es, run_cap));
      score = score * 4 + (int)std::min<int64_t>(TE * es / 4096, 4);  // then prefer tiles up to 16 KiB
      if (score > best.score) best = Choice{Ls, Ld, TE, Vs, Vd, inc, score};
    }
  if (best.score < 0) return fail("tile: no legal tile");
  const int64_t TE = best.TE, Vs = best.Vs, Vd = best.Vd;
  if (Vs * es != 16 && Vs * es != 8 && Vs * es != 4) return fail("tile: load vector");
  // tile digit pieces and outer digits
  std::vector<Dig> tile, outer;
  for (int i = 0; i < n; i++) {
    if (best.incl[i] > 1) tile.push_back(Dig{best.incl[i], D[i].ss, D[i].ds});
    if (D[i].e / best.incl[i] > 1)
      outer.push_back(Dig{D[i].e / best.incl[i], D[i].ss * best.incl[i], D[i].ds * best.incl[i]});
  }
  tile.push_back(Dig{G, 1, 1});
  if ((int)outer.size() > K1_MAXD) return fail("tile: too many tile-index digits");
  // smem order = source order (compact strides)
  std::vector<Dig> so = tile;
  std::sort(so.begin(), so.end(), [](const Dig &a, const Dig &b) { return a.ss > b.ss; });  // outermost first
  std::vector<std::pair<int64_t, int64_t>> s_src, s_sm;
  {
    int64_t st = 1;
    std::vector<int64_t> sm(so.size());
    for (int k = (int)so.size() - 1; k >= 0; k--) {
      sm[k] = st;
      st *= so[k].e;
    }
    for (size_t k = 0; k < so.size(); k++) {
      s_src.push_back({so[k].e, so[k].ss});
      s_sm.push_back({so[k].e, sm[k]});
    }
  }
  // destination order, with each piece's smem stride
  std::vector<std::pair<int64_t, int64_t>> d_dst, d_sm;
  {
    std::vector<int> o(so.size());
    std::iota(o.begin(), o.end(), 0);
    std::sort(o.begin(), o.end(), [&](int a, int b) { return so[a].ds > so[b].ds; });
    for (int k : o) {
      d_dst.push_back({so[k].e, so[k].ds});
      d_sm.push_back({so[k].e, s_sm[k].second});
    }
  }
  K2Params &k = P->k2;
  memset(&k, 0, sizeof(k));
  k.lj = (int)(TE / (Vs * NT));
  k.sj = (int)(TE / (Vd * NT));
  k.kg = (int)(Vd / G);
  // tables (elements), then verify additivity exhaustively
  for (int t = 0; t < NT; t++) {
    k.A_l[t] = (int32_t)offset_of(s_src, (int64_t)t * Vs);
    k.A_s[t] = (int32_t)offset_of(d_sm, (int64_t)t * Vd);
    k.A_d[t] = (int32_t)offset_of(d_dst, (int64_t)t * Vd);
  }
  for (int j = 0; j < k.lj; j++) k.B_l[j] = (int32_t)offset_of(s_src, (int64_t)j * NT * Vs);
  for (int j = 0; j < k.sj; j++) {
    k.B_s[j] = (int32_t)offset_of(d_sm, (int64_t)j * NT * Vd);
    k.B_d[j] = (int32_t)offset_of(d_dst, (int64_t)j * NT * Vd);
  }
  for (int q = 0; q < k.kg; q++) k.C_s[q] = (int32_t)offset_of(d_sm, (int64_t)q * G);
  for (int64_t u = 0; u < TE / Vs; u++) {
    int64_t j = u / NT, t = u % NT;
    if (offset_of(s_src, u * Vs) != k.B_l[j] + k.A_l[t]) return fail("tile: load offsets not separable");
    for (int64_t i = 1; i < Vs; i++)
      if (offset_of(s_src, u * Vs + i) != offset_of(s_src, u * Vs) + i) return fail("tile: load vector not contiguous");
  }
  for (int64_t w = 0; w < TE / Vd; w++) {
    int64_t j = w / NT, t = w % NT;
    if (offset_of(d_dst, w * Vd) != k.B_d[j] + k.A_d[t]) return fail("tile: store offsets not separable");
    for (int64_t i = 1; i < Vd; i++)
      if (offset_of(d_dst, w * Vd + i) != offset_of(d_dst, w * Vd) + i) return fail("tile: store vector not contiguous");
    for (int q = 0; q < k.kg; q++) {
      int64_t e = offset_of(d_sm, w * Vd + q * G);
      if (e != k.B_s[j] + k.A_s[t] + k.C_s[q]) return fail("tile: gather offsets not separable");
      for (int64_t i = 1; i < G; i++)
        if (offset_of(d_sm, w * Vd + q * G + i) != e + i) return fail("tile: granule not contiguous in smem");
    }
  }
  // elements -> bytes
  for (int t = 0; t < NT; t++) {
    k.A_l[t] *= es;
    k.A_s[t] *= es;
    k.A_d[t] *= es;
  }
  for (int j = 0; j < k.lj; j++) k.B_l[j] *= es;
  for (int j = 0; j < k.sj; j++) {
    k.B_s[j] *= es;
    k.B_d[j] *= es;
  }
  for (int q = 0; q < k.kg; q++) k.C_s[q] *= es;
  // shared-memory swizzle: simulate warp 0 (and 1) for every candidate, keep the fewest wavefronts
  const int VSB = (int)(Vs * es), GBB = (int)(G * es);
  Swz bestsw{0, 0, 0};
  int bestc = 1 << 30, nonec = 0;
  for (int s = 6; s <= 13; s++) {
    Swz sw = s == 6 ? Swz{0, 0, 0} : Swz{(uint32_t)s, 7u, 4u};
    if (s > 6 && (int64_t(1) << (s + 3)) > TE * es) break;
    int c = 0;
    uint32_t a[32];
    for (int w = 0; w < 2; w++) {
      for (int j = 0; j < std::min(k.lj, 2); j++) {
        for (int t = 0; t < 32; t++) a[t] = swz_host(sw, (uint32_t)((j * NT + w * 32 + t) * VSB));
        c += wavefronts(a, VSB);
      }
      for (int j = 0; j < std::min(k.sj, 2); j++)
        for (int q = 0; q < k.kg; q++) {
          for (int t = 0; t < 32; t++) a[t] = swz_host(sw, (uint32_t)(k.A_s[w * 32 + t] + k.B_s[j] + k.C_s[q]));
          c += wavefronts(a, GBB);
        }
    }
    if (s == 6) nonec = c;
    if (c < bestc) {
      bestc = c;
      bestsw = sw;
    }
  }
  k.smsw = bestsw;
  k.ntiles = 1;
  for (auto &o : outer) k.ntiles *= (uint32_t)o.e;
  k.nout = (int)outer.size();
  {
    std::vector<Joint> oj;
    for (auto &o : outer) oj.push_back(Joint{o.e, o.ss, o.ds});
    sort_fuse_outer(oj);
    outer.clear();
    for (auto &o : oj) outer.push_back(Dig{o.e, o.ss, o.ds});
    k.nout = (int)outer.size();
  }
  for (int i = 0; i < k.nout; i++) {
    k.ofd[i] = make_fastdiv((uint32_t)outer[i].e);
    k.oss[i] = outer[i].ss * es;
    k.ods[i] = outer[i].ds * es;
  }
  k.sbase = ls.base * es;
  k.dbase = ld.base * es;
  k.tile_bytes = (uint32_t)(TE * es);
  k.ssw = make_swz(sst);
  k.dsw = make_swz(dstst);
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  P->k2_vs = VSB;
  P->k2_vd = (int)(Vd * es);
  P->k2_gb = GBB;
  P->align = 16;
  int per_sm = std::max(1, std::min(8, (int)(200 * 1024 / (TE * es + 1024))));
  if (const char *ev = getenv("AXE_K2_PER_SM")) per_sm = std::max(1, atoi(ev));  // tuning knob
  P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(k.ntiles, grid_cap(per_sm)));
  k.chunk = unit_chunk(0);
  P->blocks = chunk_grid(k.ntiles, k.chunk, P->blocks);
  int64_t total = 1;
  for (auto &j : J) total *= j.e;
  P->covers_all = (int64_t)reps.size() * total == dstst.cells;
  char b[400];
  snprintf(b, sizeof b,
           "{\"kernel\":\"tile\",\"tile_bytes\":%lld,\"tiles\":%u,\"src_run_bytes\":%lld,\"dst_run_bytes\":%lld,"
           "\"load_vec\":%d,\"store_vec\":%d,\"granule\":%d,\"smem_swizzle\":[%u,%u],\"wavefronts\":[%d,%d],"
           "\"blocks\":%u,\"replicas\":%d,\"joint\":",
           (long long)(TE * es), k.ntiles, (long long)(best.Ls * es), (long long)(best.Ld * es), VSB, P->k2_vd, GBB,
           bestsw.shift, bestsw.mask, nonec, bestc, P->blocks, k.nrep);
  P->desc = std::string(b) + joint_json(J) + "}";
  return true;
}

}  // namespace axe
