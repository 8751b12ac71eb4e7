// plan_k7.cpp -- planner of K7, the register-block transpose (kernels_k7.cu).
//
// The copy qualifies when its joint digits (element strides) contain a digit a
// contiguous on the source (source stride 1: the columns of a source row) and
// a digit b contiguous on the destination (destination stride 1: the rows of a
// destination column) -- a 2-D transpose -- with 2-, 4- or 8-byte elements,
// both extents whole 16-byte vectors (multiples of n = 16 / es elements), and every other
// digit (and both row / column pitches) moving whole 16-byte vectors.  The tiles are
// (32 n rows) x (8 n cw columns); the other digits and the outer parts of a and b index
// tiles, and a last tile row / column only partly inside the extents is masked (ragged
// edges: the rows / columns past the extent are neither read nor written).  The paper's dispatch matches layouts against instruction
// atoms; this atom is LDS.128 + an n x n register transpose.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "plan.hpp"

namespace axe {

int num_sms();

static int env_i7(const char *name, int dflt) {
  const char *e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

bool build_k7(const std::vector<Joint> &J0, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why, bool forced) {
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  if (es != 2 && es != 4 && es != 8) return fail("transpose: 2-, 4- or 8-byte elements");
  if (max_align < 16) return fail("transpose: needs 16-byte aligned buffers");
  if (sst.swz_b || dstst.swz_b) return fail("transpose: swizzled storage");
  const int64_t n = 16 / es;
  // chunk columns per warp (tiles of 32 n rows x 8 n cw columns), as wide as the columns allow:
  // 4 for 4-byte elements (8192^2 fp32: 94.9 us vs 100.8 / 104.3 with 2 / 1), 2 otherwise (bf16:
  // 43.2 us vs 44.9 with 1; 8192x4096 fp64: 94.1 us vs 98.6 with 4)
  // The cp.async double-buffered form (next tile in flight while the current one is stored): fp32
  // (cw 2) 93.3 us vs 95.8 register-staged (cw 4) / 101.7 (cw 2); bf16 (cw 2) 42.4 vs 42.9; fp64 (cw 4,
  // 64 x 64 tiles) 92.8 vs 94.5 register-staged (cw 2) / 94.6 (async, cw 2)
  // async = cp.async ring stages (2..4; 0: register-staged)
  const char *ae = getenv("AXE_K7_ASYNC");
  int async = (ae && *ae) ? std::max(0, std::min(4, atoi(ae))) : 2;
  if (async == 1) async = 2;  // (1 meant "double-buffered" before the ring depth was a knob)
  const char *cwe = getenv("AXE_K7_CW");
  const int cwmax = es == 2 ? 2 : 4;
  // (bf16 with the in-order schedule, profiles/r02_sweep_front.log: cw 1 32 MiB 10.7 us vs 12.8 with cw 2,
  // 128 MiB 43.4 vs 44.6, 256 MiB 85.9 vs 87.9 -- 32 KiB tiles fit 3 CTAs per SM)
  const int cwdef = async ? (es == 8 ? 4 : es == 4 ? 2 : 1) : (es == 4 ? 4 : 2);
  int64_t cw = (cwe && *cwe) ? std::max(1, std::min(cwmax, atoi(cwe))) : cwdef;
  std::vector<Joint> J;
  for (auto &j : J0)
    if (j.e > 1) J.push_back(j);
  int a = -1, b = -1;
  for (int i = 0; i < (int)J.size(); i++) {
    if (J[i].ss == 1 && J[i].ds != 1) a = i;
    if (J[i].ds == 1 && J[i].ss != 1) b = i;
  }
  if (a < 0 || b < 0) return fail("transpose: no source-contiguous and destination-contiguous digit pair");
  const Joint A = J[a], B = J[b];
  while (cw > 1 && A.e % (8 * n * cw)) cw /= 2;
  const int64_t TC = 8 * n * cw, TR = 32 * n;
  // ragged edges (a last tile column / row only partly inside): whole 16-byte vectors on both sides
  if (A.e % n || B.e % n) return fail("transpose: extents are not whole 16-byte vectors");
  const bool rag_a = A.e % TC != 0, rag_b = B.e % TR != 0;
  if ((rag_a || rag_b) && !env_i7("AXE_K7_RAGGED", 1)) return fail("transpose: extents are not whole tiles");
  // AUTO: ragged tiles only while at least half of every tile's area is inside (a skinny transpose is
  // better served by K2 / K1); forced: any
  if ((rag_a || rag_b) && !forced &&
      2 * A.e * B.e < ((A.e + TC - 1) / TC * TC) * ((B.e + TR - 1) / TR * TR))
    return fail("transpose: ragged tiles less than half inside");
  auto v16 = [&](int64_t s) { return (s * es) % 16 == 0; };
  if (!v16(A.ds) || !v16(B.ss) || A.ds < 0 || B.ss < 0) return fail("transpose: row / column pitch not 16-byte aligned");
  if (!v16(ls.base) || !v16(ld.base)) return fail("transpose: bases not 16-byte aligned");
  std::vector<Joint> outer;
  for (int i = 0; i < (int)J.size(); i++) {
    if (i == a || i == b) continue;
    if (!v16(J[i].ss) || !v16(J[i].ds)) return fail("transpose: a digit moves partial vectors");
    outer.push_back(J[i]);
  }
  const int64_t nta = (A.e + TC - 1) / TC, ntb = (B.e + TR - 1) / TR;
  const Joint TA{nta, TC, TC * A.ds}, TB{ntb, TR * B.ss, TR};
  if (nta > 1) outer.push_back(TA);
  if (ntb > 1) outer.push_back(TB);
  std::stable_sort(outer.begin(), outer.end(), [](const Joint &x, const Joint &y) { return std::llabs(x.ds) > std::llabs(y.ds); });
  sort_fuse_outer(outer);
  // tiles in source order: consecutive tiles (a CTA's chunk, neighbouring CTAs) continue the same source
  // rows (bf16 8192^2 42.5 us vs 43.5 in destination order, 256 MiB 83.4 vs 85.9; fp32 1-2%;
  // profiles/r02_sweep_front.log).  AXE_K7_ORDER=0: destination order
  if (env_i7("AXE_K7_ORDER", 1) == 1)
    std::stable_sort(outer.begin(), outer.end(), [](const Joint &x, const Joint &y) { return std::llabs(x.ss) > std::llabs(y.ss); });
  // the ragged sides' tile digits, found again after the fusion (a fused one cannot be masked)
  auto find = [&](const Joint &t) {
    for (int i = 0; i < (int)outer.size(); i++)
      if (outer[i].e == t.e && outer[i].ss == t.ss && outer[i].ds == t.ds) return i;
    return -1;
  };
  // (a side of less than one tile has no digit: tile_offsets applies its limit to every tile)
  const int ka = rag_a && nta > 1 ? find(TA) : -1, kb = rag_b && ntb > 1 ? find(TB) : -1;
  if ((int)outer.size() > K1_MAXD) return fail("transpose: too many tile digits");
  int64_t nt = 1;
  for (auto &o : outer) nt *= o.e;
  if (nt >= (int64_t(1) << 31)) return fail("transpose: too many tiles");
  std::vector<int64_t> reps{0};
  for (auto &r : ld.R) {
    std::vector<int64_t> nx;
    for (int64_t x : reps)
      for (int64_t d = 0; d < r.e; d++) nx.push_back(x + d * r.s);
    reps.swap(nx);
    if (reps.size() > 4096) break;
  }
  std::sort(reps.begin(), reps.end());
  reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
  if ((int)reps.size() > K1_MAXREP) return fail("transpose: too many replicas");
  for (int64_t r : reps)
    if (!v16(r)) return fail("transpose: replica offsets not 16-byte aligned");
  if ((rag_a && nta > 1 && ka < 0) || (rag_b && ntb > 1 && kb < 0))
    return fail("transpose: a ragged tile digit fused with another");
  K7Params &k = P->k7;
  memset(&k, 0, sizeof(k));
  k.ntiles = (uint32_t)nt;
  k.ka = ka;
  k.kb = kb;
  k.lim_a = (uint32_t)(rag_a ? A.e : TC);
  k.lim_b = (uint32_t)(rag_b ? B.e : TR);
  k.nd = (int)outer.size();
  for (int i = 0; i < k.nd; i++) {
    k.fd[i] = make_fastdiv((uint32_t)outer[i].e);
    k.ss[i] = outer[i].ss * es;
    k.ds[i] = outer[i].ds * es;
  }
  k.sbase = ls.base * es;
  k.dbase = ld.base * es;
  k.src_row = B.ss * es;
  k.dst_col = A.ds * es;
  k.cw = (int)cw;
  while (async > 2 && TR * TC * es * async > 200 * 1024) async--;  // the ring must fit in shared memory
  if (async && TR * TC * es * async > 200 * 1024) return fail("transpose: tile ring exceeds shared memory");
  k.async = async;
  {  // opt-in streaming stores: no gain on a B200 (fp32 8192^2 93.9-94.1 us vs 93.3; fp64 93.7-94.0 vs 93.2)
    const char *se = getenv("AXE_K7_STCS");
    k.stcs = (se && *se) ? (atoi(se) != 0) : 0;
  }
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  P->align = 16;
  const int64_t tile_bytes = TR * TC * es * (k.async ? k.async : 1);
  const int per_sm = (int)std::max<int64_t>(1, std::min<int64_t>(8, (220 * 1024) / (tile_bytes + 1024)));
  P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nt, grid_cap(per_sm)));
  // from 64 MiB a side (256 MiB with one CTA per SM), the in-order schedule: 1 tile per CTA, 4 when one
  // CTA fills the SM and its own ring is the only overlap (profiles/r02_sweep_front.log: 256 MiB fp32
  // 82.0 us vs 92.4 persistent with 2 tiles per CTA, 80.4 with 1 in source-major order; bf16 one CTA per
  // SM 88.0 vs 97.8; at 32 MiB the persistent grid wins, 10.5 vs 11.4, and so does one-CTA bf16 at
  // 128 MiB, 43.8 vs 48.1)
  const int64_t bytes = nt * TR * TC * es;
  const bool front = per_sm >= 2 ? bytes >= (int64_t(64) << 20) : bytes >= (int64_t(256) << 20);
  k.chunk = unit_chunk(front && nt > (int64_t)P->blocks ? (per_sm >= 2 ? 1 : 4) : 0);
  P->blocks = chunk_grid(nt, k.chunk, P->blocks);
  const char *mc = getenv("AXE_K7_MAX_CTAS");  // tests: several tiles per CTA on small inputs
  if (mc && *mc && atoi(mc) > 0) {  // (persistent grid: a capped chunked grid would drop tiles)
    k.chunk = 0;
    P->blocks = std::min<unsigned>(std::min<unsigned>(P->blocks, (unsigned)(num_sms() * per_sm)), (unsigned)atoi(mc));
  }
  int64_t total = 1;
  for (auto &j : J0) total *= j.e;
  P->covers_all = (int64_t)reps.size() * total == dstst.cells;
  char buf[256];
  snprintf(buf, sizeof buf,
           "{\"kernel\":\"transpose\",\"block\":\"%lldx%lld register transpose\",\"tile\":[%lld,%lld],\"tiles\":%lld,"
           "\"ctas\":%u,\"chunk\":%u,\"replicas\":%d,\"async\":%d,\"joint\":",
           (long long)n, (long long)n, (long long)TR, (long long)TC, (long long)nt, P->blocks, k.chunk, k.nrep, k.async);
  P->desc = std::string(buf) + joint_json(J0) + "}";
  return true;
}

}  // namespace axe
