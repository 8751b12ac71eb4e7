// plan_k9.cpp -- planner of K9, the ragged 2-D transpose (kernels_k9.cu).
//
// The copy qualifies when its joint digits contain a digit a contiguous on the source (source stride 1)
// and a digit b contiguous on the destination (destination stride 1) -- a 2-D transpose -- with any
// extents and pitches; every other digit indexes tiles (a batch).  The paper's dispatch matches layouts
// against instruction atoms; this atom is the element-granular shared-memory tile transpose,
// the fallback of K7 when whole 16-byte vectors or whole tiles are not available.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "plan.hpp"

namespace axe {

int num_sms();
int k9_tile_a(int es);
int k9_tile_b();

bool build_k9(const std::vector<Joint> &J0, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, CopyPlan *P, std::string *why) {
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  std::vector<Joint> J;
  for (auto &j : J0)
    if (j.e > 1) J.push_back(j);
  int a = -1, b = -1;
  for (int i = 0; i < (int)J.size(); i++) {
    if (J[i].ss == 1 && J[i].ds != 1) a = i;
    if (J[i].ds == 1 && J[i].ss != 1) b = i;
  }
  if (a < 0 || b < 0) return fail("ragged transpose: no source-contiguous and destination-contiguous digit pair");
  std::vector<Joint> batch;
  for (int i = 0; i < (int)J.size(); i++)
    if (i != a && i != b) batch.push_back(J[i]);
  if ((int)batch.size() > K1_MAXD) return fail("ragged transpose: too many batch digits");
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
  if ((int)reps.size() > K1_MAXREP) return fail("ragged transpose: too many replicas");
  const Joint A = J[a], B = J[b];
  const int64_t TA = k9_tile_a(es), TB = k9_tile_b();
  const int64_t na = (A.e + TA - 1) / TA, nb = (B.e + TB - 1) / TB;
  int64_t nt = na * nb;
  for (auto &j : batch) nt *= j.e;
  if (nt >= (int64_t(1) << 31) || na >= (int64_t(1) << 31) || nb >= (int64_t(1) << 31))
    return fail("ragged transpose: too many tiles");
  K9Params &k = P->k9;
  memset(&k, 0, sizeof(k));
  k.ntiles = (uint32_t)nt;
  k.fa = make_fastdiv((uint32_t)na);
  k.fb = make_fastdiv((uint32_t)nb);
  k.nd = (int)batch.size();
  for (int i = 0; i < k.nd; i++) {
    k.fd[i] = make_fastdiv((uint32_t)batch[i].e);
    k.ss[i] = batch[i].ss * es;
    k.ds[i] = batch[i].ds * es;
  }
  k.ea = A.e;
  k.eb = B.e;
  k.s_b = B.ss * es;
  k.d_a = A.ds * es;
  k.sbase = ls.base * es;
  k.dbase = ld.base * es;
  k.ssw = make_swz(sst);
  k.dsw = make_swz(dstst);
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  // vector-load form: source buffers 16-byte aligned (the plan's alignment), 1..8-byte elements, the
  // source pitch positive (rows fetched as whole 16-byte chunks)
  const char *ve = getenv("AXE_K9_VEC");
  k.vec = (es <= 8 && B.ss > 0 && !(ve && *ve == '0')) ? 1 : 0;
  k.src_limit = (sst.cells * es + 15) / 16 * 16;
  // one tile per CTA over a covering grid once the tiles outnumber a wave (in-order schedule,
  // profiles/r02_sweep_front.log: 4095 x 4097 bf16 29.3 us vs 31.1, u8 8191 x 8193 91.0 vs 100.8)
  k.chunk = unit_chunk(nt > (int64_t)num_sms() * 8 ? 1 : 0);
  P->align = k.vec ? 16 : es;
  int64_t total = 1;
  for (auto &j : J0) total *= j.e;
  P->covers_all = (int64_t)reps.size() * total == dstst.cells;
  char buf[256];
  snprintf(buf, sizeof buf,
           "{\"kernel\":\"transpose\",\"mode\":\"ragged\",\"vector_loads\":%d,\"tile\":[%lld,%lld],\"tiles\":%lld,"
           "\"chunk\":%u,\"replicas\":%d,\"joint\":",
           k.vec, (long long)TB, (long long)TA, (long long)nt, k.chunk, k.nrep);
  P->desc = std::string(buf) + joint_json(J0) + "}";
  return true;
}

}  // namespace axe
