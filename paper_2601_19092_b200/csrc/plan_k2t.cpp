// plan_k2t.cpp -- planner of K2T, the TMA-staged transpose (source-contiguous
// and destination-contiguous digits differ).  The staging tile is one TMA box
// of H rows x 128 bytes along the source-contiguous digit, loaded with the
// 128-byte swizzle (the TMA atom of P:527) so that the gather along the
// destination-contiguous digit, done by lanes walking one 128-byte row, hits
// distinct banks.  Remaining digits index boxes (tensor-map dimensions on the
// source side, byte strides on the destination side).
#include <algorithm>
#include <cstring>

#include "plan.hpp"

namespace axe {

int num_sms();

bool build_k2t(const std::vector<Joint> &J, const Linear &ls, const Linear &ld, const Storage &sst,
               const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why) {
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  if (es != 2 && es != 4 && es != 8) return fail("tma_tile: element size");
  if (max_align < 16) return fail("tma_tile: needs 16-byte aligned buffers");
  if (sst.swz_b || dstst.swz_b) return fail("tma_tile: swizzled storages");
  int is = -1, id = -1;
  for (size_t i = 0; i < J.size(); i++) {
    if (J[i].ss <= 0 || J[i].ds <= 0) return fail("tma_tile: negative strides");
    if (J[i].e == 1) continue;
    if (J[i].ss == 1 && J[i].ds == 1) return fail("tma_tile: a run is contiguous on both sides (vector copy)");
    if (J[i].ss == 1) is = (int)i;
    if (J[i].ds == 1) id = (int)i;
  }
  if (is < 0 || id < 0) return fail("tma_tile: no source- or destination-contiguous digit");
  const Joint Ds = J[is], Dd = J[id];
  const int64_t W = 128 / es, VD = 16 / es;
  if (Ds.e % W) return fail("tma_tile: source run is not a multiple of 128 bytes");
  int64_t H = 0;
  for (int64_t h : {64, 32, 16})
    if (Dd.e % h == 0 && h % VD == 0) {
      H = h;
      break;
    }
  if (!H) return fail("tma_tile: destination run too short");
  if ((Dd.ss * es) % 16) return fail("tma_tile: row stride not a multiple of 16 bytes");
  if ((ls.base * es) % 16 || (ld.base * es) % 16 || (Ds.ds * es) % 16) return fail("tma_tile: 16-byte alignment");
  std::vector<int64_t> reps{0};
  for (auto &r : ld.R) {
    std::vector<int64_t> nx;
    for (int64_t b : reps)
      for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
    reps.swap(nx);
  }
  std::sort(reps.begin(), reps.end());
  reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
  if ((int)reps.size() > K1_MAXREP) return fail("tma_tile: too many replicas");
  for (int64_t r : reps)
    if ((r * es) % 16) return fail("tma_tile: replica offsets not 16-byte aligned");
  // tensor map (byte elements): dim0 = the source-contiguous digit in bytes, dim1 = the
  // destination-contiguous digit, dims 2..4 = the other digits
  std::vector<std::array<int64_t, 4>> digs;  // extent, cdim, cmul, dst byte stride (innermost first)
  if (Ds.e / W > 1) digs.push_back({Ds.e / W, 0, 128, W * Ds.ds * es});
  if (Dd.e / H > 1) digs.push_back({Dd.e / H, 1, H, H * es});
  P->tm_dims[0] = (uint64_t)(Ds.e * es);
  P->tm_box[0] = 128;
  P->tm_dims[1] = (uint64_t)Dd.e;
  P->tm_strides[0] = (uint64_t)(Dd.ss * es);
  P->tm_box[1] = (uint32_t)H;
  int dim = 2;
  for (size_t i = 0; i < J.size(); i++) {
    if ((int)i == is || (int)i == id || J[i].e == 1) continue;
    if (dim > 4) return fail("tma_tile: more than 5 tensor dimensions");
    if ((J[i].ss * es) % 16 || (J[i].ds * es) % 16) return fail("tma_tile: outer stride not a multiple of 16 bytes");
    P->tm_dims[dim] = (uint64_t)J[i].e;
    P->tm_strides[dim - 1] = (uint64_t)(J[i].ss * es);
    P->tm_box[dim] = 1;
    digs.push_back({J[i].e, dim, 1, J[i].ds * es});
    dim++;
  }
  for (int i = dim; i < 5; i++) {
    P->tm_dims[i] = 1;
    P->tm_box[i] = 1;
    P->tm_strides[i - 1] = P->tm_strides[0];
  }
  if ((int)digs.size() > TMA_MAXD) return fail("tma_tile: too many box digits");
  // boxes in destination order: the smallest destination stride fastest
  std::stable_sort(digs.begin(), digs.end(), [](const std::array<int64_t, 4> &a, const std::array<int64_t, 4> &b) {
    return a[3] < b[3];
  });
  int64_t nt = 1;
  for (auto &g : digs) nt *= g[0];
  if (nt >= (int64_t(1) << 31)) return fail("tma_tile: too many tiles");
  K2TParams &k = P->k2t;
  memset(&k, 0, sizeof(k));
  k.ntiles = (uint32_t)nt;
  k.nd = (int)digs.size();
  for (int i = 0; i < k.nd; i++) {
    auto &g = digs[digs.size() - 1 - i];
    k.fd[i] = make_fastdiv((uint32_t)g[0]);
    k.cdim[i] = (int32_t)g[1];
    k.cmul[i] = (int32_t)g[2];
    k.dstride[i] = g[3];
  }
  k.dbase = ld.base * es;
  k.W = (uint32_t)W;
  k.H = (uint32_t)H;
  k.dcol = Ds.ds * es;
  k.stages = 4;
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  P->tm_swizzle = 128;
  P->tm_base = ls.base * es;
  P->tm_cache = std::make_shared<TmaCache>();
  P->align = 16;
  int per_sm = (int)std::max<int64_t>(1, std::min<int64_t>(8, (200 * 1024) / (int64_t)k2t_smem_bytes(k)));
  P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nt, (int64_t)num_sms() * per_sm));
  int64_t total = 1;
  for (auto &j : J) total *= j.e;
  P->covers_all = (int64_t)reps.size() * total == dstst.cells;
  char b[256];
  snprintf(b, sizeof b,
           "{\"kernel\":\"tma_tile\",\"box\":[%lld,128],\"tiles\":%lld,\"stages\":%d,\"blocks\":%u,\"replicas\":%d,"
           "\"joint\":",
           (long long)H, (long long)nt, k.stages, P->blocks, k.nrep);
  P->desc = std::string(b) + joint_json(J) + "}";
  return true;
}

}  // namespace axe
