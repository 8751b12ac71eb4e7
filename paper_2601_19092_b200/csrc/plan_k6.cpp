// plan_k6.cpp -- planner of K6, the granule transpose across lane groups.
//
// After joint refinement (element strides) the copy qualifies when:
//   * the innermost joint digit is a run contiguous on both sides of G bytes,
//     G = 4 or 8 (the granule; n = 16 / G granules per 16-byte vector);
//   * a digit A of extent n steps 16 bytes on the source (the next source
//     vector) and G bytes on the destination (the next granule of the same
//     destination vector);
//   * digits B (extent product n) step through the granules of one source
//     vector (source strides G, 2G, ...) and land in whole destination vectors;
//   * every other digit ("group" digits) moves whole 16-byte vectors on both
//     sides.
// Then n source vectors of a group form an n x n granule matrix whose
// transpose is n destination vectors (K6, kernels_k6.cu).  The paper's
// dispatch picks an instruction-level schedule by matching the layout against
// an atom (App. D); this atom is the warp-shuffle transpose.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "plan.hpp"

namespace axe {

Swz make_swz(const Storage &st);
int num_sms();

bool build_k6(const std::vector<Joint> &J0, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why) {
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  if (max_align < 16) return fail("shuffle: needs 16-byte aligned buffers");
  if ((sst.swz_b && sst.swz_m < 4) || (dstst.swz_b && dstst.swz_m < 4)) return fail("shuffle: swizzle below 16 bytes");
  std::vector<Joint> J;
  for (auto &j : J0)
    if (j.e > 1) J.push_back(j);
  if (J.empty()) return fail("shuffle: empty");
  int64_t run = 1;  // the granule: innermost run contiguous on both sides (elements)
  if (J.back().ss == 1 && J.back().ds == 1) {
    run = J.back().e;
    J.pop_back();
  }
  const int64_t G = run * es;
  if (G != 4 && G != 8) return fail("shuffle: granule is not 4 or 8 bytes");
  const int n = (int)(16 / G);
  const int64_t vs = 16 / es;  // elements per 16-byte vector
  // digit A: extent n, source stride one vector, destination stride one granule
  int a = -1;
  for (int i = 0; i < (int)J.size(); i++)
    if (J[i].e == n && J[i].ss == vs && J[i].ds == run) a = i;
  if (a < 0) return fail("shuffle: no digit steps source vectors and destination granules");
  // digits B: source strides inside one vector (multiples of the granule), destination whole vectors
  std::vector<Joint> B, grp;
  int64_t bprod = 1;
  for (int i = 0; i < (int)J.size(); i++) {
    if (i == a) continue;
    const Joint &j = J[i];
    if (j.ss > 0 && j.ss % run == 0 && (j.e - 1) * j.ss < vs && j.ds % vs == 0) {
      B.push_back(j);
      bprod *= j.e;
    } else if (j.ss % vs == 0 && j.ds % vs == 0) {
      grp.push_back(j);
    } else {
      return fail("shuffle: a digit splits a 16-byte vector");
    }
  }
  if (bprod != n) return fail("shuffle: the granule digits do not cover a vector");
  // granule position p (source offset p * run inside the vector) -> destination offset of its vector
  int64_t dpos[4] = {-1, -1, -1, -1};
  for (int64_t c = 0; c < n; c++) {
    int64_t rem = c, so = 0, dof = 0;
    for (int k = (int)B.size() - 1; k >= 0; k--) {
      const int64_t d = rem % B[k].e;
      rem /= B[k].e;
      so += d * B[k].ss;
      dof += d * B[k].ds;
    }
    const int64_t p = so / run;
    if (so % run || p < 0 || p >= n || dpos[p] >= 0) return fail("shuffle: granule digits are not a permutation");
    dpos[p] = dof;
  }
  if (ls.base % vs || ld.base % vs) return fail("shuffle: bases are not 16-byte aligned");
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
  if ((int)reps.size() > K1_MAXREP) return fail("shuffle: too many replicas");
  for (int64_t r : reps)
    if (r % vs) return fail("shuffle: replica offsets not 16-byte aligned");
  // group digits: destination-contiguous first (consecutive groups store consecutive vectors)
  std::stable_sort(grp.begin(), grp.end(), [](const Joint &x, const Joint &y) { return std::llabs(x.ds) > std::llabs(y.ds); });
  sort_fuse_outer(grp);
  int64_t ng = 1;
  for (auto &g : grp) ng *= g.e;
  if (ng >= (int64_t(1) << 31)) return fail("shuffle: too many groups");
  // tiles of (256 / n) * K6_U groups: the innermost group digits (split where needed, Lemma split)
  const int64_t tile_g = (256 / n) * K6_U;
  if (ng % tile_g) return fail("shuffle: group count is not a whole number of tiles");
  std::vector<Joint> inner, outer, rest(grp.rbegin(), grp.rend());  // rest: innermost first
  int64_t prefix = 1;
  size_t q = 0;
  while (prefix < tile_g && q < rest.size()) {
    const int64_t need = tile_g / prefix;
    Joint jj = rest[q];
    const int64_t g = std::gcd(jj.e, need);
    if (g == jj.e) {
      inner.push_back(jj);
      prefix *= jj.e;
      q++;
    } else if (g > 1) {
      inner.push_back(Joint{g, jj.ss, jj.ds});
      rest[q] = Joint{jj.e / g, jj.ss * g, jj.ds * g};
      prefix *= g;
    } else {
      break;
    }
  }
  if (prefix != tile_g) return fail("shuffle: no tile boundary in the group digits");
  for (; q < rest.size(); q++) outer.push_back(rest[q]);
  std::reverse(inner.begin(), inner.end());  // outermost first
  std::reverse(outer.begin(), outer.end());
  sort_fuse_outer(outer);
  if ((int)inner.size() > K1_MAXD || (int)outer.size() > K1_MAXD) return fail("shuffle: too many group digits");
  K6Params &k = P->k6;
  memset(&k, 0, sizeof(k));
  k.ngroups = (uint32_t)ng;
  k.n = n;
  k.tile_g = (uint32_t)tile_g;
  k.ntiles = (uint32_t)(ng / tile_g);
  k.nin = (int)inner.size();
  for (int i = 0; i < k.nin; i++) {
    k.ifd[i] = make_fastdiv((uint32_t)inner[i].e);
    k.iss[i] = inner[i].ss * es;
    k.ids[i] = inner[i].ds * es;
  }
  k.nout = (int)outer.size();
  for (int i = 0; i < k.nout; i++) {
    k.ofd[i] = make_fastdiv((uint32_t)outer[i].e);
    k.oss[i] = outer[i].ss * es;
    k.ods[i] = outer[i].ds * es;
  }
  k.sbase = ls.base * es;
  k.dbase = ld.base * es;
  k.sstep = J[a].ss * es;
  for (int p = 0; p < n; p++) k.dpos[p] = dpos[p] * es;
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  k.ssw = make_swz(sst);
  k.dsw = make_swz(dstst);
  P->align = 16;
  P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(k.ntiles, grid_cap(8)));
  // in-order schedule, 4 tiles (of 4 groups per thread) per CTA, when the tiles outnumber the persistent
  // grid (config 3a: 1277 us vs 1364 persistent, profiles/r02_sweep_front.log)
  k.chunk = unit_chunk(k.ntiles > (int64_t)P->blocks ? 4 : 0);
  P->blocks = chunk_grid(k.ntiles, k.chunk, P->blocks);
  int64_t total = ng * n * n;  // granules
  P->covers_all = (int64_t)reps.size() * total * run == dstst.cells;
  char b[256];
  snprintf(b, sizeof b,
           "{\"kernel\":\"shuffle\",\"atom\":\"%dx%d transpose of %lld-byte granules across lanes\",\"groups\":%lld,"
           "\"ctas\":%u,\"replicas\":%d,\"joint\":",
           n, n, (long long)G, (long long)ng, P->blocks, k.nrep);
  P->desc = std::string(b) + joint_json(J0) + "}";
  return true;
}

}  // namespace axe
