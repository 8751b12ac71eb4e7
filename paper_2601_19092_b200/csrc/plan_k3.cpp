// plan_k3.cpp -- planner of K3, the movmatrix register permute.
//
// The copy qualifies when (after joint refinement, element strides) its digits
// split into in-block digits acting inside 256-element (512-byte) blocks and
// block digits whose strides are whole blocks on both sides, and when the
// in-block map equals the movmatrix.m8n8.trans.b16 atom applied to every
// 32-bit register of a 32-lane x 8-register warp row: element (lane, 2q + v)
// with lane = 4i + j goes to (4 (2j + v) + i/2, 2q + i mod 2).  This is the
// "tile of an instruction atom" test of the paper's dispatch (P:519-536,
// App. D) for one concrete atom.
#include <algorithm>
#include <cstring>

#include "plan.hpp"

#include <cstdlib>

namespace axe {

Swz make_swz(const Storage &st);
int num_sms();

static int64_t movm_atom(int64_t e) {  // in-block element offset -> destination offset
  int64_t lane = e / 8, lo = e % 8, q = lo / 2, v = lo % 2;
  int64_t i = lane / 4, j = lane % 4;
  return (4 * (2 * j + v) + i / 2) * 8 + 2 * q + (i % 2);
}

bool build_k3(const std::vector<Joint> &J, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why) {
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  if (es != 2) return fail("register: movmatrix moves b16 elements");
  if (max_align < 16) return fail("register: needs 16-byte aligned buffers");
  if ((sst.swz_b && sst.swz_m < 4) || (dstst.swz_b && dstst.swz_m < 4)) return fail("register: swizzle below 16 bytes");
  const int64_t BLK = 256;
  if (ls.base % BLK || ld.base % BLK) return fail("register: bases are not whole blocks");
  std::vector<int64_t> reps{0};
  for (auto &r : ld.R) {
    std::vector<int64_t> nx;
    for (int64_t b : reps)
      for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
    reps.swap(nx);
  }
  std::sort(reps.begin(), reps.end());
  reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
  if ((int)reps.size() > K1_MAXREP) return fail("register: too many replicas");
  for (int64_t r : reps)
    if (r % 8) return fail("register: replica offsets not 16-byte aligned");
  std::vector<Joint> in, out;
  int64_t inprod = 1;
  for (auto &j : J) {
    if (j.e == 1) continue;
    if (j.ss > 0 && j.ds > 0 && (j.e - 1) * j.ss < BLK && (j.e - 1) * j.ds < BLK) {
      in.push_back(j);
      inprod *= j.e;
    } else if (j.ss % BLK == 0 && j.ds % BLK == 0) {
      out.push_back(j);
    } else {
      return fail("register: a digit straddles the 512-byte blocks");
    }
  }
  if (inprod != BLK) return fail("register: in-block digits do not cover a warp row");
  std::vector<int> seen(BLK, 0);
  for (int64_t x = 0; x < BLK; x++) {
    int64_t rem = x, s = 0, d = 0;
    for (int k = (int)in.size() - 1; k >= 0; k--) {
      int64_t dg = rem % in[k].e;
      rem /= in[k].e;
      s += dg * in[k].ss;
      d += dg * in[k].ds;
    }
    if (s < 0 || s >= BLK || seen[s]) return fail("register: in-block map is not a permutation");
    seen[s] = 1;
    if (movm_atom(s) != d) return fail("register: in-block map is not the movmatrix atom");
  }
  if ((int)out.size() > K1_MAXD) return fail("register: too many block digits");
  int64_t nb = 1;
  for (auto &o : out) nb *= o.e;
  if (nb >= (int64_t(1) << 31)) return fail("register: too many blocks");
  K3Params &k = P->k3;
  memset(&k, 0, sizeof(k));
  sort_fuse_outer(out);
  k.nblocks = (uint32_t)nb;
  k.nd = (int)out.size();
  for (int i = 0; i < k.nd; i++) {
    k.fd[i] = make_fastdiv((uint32_t)out[i].e);
    k.ss[i] = out[i].ss * es;
    k.ds[i] = out[i].ds * es;
  }
  k.sbase = ls.base * es;
  k.dbase = ld.base * es;
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  k.ssw = make_swz(sst);
  k.dsw = make_swz(dstst);
  P->align = 16;
  const int64_t per_cta = 8;  // warps x blocks per warp per iteration (AXE_K3_U = 1)
  const char *ev = getenv("AXE_K3_PER_SM");  // CTAs per SM (tuning knob)
  const int64_t per_sm = (ev && *ev) ? std::max(1, atoi(ev)) : 8;
  P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nb + per_cta - 1) / per_cta, (int64_t)num_sms() * per_sm));
  P->covers_all = (int64_t)reps.size() * nb * BLK == dstst.cells;
  char b[256];
  snprintf(b, sizeof b,
           "{\"kernel\":\"register\",\"atom\":\"movmatrix.m8n8.trans.b16\",\"blocks_512B\":%lld,\"ctas\":%u,"
           "\"replicas\":%d,\"joint\":",
           (long long)nb, P->blocks, k.nrep);
  P->desc = std::string(b) + joint_json(J) + "}";
  return true;
}

// K3-TMA: the K3 copy with its 512-byte blocks moved by cp.async.bulk -- boxes of up to 32 blocks
// (16 KiB) where consecutive blocks are contiguous on both sides; the warp applies the movmatrix atom
// to the box in shared memory between the bulk load and the bulk store (TmaParams.xform).
size_t tma_smem_bytes(const TmaParams &p);
bool build_k3_bulk(CopyPlan *P, std::string *why) {
  auto fail = [&](const char *m) {
    *why = m;
    return false;
  };
  const K3Params &k = P->k3;
  if (k.ssw.mask || k.dsw.mask) return fail("k3-tma: swizzled storage");
  struct D3 {
    int64_t e, ss, ds;
  };
  std::vector<D3> D;
  for (int i = 0; i < k.nd; i++) D.push_back(D3{(int64_t)k.fd[i].d, k.ss[i], k.ds[i]});
  // a digit whose blocks are consecutive on both sides (byte stride 512) gives the box run
  int r = -1;
  for (int i = 0; i < (int)D.size(); i++)
    if (D[i].ss == 512 && D[i].ds == 512) r = i;
  if (r < 0) return fail("k3-tma: no run of blocks contiguous on both sides");
  // 512-byte blocks per box: 16 (8 KiB boxes, 2 stages, 8 CTAs/SM) measured 1297 us on config 3b
  // against 1381 us with 16 KiB boxes and 1417-2569 us with 4 KiB boxes
  const char *bbe = getenv("AXE_K3_TMA_BOX_BLOCKS");
  const int64_t bmax = (bbe && *bbe) ? std::max(1, atoi(bbe)) : 16;
  int64_t bb = 1;
  for (int64_t c = 1; c <= bmax; c++)
    if (D[r].e % c == 0) bb = c;
  if (bb < 4) return fail("k3-tma: box under 2 KiB");  // (a run whose extent has no divisor 4..16)
  std::vector<D3> B;
  for (int i = 0; i < (int)D.size(); i++) {
    if (i == r) {
      if (D[i].e / bb > 1) B.push_back(D3{D[i].e / bb, 512 * bb, 512 * bb});
    } else {
      B.push_back(D[i]);
    }
  }
  if ((int)B.size() > TMA_MAXD) return fail("k3-tma: too many box digits");
  int64_t nboxes = 1;
  for (auto &d : B) nboxes *= d.e;
  TmaParams &t = P->tma;
  memset(&t, 0, sizeof(t));
  t.nboxes = (uint32_t)nboxes;
  t.nd = (int)B.size();
  for (int i = 0; i < t.nd; i++) {
    t.fd[i] = make_fastdiv((uint32_t)B[i].e);
    t.cdim[i] = -1;
    t.bstride[i] = B[i].ds;
    t.sstride[i] = B[i].ss;
  }
  t.bbase = k.dbase;
  t.sbase = k.sbase;
  t.box_bytes = (uint32_t)(512 * bb);
  t.slot_bytes = (uint32_t)((t.box_bytes + 127) / 128 * 128);
  t.mode = 2;
  t.xform = 1;
  t.nrep = k.nrep;
  for (int i = 0; i < k.nrep; i++) t.rep[i] = k.rep[i];
  const char *sb = getenv("AXE_TMA_STAGE_BYTES");
  const int64_t stage_bytes = (sb && *sb) ? atoll(sb) : 16384;
  t.stages = (int)std::max<int64_t>(2, std::min<int64_t>(16, stage_bytes / t.slot_bytes));
  const char *ps = getenv("AXE_K3_TMA_PER_SM");
  int per_sm = (int)std::max<int64_t>(1, std::min<int64_t>(16, (220 * 1024) / (int64_t)tma_smem_bytes(t)));
  per_sm = std::min(per_sm, (ps && *ps) ? std::max(1, atoi(ps)) : 8);
  P->blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nboxes, (int64_t)num_sms() * per_sm));
  // in-order schedule, one box per CTA, when the boxes outnumber the persistent grid (config 3b:
  // 1223.5 us vs 1293.7, profiles/r02_sweep_front.log)
  t.chunk = unit_chunk(nboxes > (int64_t)P->blocks ? 1 : 0);
  P->blocks = chunk_grid(nboxes, t.chunk, P->blocks);
  if (t.chunk) t.stages = (int)std::min<int64_t>(t.stages, std::max<uint32_t>(2, t.chunk));
  P->tm_swizzle = 0;
  P->tm_cache.reset();
  P->align = 16;
  char b[256];
  snprintf(b, sizeof b,
           "{\"kernel\":\"tma\",\"mode\":\"bulk-load/movmatrix/bulk-store\",\"atom\":\"movmatrix.m8n8.trans.b16\","
           "\"box_bytes\":%u,\"boxes\":%lld,\"stages\":%d,\"blocks\":%u,\"replicas\":%d}",
           t.box_bytes, (long long)nboxes, t.stages, P->blocks, t.nrep);
  P->desc = b;
  return true;
}

}  // namespace axe
