// algebra.cpp -- the layout operators of the paper (§3.3, Apps. B-F), on the
// host: Group-By-Shape (Alg. 1), Tile (Alg. 2),
// TileOf_AndRecoverC (Alg. 3), SliceBlockAfterCanon_Sufficient
// (Alg. 4) and the direct sum on the tiling domain (App. F,
// P:1550-1747).  These are the building blocks of the paper's TMA lowering
// (slice -> tile_of against the swizzle atom -> tensor map).
#include <cstring>
#include <numeric>

#include "handles.hpp"

using namespace axe;

namespace axe {

// Alg. 1: refine D left to right into blocks whose extent products are S_i.
// On success `out` is the refined D and `bounds` has rank+1 block boundaries.
static axe_status group_by_shape(const std::vector<Iter> &D, const std::vector<int64_t> &S, std::vector<Iter> *out,
                                 std::vector<int> *bounds) {
  int64_t pe = 1, ps = 1;
  for (auto &it : D)
    if (__builtin_mul_overflow(pe, it.e, &pe)) AXE_FAIL(AXE_ERR_OVERFLOW, "extent product overflow");
  for (int64_t s : S) {
    if (s < 1) AXE_FAIL(AXE_ERR_INVALID_ARG, "shape dimension %lld < 1", (long long)s);
    if (__builtin_mul_overflow(ps, s, &ps)) AXE_FAIL(AXE_ERR_OVERFLOW, "shape product overflow");
  }
  if (pe != ps) AXE_FAIL(AXE_ERR_SIZE_MISMATCH, "shape not admitted: prod S = %lld != E_D = %lld", (long long)ps, (long long)pe);
  std::vector<Iter> src = D, res;
  std::vector<int> b{0};
  size_t j = 0;
  for (size_t i = 0; i < S.size(); i++) {
    const int64_t T = S[i];
    int64_t cur = 1;
    while (cur < T) {
      if (j >= src.size()) AXE_FAIL(AXE_ERR_UNSUPPORTED, "grouping ran out of iters (block %zu)", i);
      Iter it = src[j];
      const int64_t rem = T / cur;
      int64_t g = std::gcd(it.e, rem);
      if (g == 1) AXE_FAIL(AXE_ERR_UNSUPPORTED, "grouping fails: gcd(%lld, %lld) = 1 in block %zu (Alg. 1, P:978)",
                           (long long)it.e, (long long)rem, i);
      const int64_t tail = it.e / g;
      res.push_back(Iter{g, tail * it.s, it.a});  // split (Lemma split): head keeps e_tail * s
      cur *= g;
      if (tail > 1)
        src[j] = Iter{tail, it.s, it.a};
      else
        j++;
    }
    b.push_back((int)res.size());
  }
  // trailing unit iters (extent 1) are semantically empty
  for (; j < src.size(); j++)
    if (src[j].e != 1) AXE_FAIL(AXE_ERR_UNSUPPORTED, "grouping left iters unconsumed");
  *out = std::move(res);
  *bounds = std::move(b);
  return AXE_OK;
}

// closed-form axis-wise span (Lemma span-closed) of D and R
static std::vector<std::pair<int, int64_t>> span_of(const std::vector<Iter> &D, const std::vector<Iter> &R) {
  std::vector<std::pair<int, int64_t>> w;
  auto add = [&](int a, int64_t v) {
    for (auto &p : w)
      if (p.first == a) {
        p.second += v;
        return;
      }
    w.push_back({a, 1 + v});
  };
  for (auto *lst : {&D, &R})
    for (auto &it : *lst) add(it.a, (it.s < 0 ? -it.s : it.s) * (it.e - 1));
  return w;
}
static int64_t span_at(const std::vector<std::pair<int, int64_t>> &w, int a) {
  for (auto &p : w)
    if (p.first == a) return p.second;
  return 1;  // an axis B never names has span 1
}

}  // namespace axe

static std::vector<int64_t> shape_vec(const int64_t *S, int rank) { return std::vector<int64_t>(S, S + rank); }

extern "C" {

axe_status axe_layout_group(const axe_layout *L, const int64_t *shape, int rank, axe_layout **out, int *bounds) {
  if (!L || !shape || rank < 1 || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad argument");
  *out = nullptr;
  std::vector<Iter> D;
  std::vector<int> b;
  AXE_TRY(group_by_shape(L->L.D, shape_vec(shape, rank), &D, &b));
  if (D.empty()) D.push_back(Iter{1, 1, axis_m()});
  auto *h = new axe_layout;
  axe_status st = make_layout(D, L->L.R, L->L.O, &h->L);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  if (bounds)
    for (int i = 0; i <= rank; i++) bounds[i] = b[i];
  *out = h;
  return AXE_OK;
}

axe_status axe_layout_span(const axe_layout *L, const char *axis, int64_t *span) {
  if (!L || !span) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad argument");
  int a = intern_axis(axis ? axis : "m");
  if (a < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "axis name is not an identifier");
  *span = span_at(span_of(L->L.D, L->L.R), a);
  return AXE_OK;
}

// Alg. 2: T = A (x) B over the interleaved shape (S_A[0], S_B[0], ...).
axe_status axe_layout_tile(const axe_layout *A, const int64_t *SA, const axe_layout *B, const int64_t *SB, int rank,
                           axe_layout **out) {
  if (!A || !B || !SA || !SB || rank < 1 || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad argument");
  *out = nullptr;
  std::vector<Iter> DA, DB;
  std::vector<int> bA, bB;
  AXE_TRY(group_by_shape(A->L.D, shape_vec(SA, rank), &DA, &bA));
  AXE_TRY(group_by_shape(B->L.D, shape_vec(SB, rank), &DB, &bB));
  auto W = span_of(DB, B->L.R);
  std::vector<Iter> DT, RT;
  for (int i = 0; i < rank; i++) {
    for (int k = bA[i]; k < bA[i + 1]; k++) DT.push_back(Iter{DA[k].e, span_at(W, DA[k].a) * DA[k].s, DA[k].a});
    for (int k = bB[i]; k < bB[i + 1]; k++) DT.push_back(DB[k]);
  }
  if (DT.empty()) DT.push_back(Iter{1, 1, axis_m()});
  for (auto &it : A->L.R) RT.push_back(Iter{it.e, span_at(W, it.a) * it.s, it.a});
  for (auto &it : B->L.R) RT.push_back(it);
  std::vector<std::pair<int, int64_t>> OT;
  for (auto &p : A->L.O) OT.push_back({p.first, p.second * span_at(W, p.first)});
  for (auto &p : B->L.O) OT.push_back(p);
  auto *h = new axe_layout;
  axe_status st = make_layout(DT, RT, OT, &h->L);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *out = h;
  return AXE_OK;
}

// App. F: A + B on the tiling domain -- per rank, A's block then B's block, unscaled.
axe_status axe_layout_direct_sum(const axe_layout *A, const int64_t *SA, const axe_layout *B, const int64_t *SB,
                                 int rank, axe_layout **out) {
  if (!A || !B || !SA || !SB || rank < 1 || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad argument");
  *out = nullptr;
  std::vector<Iter> DA, DB;
  std::vector<int> bA, bB;
  AXE_TRY(group_by_shape(A->L.D, shape_vec(SA, rank), &DA, &bA));
  AXE_TRY(group_by_shape(B->L.D, shape_vec(SB, rank), &DB, &bB));
  std::vector<Iter> D, R;
  for (int i = 0; i < rank; i++) {
    for (int k = bA[i]; k < bA[i + 1]; k++) D.push_back(DA[k]);
    for (int k = bB[i]; k < bB[i + 1]; k++) D.push_back(DB[k]);
  }
  if (D.empty()) D.push_back(Iter{1, 1, axis_m()});
  R = A->L.R;
  R.insert(R.end(), B->L.R.begin(), B->L.R.end());
  std::vector<std::pair<int, int64_t>> O = A->L.O;
  O.insert(O.end(), B->L.O.begin(), B->L.O.end());
  auto *h = new axe_layout;
  axe_status st = make_layout(D, R, O, &h->L);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *out = h;
  return AXE_OK;
}

// Alg. 3 with the offset and replication checks of P:1332-1380.
axe_status axe_layout_tile_of(const axe_layout *A, const int64_t *SA, const axe_layout *B, const int64_t *SB, int rank,
                              axe_layout **C_out, int64_t *SC) {
  if (!A || !B || !SA || !SB || rank < 1 || !C_out || !SC) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad argument");
  *C_out = nullptr;
  for (int j = 0; j < rank; j++) {
    if (SB[j] < 1 || SA[j] % SB[j]) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tile_of: S_B[%d] does not divide S_A[%d]", j, j);
    SC[j] = SA[j] / SB[j];
  }
  // canonical D parts (the algorithm assumes D0/D1)
  std::vector<Iter> cA = normalize_shard(A->L.D), cB = normalize_shard(B->L.D);
  std::vector<Iter> DA, DB;
  std::vector<int> bA, bB;
  AXE_TRY(group_by_shape(cA, shape_vec(SA, rank), &DA, &bA));
  AXE_TRY(group_by_shape(cB, shape_vec(SB, rank), &DB, &bB));
  auto W = span_of(DB, B->L.R);
  std::vector<Iter> DC;
  for (int j = 0; j < rank; j++) {
    int p = bA[j], q = bB[j];
    int64_t prod = 1;
    while (p < bA[j + 1]) {
      const Iter &x = DA[p];
      if (q < bB[j + 1] && x.e == DB[q].e && x.s == DB[q].s && x.a == DB[q].a) {
        p++;
        q++;
        continue;
      }
      int64_t w = span_at(W, x.a);
      if (x.s % w) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tile_of: residual stride %lld not divisible by span %lld", (long long)x.s, (long long)w);
      DC.push_back(Iter{x.e, x.s / w, x.a});
      prod *= x.e;
      p++;
    }
    if (q != bB[j + 1]) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tile_of: block %d of B is not a subsequence of A's", j);
    if (prod != SC[j]) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tile_of: block %d extent product mismatch", j);
  }
  if (DC.empty()) DC.push_back(Iter{1, 1, axis_m()});
  // offsets: O_A = O_C (.) W + O_B, axiswise
  std::vector<std::pair<int, int64_t>> OC;
  std::vector<int> axes;
  for (auto &p : A->L.O) axes.push_back(p.first);
  for (auto &p : B->L.O) axes.push_back(p.first);
  for (int a : axes) {
    bool seen = false;
    for (auto &p : OC)
      if (p.first == a) seen = true;
    if (seen) continue;
    int64_t d = A->L.offset(a) - B->L.offset(a), w = span_at(W, a);
    if (d % w) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tile_of: offset on %s not divisible by the span", axis_name(a));
    if (d) OC.push_back({a, d / w});
  }
  // replication: canonical R_A must be canonical(W-scaled R_C + R_B); R_C = A's replica iters not in B, descaled
  std::vector<Iter> RB = B->L.R, RC;
  std::vector<Iter> RA = A->L.R;
  for (auto &x : RA) {
    bool matched = false;
    for (size_t i = 0; i < RB.size(); i++)
      if (RB[i].e == x.e && RB[i].s == x.s && RB[i].a == x.a) {
        RB.erase(RB.begin() + i);
        matched = true;
        break;
      }
    if (matched) continue;
    int64_t w = span_at(W, x.a);
    if (x.s % w) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tile_of: replica stride not divisible by the span");
    RC.push_back(Iter{x.e, x.s / w, x.a});
  }
  if (!RB.empty()) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tile_of: B's replication is not part of A's");
  auto *h = new axe_layout;
  axe_status st = make_layout(DC, RC, OC, &h->L);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *C_out = h;
  return AXE_OK;
}

// Alg. 4 per grouped block, blocks composed by concatenation and
// offset summation.  Readings: a fully peeled block returns its peeled iters;
// otherwise the pivot forms run with the remaining extent (which reproduces the
// paper's printed (1,8,2,8):(192,8,64,1) + 64); the one-wrap form
// needs S_{k-1} and S_k on one axis (Delta is one iter).
axe_status axe_layout_slice(const axe_layout *L, const int64_t *S, int rank, const int64_t *begin,
                            const int64_t *extent, axe_layout **out) {
  if (!L || !S || !begin || !extent || rank < 1 || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad argument");
  *out = nullptr;
  for (int i = 0; i < rank; i++)
    if (begin[i] < 0 || extent[i] < 1 || begin[i] + extent[i] > S[i])
      AXE_FAIL(AXE_ERR_DOMAIN, "region dimension %d outside the shape", i);
  std::vector<Iter> D;
  std::vector<int> bd;
  AXE_TRY(group_by_shape(L->L.D, shape_vec(S, rank), &D, &bd));
  std::vector<Iter> res;
  std::vector<std::pair<int, int64_t>> O = L->L.O;
  for (int i = 0; i < rank; i++) {
    std::vector<Iter> blk = normalize_shard(std::vector<Iter>(D.begin() + bd[i], D.begin() + bd[i + 1]));
    if (blk.size() == 1 && blk[0].e == 1) blk.clear();
    const int m = (int)blk.size();
    std::vector<int64_t> d0(m, 0);
    {
      int64_t rem = begin[i];
      for (int k = m - 1; k >= 0; k--) {
        d0[k] = rem % blk[k].e;
        rem /= blk[k].e;
      }
    }
    for (int k = 0; k < m; k++) O.push_back({blk[k].a, d0[k] * blk[k].s});  // block origin contribution
    std::vector<Iter> peeled;
    int64_t rem = extent[i];
    int j = m - 1;
    for (; j >= 0; j--) {
      if (d0[j] == 0 && rem % blk[j].e == 0) {
        peeled.insert(peeled.begin(), blk[j]);
        rem /= blk[j].e;
      } else {
        break;
      }
    }
    std::vector<Iter> out_blk;
    if (j >= 0) {
      const int k = j;
      if (d0[k] + rem <= blk[k].e) {  // no-wrap (Lemma)
        out_blk.push_back(Iter{rem, blk[k].s, blk[k].a});
      } else if (rem % 2 == 0 && d0[k] + rem / 2 == blk[k].e && (k == 0 || d0[k - 1] + 1 < blk[k - 1].e)) {
        // reading R22: the paper's capacity test d_{k-1} + 1 <= E_{k-1} lets digit k-1
        // reach E_{k-1}, which itself carries; the carry-free condition is d_{k-1} + 1 < E_{k-1}
        const int64_t c = rem / 2;  // symmetric one-wrap (Lemma)
        if (k > 0 && blk[k - 1].a != blk[k].a)
          AXE_FAIL(AXE_ERR_UNSUPPORTED, "slice: one-wrap step spans two axes (not a single iter)");
        int64_t delta = (k > 0 ? blk[k - 1].s : 0) - (blk[k].e - c) * blk[k].s;
        if (delta == 0) AXE_FAIL(AXE_ERR_UNSUPPORTED, "slice: zero one-wrap step");
        out_blk.push_back(Iter{2, delta, blk[k].a});
        out_blk.push_back(Iter{c, blk[k].s, blk[k].a});
      } else {
        AXE_FAIL(AXE_ERR_UNSUPPORTED, "slice: block %d admits neither sufficient form (Alg. 4)", i);
      }
    } else if (rem != 1) {
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "slice: block %d over-peeled", i);
    }
    out_blk.insert(out_blk.end(), peeled.begin(), peeled.end());
    res.insert(res.end(), out_blk.begin(), out_blk.end());
  }
  if (res.empty()) res.push_back(Iter{1, 1, axis_m()});
  auto *h = new axe_layout;
  axe_status st = make_layout(res, L->L.R, O, &h->L);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *out = h;
  return AXE_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// The paper's TMA lowering (§3.4 "TMA asynchronous copy"), on the
// algebra above: (1) slice the global view L_G[R_G : E_G] (Alg. 4); (2) the
// swizzle atom E_{d,a} = (1, .., 1, 8, a / sizeof(d)) (reading R14: rank equal to
// E_S's) and the tiler T with (L_S)||E_S = T||E_o (x) (L_{d,a})||E_{d,a}: L_S is
// grouped by the interleaved shape (E_o[0], E_{d,a}[0], ...) (Alg. 1, splitting
// iters) and every inner block must equal the atom's block (Alg. 3's EqualIter);
// the outer blocks, divided by the atom's span, are T (reading R26); (3) the
// atom's global counterpart is a suffix product of the iters of each group of
// (L_G)||E_G -- at most one iter split (Lemma split) -- and the iters of the
// grouped L_G become the CuTensorMap dimensions (innermost first), the box
// covering exactly the atom's iters.
// ---------------------------------------------------------------------------
extern "C" {

axe_status axe_tma_lower(const axe_layout *LG, const int64_t *EG, const int64_t *begin, const int64_t *extent,
                         const axe_layout *LS, const int64_t *ES, int rank, int elem_size, int swizzle_bytes,
                         axe_tma_desc *out, axe_layout **tiler) {
  if (!LG || !EG || !LS || !ES || !out || rank < 2 || rank > 5) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad argument (rank 2..5)");
  if (tiler) *tiler = nullptr;
  memset(out, 0, sizeof(*out));
  const int es = elem_size;
  if (es != 1 && es != 2 && es != 4 && es != 8 && es != 16) AXE_FAIL(AXE_ERR_ALIGNMENT, "elem_size %d", es);
  if (swizzle_bytes != 32 && swizzle_bytes != 64 && swizzle_bytes != 128)
    AXE_FAIL(AXE_ERR_INVALID_ARG, "swizzle mode %d B is not 32 / 64 / 128 (P:527)", swizzle_bytes);
  const int m = axis_m();
  for (const axe_layout *L : {LG, LS}) {
    if (!L->L.R.empty()) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: replicated layouts are not a TMA box");
    for (auto &it : L->L.D)
      if (it.a != m) AXE_FAIL(AXE_ERR_UNSUPPORTED_AXIS, "tma: every iter must be on the memory axis m");
    for (auto &o : L->L.O)
      if (o.first != m) AXE_FAIL(AXE_ERR_UNSUPPORTED_AXIS, "tma: offsets must be on the memory axis m");
  }
  if (LS->L.offset(m)) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: the shared-memory tensor starts at its base");
  // (1) slice view of the global tensor
  axe_layout *Gs = nullptr;
  std::vector<int64_t> E(EG, EG + rank);
  if (begin) {
    if (!extent) AXE_FAIL(AXE_ERR_INVALID_ARG, "begin without extent");
    AXE_TRY(axe_layout_slice(LG, EG, rank, begin, extent, &Gs));
    E.assign(extent, extent + rank);
  }
  std::unique_ptr<axe_layout, void (*)(axe_layout *)> Gown(Gs, [](axe_layout *p) { delete p; });
  const Layout &G = Gs ? Gs->L : LG->L;
  for (int j = 0; j < rank; j++)
    if (E[j] != ES[j]) AXE_FAIL(AXE_ERR_SIZE_MISMATCH, "region shape differs from E_S in dimension %d", j);
  // (2) the swizzle atom and the tiler T
  const int64_t inner = swizzle_bytes / es;
  if (inner < 1) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: element wider than the swizzle span");
  std::vector<int64_t> Ea(rank, 1), Eo(rank), I;
  Ea[rank - 1] = inner;
  Ea[rank - 2] = 8;
  for (int j = 0; j < rank; j++) {
    if (ES[j] % Ea[j]) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: atom extent %lld does not divide E_S[%d]", (long long)Ea[j], j);
    Eo[j] = ES[j] / Ea[j];
    I.push_back(Eo[j]);
    I.push_back(Ea[j]);
  }
  std::vector<Iter> DS, DA;
  std::vector<int> bS, bA;
  AXE_TRY(group_by_shape(normalize_shard(LS->L.D), I, &DS, &bS));
  const std::vector<Iter> atom{Iter{8, inner, m}, Iter{inner, 1, m}};
  AXE_TRY(group_by_shape(normalize_shard(atom), Ea, &DA, &bA));
  const int64_t W = 8 * inner;  // span of the atom on m
  std::vector<Iter> DT;
  for (int j = 0; j < rank; j++) {
    std::vector<Iter> in(DS.begin() + bS[2 * j + 1], DS.begin() + bS[2 * j + 2]);
    std::vector<Iter> at(DA.begin() + bA[j], DA.begin() + bA[j + 1]);
    in = normalize_shard(in);
    at = normalize_shard(at);
    if (in.size() == 1 && in[0].e == 1) in.clear();
    if (at.size() == 1 && at[0].e == 1) at.clear();
    bool eq = in.size() == at.size();
    for (size_t k = 0; eq && k < in.size(); k++) eq = in[k].e == at[k].e && in[k].s == at[k].s;
    if (!eq) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: L_S is not a tiling of the %d-byte swizzle atom (dimension %d)", swizzle_bytes, j);
    for (int k = bS[2 * j]; k < bS[2 * j + 1]; k++) {
      if (DS[k].s % W) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: atom-grid stride %lld is not a multiple of the atom span", (long long)DS[k].s);
      DT.push_back(Iter{DS[k].e, DS[k].s / W, m});
    }
  }
  // (3) the tensor map from the grouped global layout
  std::vector<Iter> DG;
  std::vector<int> bG;
  AXE_TRY(group_by_shape(G.D, E, &DG, &bG));
  struct Dim {
    int64_t e, s;
    bool box;
    int j;  // logical dimension
  };
  std::vector<Dim> dims;  // innermost first
  for (int j = rank - 1; j >= 0; j--) {
    std::vector<Iter> blk(DG.begin() + bG[j], DG.begin() + bG[j + 1]);
    int64_t p = 1;
    int k = (int)blk.size() - 1;
    for (; k >= 0 && p < Ea[j]; k--) {
      const int64_t need = Ea[j] / p;
      if (Ea[j] % p) break;
      if (blk[k].e <= need && need % blk[k].e == 0) {
        dims.push_back(Dim{blk[k].e, blk[k].s, true, j});
        p *= blk[k].e;
      } else if (blk[k].e % need == 0) {  // split: inner `need` in the box, the rest outside (Lemma split)
        dims.push_back(Dim{need, blk[k].s, true, j});
        blk[k] = Iter{blk[k].e / need, blk[k].s * need, blk[k].a};
        p *= need;
        break;  // (no decrement: the outer part blk[k] is pushed next as a non-box iter)
      } else {
        break;
      }
    }
    if (p != Ea[j])
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: atom extent %lld is not a suffix product of group %d of L_G", (long long)Ea[j], j);
    for (; k >= 0; k--)
      if (blk[k].e > 1) dims.push_back(Dim{blk[k].e, blk[k].s, false, j});
  }
  if (dims.empty() || !dims[0].box || dims[0].s != 1)
    AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: the innermost box dimension must be contiguous (stride 1)");
  // fuse neighbours that continue one another with the same box status (fewer tensor-map dims)
  std::vector<Dim> fz;
  for (auto &d : dims) {
    if (d.e == 1 && !d.box) continue;
    if (!fz.empty() && fz.back().box == d.box && fz.back().j == d.j && d.s == fz.back().s * fz.back().e &&
        (!d.box || fz.size() == 1))
      fz.back().e *= d.e;
    else
      fz.push_back(d);
  }
  if (fz.size() > 5) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: %zu tensor-map dimensions (max 5)", fz.size());
  out->rank = (int)fz.size();
  for (size_t i = 0; i < fz.size(); i++) {
    out->dims[i] = (uint64_t)fz[i].e;
    out->strides[i] = (uint64_t)(fz[i].s * es);
    out->box[i] = (uint32_t)(fz[i].box ? fz[i].e : 1);
    out->logical_dim[i] = fz[i].j;
    if (fz[i].s < 0) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: negative global stride");
    if (i > 0 && (fz[i].s * es) % 16) AXE_FAIL(AXE_ERR_ALIGNMENT, "tma: global stride %lld B is not a multiple of 16", (long long)(fz[i].s * es));
    if (out->box[i] > 256) AXE_FAIL(AXE_ERR_UNSUPPORTED, "tma: box dimension > 256");
  }
  out->swizzle_bytes = swizzle_bytes;
  out->base_bytes = G.offset(m) * es;
  int64_t atoms = 1;
  for (auto &t : DT) atoms *= t.e;
  out->atoms = atoms;
  // atoms that stack along the row dimension in both memories can share one box: T's innermost
  // row-dimension iter with unit (atom) stride, and the global rows continuing past the atom
  out->fused_rows = 8;
  {
    std::vector<Iter> trow(DS.begin() + bS[2 * (rank - 2)], DS.begin() + bS[2 * (rank - 2) + 1]);
    trow = normalize_shard(trow);
    int64_t f = 1;
    if (!trow.empty() && trow.back().s == W) f = trow.back().e;
    // the global row iter just outside the box (stride = 8 rows) must hold at least f atoms
    int64_t rows_out = 0;
    for (size_t i = 0; i < dims.size(); i++)
      if (!dims[i].box && i > 0 && dims[i - 1].box && dims[i].s == dims[i - 1].s * dims[i - 1].e) {
        rows_out = dims[i].e;
        break;
      }
    while (f > 1 && (8 * f > 256 || rows_out % f)) f /= 2;
    if (rows_out > 0) out->fused_rows = (uint32_t)(8 * f);
  }
  if (tiler) {
    if (DT.empty()) DT.push_back(Iter{1, 1, m});
    auto *h = new axe_layout;
    axe_status st = make_layout(DT, {}, {}, &h->L);
    if (st != AXE_OK) {
      delete h;
      return st;
    }
    *tiler = h;
  }
  return AXE_OK;
}

}  // extern "C"
