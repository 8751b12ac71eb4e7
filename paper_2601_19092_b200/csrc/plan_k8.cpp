// plan_k8.cpp -- planner of K8, the dual-decoding copy (kernels.cu k8_dual) for layout pairs whose digit
// systems do not nest (SURVEY §7 hard part 3; Alg. 1's gcd = 1 failure, P:960-993 / P:978).
//
// joint_refine_partial gives the innermost joint digits (down to the gcd of the first non-nesting
// pair: an aligned run of that many consecutive x lies inside one digit on both sides) and the two
// remaining digit lists, which decode the outer index o = x / G independently.  The inner block is
// vectorised exactly as K1 does (the shared contiguous run, <= 16 bytes, dividing every stride, base
// and replica offset); the outer digits cost two fast-division chains per vector.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "plan.hpp"

namespace axe {

int k8_chunk(int vb);

static int64_t env_i8(const char *name, int64_t dflt) {
  const char *e = getenv(name);
  return (e && *e) ? atoll(e) : dflt;
}

static bool env_chunked() {  // AXE_K8_CHUNKED=0: per-vector decoding only (tests compare both forms)
  const char *e = getenv("AXE_K8_CHUNKED");
  return !(e && *e == '0');
}

bool build_k8(const Linear &ls, const Linear &ld, const Storage &sst, const Storage &dstst, int es, int max_align,
              CopyPlan *P, std::string *why) {
  auto fail = [&](const std::string &m) {
    *why = "dual: " + m;
    return false;
  };
  std::vector<Joint> Jin;
  std::vector<LinIter> A, B;
  if (!joint_refine_partial(ls.D, ld.D, &Jin, &A, &B)) return fail("no digit lists");
  if (Jin.empty()) Jin.push_back(Joint{1, 1, 1});  // gcd 1: element by element, both decodings per element
  for (auto &j : Jin)
    if (j.sdev || j.ddev) return fail("device-axis digits");
  for (auto *L : {&A, &B})
    for (auto &x : *L)
      if (x.dev) return fail("device-axis digits");
  if ((int)A.size() > K8_MAXD || (int)B.size() > K8_MAXD) return fail("too many outer digits");
  // destination replicas (set semantics)
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
  if ((int)reps.size() > K1_MAXREP) return fail("too many destination replicas");
  // vector width V (elements): K1's rule on the inner block, and every outer stride must be a multiple
  int64_t V = 1;
  const Joint in = Jin.back();
  if (in.ss == 1 && in.ds == 1) {
    std::vector<int64_t> all{ls.base, ld.base};
    for (size_t k = 0; k + 1 < Jin.size(); k++) {
      all.push_back(Jin[k].ss);
      all.push_back(Jin[k].ds);
    }
    for (auto &x : A) all.push_back(x.s);
    for (auto &x : B) all.push_back(x.s);
    for (int64_t r : reps) all.push_back(r);
    int64_t cap = std::min<int64_t>(16, max_align) / es;
    if (sst.swz_b > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(1) << sst.swz_m) / es));
    if (dstst.swz_b > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(1) << dstst.swz_m) / es));
    for (int64_t v = 2; v <= cap; v *= 2) {
      bool ok = in.e % v == 0;
      for (int64_t x : all) ok = ok && x % v == 0;
      if (ok) V = v;
    }
  }
  std::vector<Joint> I;  // inner digits without the vector, outermost first
  for (size_t k = 0; k + 1 < Jin.size(); k++)
    if (Jin[k].e > 1) I.push_back(Jin[k]);
  if (in.e / V > 1) I.push_back(Joint{in.e / V, in.ss * V, in.ds * V});
  if ((int)I.size() > K1_MAXD) return fail("too many inner digits");
  int64_t vin = 1, nout = 1;
  for (auto &j : I) vin *= j.e;
  for (auto &x : A) nout *= x.e;
  int64_t nb = 1;
  for (auto &x : B) nb *= x.e;
  if (nb != nout) return fail("outer decodings of different sizes");
  if (vin * nout >= (int64_t(1) << 31)) return fail("2^31 or more vectors");
  K8Params &k = P->k8;
  memset(&k, 0, sizeof(k));
  k.total = (uint32_t)(vin * nout);
  k.vin = make_fastdiv((uint32_t)vin);
  k.nin = (int)I.size();
  for (size_t i = 0; i < I.size(); i++) {
    k.ifd[i] = make_fastdiv((uint32_t)I[i].e);
    k.iss[i] = I[i].ss * es;
    k.ids[i] = I[i].ds * es;
  }
  k.na = (int)A.size();
  for (size_t i = 0; i < A.size(); i++) {
    k.afd[i] = make_fastdiv((uint32_t)A[i].e);
    k.as[i] = A[i].s * es;
  }
  k.nb = (int)B.size();
  for (size_t i = 0; i < B.size(); i++) {
    k.bfd[i] = make_fastdiv((uint32_t)B[i].e);
    k.bs[i] = B[i].s * es;
  }
  k.sbase = ls.base * es;
  k.dbase = ld.base * es;
  k.nrep = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
  k.ssw = make_swz(sst);
  k.dsw = make_swz(dstst);
  P->vb = (int)(V * es);
  // bulk form: the inner block is ONE run contiguous on both sides, unswizzled, 16-byte aligned throughout
  // -- it moves by cp.async.bulk in boxes of at most 16 KiB (AUTO: runs of >= 1 KiB)
  {
    const int64_t run = in.e * es;
    bool ok = Jin.size() == 1 && in.ss == 1 && in.ds == 1 && !sst.swz_b && !dstst.swz_b && max_align >= 16 &&
              run % 16 == 0 && run >= env_i8("AXE_K8_BULK_MIN_RUN", 1024) && env_i8("AXE_K8_BULK", 1) &&
              (ls.base * es) % 16 == 0 && (ld.base * es) % 16 == 0;
    for (auto &x : A) ok = ok && (x.s * es) % 16 == 0;
    for (auto &x : B) ok = ok && (x.s * es) % 16 == 0;
    for (int64_t r : reps) ok = ok && (r * es) % 16 == 0;
    int64_t box = 0;
    if (ok)
      for (int64_t d = std::min<int64_t>(run, 16384); d >= 16; d -= 16)
        if (run % d == 0) {
          box = d;
          break;
        }
    if (ok && box && (run / box) * nout < (int64_t(1) << 31)) {
      k.bulk = 1;
      P->align = std::max(P->align, 16);  // cp.async.bulk: 16-byte aligned global addresses
      k.box = (uint32_t)box;
      k.per_run = make_fastdiv((uint32_t)(run / box));
      k.nboxes = (uint32_t)((run / box) * nout);
    }
  }
  // odometer form: gcd 1 (an empty inner block, one element per vector) -- per-lane digit carries
  if (vin == 1 && V == 1 && Jin.size() == 1 && in.e == 1 && !A.empty() && !B.empty() && env_i8("AXE_K8_ODO", 1) &&
      k.total < (uint32_t)0xFFFFFFFF - 32 * K8_ODO_J) {
    k.odo = 1;
    k.nchunk = (uint32_t)((k.total + 32 * K8_ODO_J - 1) / (32 * K8_ODO_J));
  }
  // chunked form: the inner block is one run (a single digit) of at least one vector per thread
  const int64_t CH = k8_chunk(P->vb);
  if (I.size() == 1 && vin >= CH / (P->vb >= 8 ? 4 : 8) && env_chunked()) {  // >= one vector per thread
    const int64_t nch = (vin + CH - 1) / CH;
    if (nch * nout < (int64_t(1) << 31)) {
      k.chunked = 1;
      k.nchunks = make_fastdiv((uint32_t)nch);
      k.nitems = (uint32_t)(nch * nout);
    }
  }
  // the in-order schedule once the units outnumber the persistent grid (profiles/r02_sweep_front.log,
  // nonnested 1.5 GiB): bulk form 2 boxes per CTA (236.9 us vs 262.8), chunked item form 1 item (234.0
  // vs ~280), odometer 2 units of 8 warp chunks (947.5 vs ~985)
  const int64_t wave = (int64_t)num_sms() * 8;
  k.chunk = k.bulk      ? unit_chunk(k.nboxes > (uint32_t)(4 * num_sms()) ? 2 : 0)
            : k.chunked ? unit_chunk((int64_t)k.nitems > wave ? 1 : 0)
            : k.odo     ? unit_chunk((int64_t)k.nchunk / 8 > wave ? 2 : 0)
                        : unit_chunk(0);
  P->align = std::max(P->align, P->vb);
  P->covers_all = (int64_t)reps.size() * vin * nout * V == dstst.cells;
  auto lin_json = [](const std::vector<LinIter> &L) {
    std::string s = "[";
    for (size_t i = 0; i < L.size(); i++)
      s += (i ? "," : "") + std::string("[") + std::to_string(L[i].e) + "," + std::to_string(L[i].s) + "]";
    return s + "]";
  };
  P->desc = "{\"kernel\":\"dual\",\"odometer\":" + std::to_string(k.odo) + ",\"bulk\":" + std::to_string(k.bulk) + ",\"box_bytes\":" +
            std::to_string(k.box) + ",\"chunked\":" + std::to_string(k.chunked) + ",\"chunk\":" + std::to_string(k.chunk) + ",\"vec_bytes\":" + std::to_string(P->vb) + ",\"vectors\":" +
            std::to_string(k.total) + ",\"inner_block_vectors\":" + std::to_string(vin) +
            ",\"outer_blocks\":" + std::to_string(nout) + ",\"replicas\":" + std::to_string(reps.size()) +
            ",\"inner\":" + joint_json(Jin) + ",\"outer_src\":" + lin_json(A) + ",\"outer_dst\":" + lin_json(B) + "}";
  return true;
}

}  // namespace axe
