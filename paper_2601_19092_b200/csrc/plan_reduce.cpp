// plan_reduce.cpp -- planning of the K4 reduction and its C-ABI.
//
// dst(y) = sum_{k<K} src(k * E_D(dst) + y), K = E_D(src) / E_D(dst) (reading R24;
// P:399-403 the DTensor reduce-scatter "sums over 0", P:628 the sum operator).
// The plan composes both layouts with their storages (as a copy does), prepends
// a stride-0 digit of extent K to the destination -- the summed dimension has
// no destination coordinate -- and refines the two digit systems jointly.
// Joint digits with destination stride 0 are the reduction digits; the others
// index output vectors.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <unordered_map>

#include "handles.hpp"

namespace axe {

static int64_t env_int_r(const char *name, int64_t dflt) {
  const char *e = getenv(name);
  return (e && *e) ? atoll(e) : dflt;
}

int dtype_size(int dt) {
  switch (dt) {
    case DT_F32: case DT_I32: return 4;
    case DT_F64: case DT_I64: return 8;
    case DT_F16: case DT_BF16: return 2;
  }
  return 0;
}

static const char *dtype_name(int dt) {
  switch (dt) {
    case DT_F32: return "f32";
    case DT_F64: return "f64";
    case DT_F16: return "f16";
    case DT_BF16: return "bf16";
    case DT_I32: return "i32";
    case DT_I64: return "i64";
  }
  return "?";
}

axe_status plan_reduce(const Layout &S, const Storage &sst, const Layout &D, const Storage &dstst, int dtype,
                       int max_align, ReducePlan *out) {
  const int es = dtype_size(dtype);
  if (!es) AXE_FAIL(AXE_ERR_INVALID_ARG, "unknown dtype %d", dtype);
  if (S.ED % D.ED)
    AXE_FAIL(AXE_ERR_SIZE_MISMATCH, "E_D(src) = %lld is not a multiple of E_D(dst) = %lld", (long long)S.ED,
             (long long)D.ED);
  AXE_TRY(check_side(S, sst, -1, "source"));
  AXE_TRY(check_side(D, dstst, -1, "destination"));
  for (const Storage *st : {&sst, &dstst})
    if (st->swz_b > 0 && (st->cells * es) % (int64_t(1) << (st->swz_b + st->swz_m + st->swz_s)))
      AXE_FAIL(AXE_ERR_BOUNDS, "swizzled storage is not a whole number of swizzle blocks");
  AXE_TRY(check_injective(D, dstst, -1));

  ReducePlan P;
  P.dtype = dtype;
  P.es = es;
  P.K = S.ED / D.ED;
  P.src_bytes = sst.cells * es;
  P.dst_bytes = dstst.cells * es;
  P.align = es;

  Linear ls, ld;
  std::vector<Joint> J;
  bool joint = compose_linear(S, sst, -1, &ls) && compose_linear(D, dstst, -1, &ld);
  if (joint) {
    std::vector<LinIter> ldx = ld.D;
    if (P.K > 1) ldx.insert(ldx.begin(), LinIter{P.K, 0, 0});  // the summed dimension: no destination stride
    joint = joint_refine(ls.D, ldx, &J);
  }
  std::vector<int64_t> reps{0};
  if (joint) {
    for (auto &r : ld.R) {
      std::vector<int64_t> nx;
      for (int64_t b : reps)
        for (int64_t d = 0; d < r.e; d++) nx.push_back(b + d * r.s);
      reps.swap(nx);
      if (reps.size() > 4096) break;
    }
    std::sort(reps.begin(), reps.end());
    reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
    if ((int)reps.size() > K1_MAXREP) joint = false;
  }
  std::vector<Joint> Y, Kd;  // output digits / reduction digits (outermost first)
  if (joint) {
    for (auto &j : J)
      if (j.e > 1) (j.ds == 0 ? Kd : Y).push_back(j);
    if ((int)Kd.size() > K4_MAXD) joint = false;
  }
  // (A TMA-fed form -- K tensor or bulk loads per output box, the sum in shared memory, one bulk store --
  // was measured against this vector form with the in-order schedule and lost everywhere: into SW128
  // tiles 96.7 us vs 89.2, K = 8 contiguous 90.6 vs 87.0, 8 MiB outputs 13.3 vs 12.2; removed, numbers in
  // profiles/r02_k4b_sweep.log)
  if (joint) {
    // vector width: a power of two V with V * es <= 16 dividing the innermost shared stride-1 run,
    // every other stride, both bases and every replica offset (as K1)
    int64_t V = 1;
    if (!Y.empty() && Y.back().ss == 1 && Y.back().ds == 1) {
      std::vector<int64_t> all{ls.base, ld.base};
      for (size_t k = 0; k + 1 < Y.size(); k++) {
        all.push_back(Y[k].ss);
        all.push_back(Y[k].ds);
      }
      for (auto &j : Kd) all.push_back(j.ss);
      for (int64_t r : reps) all.push_back(r);
      int64_t cap = std::min<int64_t>(16, max_align) / es;
      if (sst.swz_b > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(1) << sst.swz_m) / es));
      if (dstst.swz_b > 0) cap = std::min<int64_t>(cap, std::max<int64_t>(1, (int64_t(1) << dstst.swz_m) / es));
      for (int64_t v = 2; v <= cap; v *= 2) {
        bool ok = Y.back().e % v == 0;
        for (int64_t a : all) ok = ok && a % v == 0;
        if (ok) V = v;
      }
    }
    if (V > 1) {
      Joint last = Y.back();
      Y.pop_back();
      if (last.e / V > 1) Y.push_back(Joint{last.e / V, V, V});
    }
    // destination-contiguous output digits first (every warp writes whole lines). Ordering by the
    // summand strides instead (every warp reads whole source runs) measured the same on a B200:
    // K = 8 bf16 into SW128 tiles 99.3-99.6 us either way, row-major rows 96.4-96.6
    std::stable_sort(Y.begin(), Y.end(), [](const Joint &a, const Joint &b) { return std::llabs(a.ds) > std::llabs(b.ds); });
    sort_fuse_outer(Y);
    int64_t total = 1;
    for (auto &j : Y) total *= j.e;
    // (32-bit grid-stride index in k4_reduce / k4_multimem: i + stride must not wrap)
    if ((int)Y.size() > K4_MAXD || total >= (int64_t(1) << 31)) joint = false;
    if (joint) {
      K4Params &k = P.k4;
      memset(&k, 0, sizeof(k));
      k.total = (uint32_t)total;
      k.nd = (int)Y.size();
      for (int i = 0; i < k.nd; i++) {
        k.fd[i] = make_fastdiv((uint32_t)Y[i].e);
        k.ss[i] = Y[i].ss * es;
        k.ds[i] = Y[i].ds * es;
      }
      k.sbase = ls.base * es;
      k.dbase = ld.base * es;
      k.nrep = (int)reps.size();
      for (size_t i = 0; i < reps.size(); i++) k.rep[i] = reps[i] * es;
      k.ssw = make_swz(sst);
      k.dsw = make_swz(dstst);
      if (P.K <= K4_MAXK) {
        // summand offsets in k order: the reduction digits unflatten k lexicographically
        k.nk = (int)P.K;
        for (int64_t kk = 0; kk < P.K; kk++) {
          int64_t rem = kk, off = 0;
          for (int t = (int)Kd.size() - 1; t >= 0; t--) {
            off += (rem % Kd[t].e) * Kd[t].ss;
            rem /= Kd[t].e;
          }
          k.koff[kk] = off * es;
        }
      } else {
        k.nk = 0;
        k.ktotal = (uint32_t)P.K;
        k.nkd = (int)Kd.size();
        for (int t = 0; t < k.nkd; t++) {
          k.kfd[t] = make_fastdiv((uint32_t)Kd[t].e);
          k.kss[t] = Kd[t].ss * es;
        }
      }
      P.kind = 2;
      P.vb = (int)(V * es);
      P.align = P.vb;
      {
        // streaming (st.global.cs) stores for 4- and 8-byte elements, measured on a B200 (perf_configs
        // --reduce, 2 runs each): f32 K = 8 (8192 x 2048) 88.4 us vs 94.9 plain; bf16 K = 8 96.9-97.1
        // vs 96.2 and into SW128 tiles 99.7-100.0 vs 99.7, so 2-byte elements keep plain stores
        k.stcs = (int)env_int_r("AXE_K4_STCS", es >= 4 ? 1 : 0);
        const int64_t blocks = (total + 255) / 256, cap = (int64_t)num_sms() * 8;  // 4 per SM: 5-19% slower
        P.blocks = (unsigned)std::max<int64_t>(1, std::min(blocks, cap));
        // in-order schedule (kernels.cuh unit_range) once the blocks outnumber the persistent grid:
        // max(1, 8 / K) blocks of 256 vectors per CTA, about 32 KiB of summands (profiles/
        // r02_sweep_front.log: bf16 K = 8 87.0 us vs 94.2, K = 2 125.9 vs 131.3, K = 3 163.0 vs 170.5)
        k.chunk = unit_chunk(blocks > (int64_t)P.blocks ? std::max<int64_t>(1, 8 / std::max<int64_t>(1, P.K)) : 0);
      }
      char b[320];
      snprintf(b, sizeof b,
               "{\"kernel\":\"reduce\",\"mode\":\"vector\",\"dtype\":\"%s\",\"K\":%lld,\"vec_bytes\":%d,"
               "\"vectors\":%lld,\"replicas\":%d,\"blocks\":%u,\"chunk\":%u,\"table\":%d,\"streaming_stores\":%d,\"digits\":",
               dtype_name(dtype), (long long)P.K, P.vb, (long long)total, k.nrep, P.blocks, k.chunk, k.nk > 0, k.stcs);
      P.desc = std::string(b) + joint_json(Y) + ",\"reduce_digits\":" + joint_json(Kd) + "}";
      *out = std::move(P);
      return AXE_OK;
    }
  }
  // generic: both layouts evaluated per element
  memset(&P.k4g, 0, sizeof(P.k4g));
  AXE_TRY(build_k0_side(S, sst, -1, &P.k4g.src));
  AXE_TRY(build_k0_side(D, dstst, -1, &P.k4g.dst));
  P.k4g.src.nR = 0;  // read the representative (reading R4)
  P.k4g.Y = D.ED;
  P.k4g.K = P.K;
  P.k4g.ER = D.ER;
  P.kind = 1;
  char b[192];
  snprintf(b, sizeof b, "{\"kernel\":\"reduce_generic\",\"dtype\":\"%s\",\"K\":%lld,\"elements\":%lld}",
           dtype_name(dtype), (long long)P.K, (long long)D.ED);
  P.desc = b;
  *out = std::move(P);
  return AXE_OK;
}

axe_status run_reduce(const ReducePlan &p, const void *src, void *dst, cudaStream_t st) {
  const uintptr_t s = (uintptr_t)src, d = (uintptr_t)dst;
  if (!src || !dst) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL buffer");
  if (s % p.align || d % p.align) AXE_FAIL(AXE_ERR_ALIGNMENT, "buffers must be %d-byte aligned for this plan", p.align);
  if (s < d + p.dst_bytes && d < s + p.src_bytes) AXE_FAIL(AXE_ERR_ALIAS, "source and destination buffers overlap");
  const int dep = stream_dependency(st, s, s + p.src_bytes, d, d + p.dst_bytes);
  cudaError_t e;
  if (p.kind == 2) {
    K4Params k = p.k4;
    k.dep = dep;
    e = launch_k4(k, p.dtype, p.vb, p.blocks, src, dst, st);
  } else {
    K4GParams k = p.k4g;
    k.dep = dep;
    e = launch_k4g(k, p.dtype, src, dst, st);
  }
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "reduce launch failed: %s", cudaGetErrorString(e));
  return AXE_OK;
}

}  // namespace axe

using namespace axe;

struct axe_reduce_plan {
  ReducePlan P;
};

extern "C" {

axe_status axe_reduce_plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                  const axe_storage *dst_st, int dtype, axe_reduce_plan **out) {
  if (!src || !dst || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  Storage ss, ds;
  AXE_TRY(make_storage(src_st, &ss));
  AXE_TRY(make_storage(dst_st, &ds));
  auto *h = new axe_reduce_plan;
  axe_status st = plan_reduce(src->L, ss, dst->L, ds, dtype, 16, &h->P);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *out = h;
  return AXE_OK;
}

axe_status axe_reduce_plan_execute(const axe_reduce_plan *plan, const void *src_ptr, void *dst_ptr, void *stream) {
  if (!plan) AXE_FAIL(AXE_ERR_INVALID_ARG, "plan is NULL");
  return run_reduce(plan->P, src_ptr, dst_ptr, (cudaStream_t)stream);
}

axe_status axe_reduce_plan_sizes(const axe_reduce_plan *plan, int64_t *src_bytes, int64_t *dst_bytes) {
  if (!plan || !src_bytes || !dst_bytes) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *src_bytes = plan->P.src_bytes;
  *dst_bytes = plan->P.dst_bytes;
  return AXE_OK;
}

axe_status axe_reduce_plan_describe(const axe_reduce_plan *plan, char *buf, int capacity) {
  if (!plan || !buf) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  if ((int)plan->P.desc.size() + 1 > capacity) AXE_FAIL(AXE_ERR_CAPACITY, "need %d bytes", (int)plan->P.desc.size() + 1);
  memcpy(buf, plan->P.desc.c_str(), plan->P.desc.size() + 1);
  return AXE_OK;
}

void axe_reduce_plan_destroy(axe_reduce_plan *plan) { delete plan; }

axe_status axe_reduce(const axe_layout *src, const axe_storage *src_st, const void *src_ptr, const axe_layout *dst,
                      const axe_storage *dst_st, void *dst_ptr, int dtype, void *stream) {
  if (!src || !dst) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL layout");
  static std::mutex mu;
  static std::unordered_map<std::string, std::shared_ptr<ReducePlan>> cache;
  Storage ss, ds;
  AXE_TRY(make_storage(src_st, &ss));
  AXE_TRY(make_storage(dst_st, &ds));
  uintptr_t al = (uintptr_t)src_ptr | (uintptr_t)dst_ptr | 16;
  const int align = (int)(al & (~al + 1));
  const std::string key = layout_key(src->L) + "#" + storage_key(ss) + "#" + layout_key(dst->L) + "#" +
                          storage_key(ds) + "#" + std::to_string(dtype) + "#" + std::to_string(align);
  std::shared_ptr<ReducePlan> p;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) p = it->second;
  }
  if (!p) {
    auto np = std::make_shared<ReducePlan>();
    AXE_TRY(plan_reduce(src->L, ss, dst->L, ds, dtype, align, np.get()));
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() > 4096) cache.clear();
    cache[key] = np;
    p = np;
  }
  return run_reduce(*p, src_ptr, dst_ptr, (cudaStream_t)stream);
}

}  // extern "C"
