// capi.cpp -- the extern "C" boundary of libaxe (include/axe.h).
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>

#include "handles.hpp"

using namespace axe;

namespace axe {
extern std::atomic<int64_t> g_launches;
}

#define CHECK_NULL(p, what) \
  if (!(p)) AXE_FAIL(AXE_ERR_INVALID_ARG, "%s is NULL", what)

static axe_status to_iters(const axe_iter *it, int n, std::vector<Iter> *out) {
  if (n < 0 || (n > 0 && !it)) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad iter array");
  for (int i = 0; i < n; i++) {
    int a = intern_axis(it[i].axis ? it[i].axis : "m");
    if (a < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "iter %d: axis name is not an identifier", i);
    out->push_back(Iter{it[i].extent, it[i].stride, a});
  }
  return AXE_OK;
}

extern "C" {

const char *axe_last_error(void) { return axe::last_error(); }
const char *axe_version(void) { return "libaxe 0.1 (sm_100a)"; }
int64_t axe_kernel_launch_count(void) { return axe::g_launches.load(); }

axe_status axe_layout_create(const axe_iter *shard, int n_shard, const axe_iter *replica, int n_replica,
                             const axe_axis_coord *offset, int n_offset, axe_layout **out) {
  CHECK_NULL(out, "out");
  *out = nullptr;
  if (n_shard < 1) AXE_FAIL(AXE_ERR_INVALID_ARG, "n_shard must be >= 1 (Def. Layout, P:237)");
  std::vector<Iter> D, R;
  std::vector<std::pair<int, int64_t>> O;
  AXE_TRY(to_iters(shard, n_shard, &D));
  AXE_TRY(to_iters(replica, n_replica, &R));
  if (n_offset < 0 || (n_offset > 0 && !offset)) AXE_FAIL(AXE_ERR_INVALID_ARG, "bad offset array");
  for (int i = 0; i < n_offset; i++) {
    int a = intern_axis(offset[i].axis ? offset[i].axis : "m");
    if (a < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "offset %d: axis name is not an identifier", i);
    O.push_back({a, offset[i].value});
  }
  auto *h = new axe_layout;
  axe_status st = make_layout(std::move(D), std::move(R), std::move(O), &h->L);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *out = h;
  return AXE_OK;
}

void axe_layout_destroy(axe_layout *layout) { delete layout; }

axe_status axe_layout_info(const axe_layout *l, int64_t *E_D, int64_t *E_R, int *n_axes) {
  CHECK_NULL(l, "layout");
  if (E_D) *E_D = l->L.ED;
  if (E_R) *E_R = l->L.ER;
  if (n_axes) *n_axes = (int)l->L.axes.size();
  return AXE_OK;
}

axe_status axe_layout_axis_name(const axe_layout *l, int i, const char **name) {
  CHECK_NULL(l, "layout");
  CHECK_NULL(name, "name");
  if (i < 0 || i >= (int)l->L.axes.size()) AXE_FAIL(AXE_ERR_DOMAIN, "axis index %d out of range", i);
  *name = axis_name(l->L.axes[i]);
  return AXE_OK;
}

axe_status axe_layout_iters(const axe_layout *l, int which, axe_iter *out, int capacity, int *n) {
  CHECK_NULL(l, "layout");
  CHECK_NULL(n, "n");
  const std::vector<Iter> &v = which == 0 ? l->L.D : l->L.R;
  *n = (int)v.size();
  if (capacity < *n) AXE_FAIL(AXE_ERR_CAPACITY, "need %d iters", *n);
  for (int i = 0; i < *n; i++) out[i] = axe_iter{v[i].e, v[i].s, axis_name(v[i].a)};
  return AXE_OK;
}

axe_status axe_layout_offset(const axe_layout *l, axe_axis_coord *out, int capacity, int *n) {
  CHECK_NULL(l, "layout");
  CHECK_NULL(n, "n");
  *n = (int)l->L.O.size();
  if (capacity < *n) AXE_FAIL(AXE_ERR_CAPACITY, "need %d offsets", *n);
  for (int i = 0; i < *n; i++) out[i] = axe_axis_coord{axis_name(l->L.O[i].first), l->L.O[i].second};
  return AXE_OK;
}

axe_status axe_layout_eval(const axe_layout *l, int64_t x, int64_t *coords, int64_t capacity) {
  CHECK_NULL(l, "layout");
  CHECK_NULL(coords, "coords");
  if (x < 0 || x >= l->L.ED) AXE_FAIL(AXE_ERR_DOMAIN, "x = %lld outside [0, %lld)", (long long)x, (long long)l->L.ED);
  int64_t need = l->L.ER * (int64_t)l->L.axes.size();
  if (capacity < need) AXE_FAIL(AXE_ERR_CAPACITY, "need %lld values", (long long)need);
  eval_layout(l->L, x, coords);
  return AXE_OK;
}

axe_status axe_layout_canonicalize(const axe_layout *l, axe_layout **out, int *gap_ok) {
  CHECK_NULL(l, "layout");
  CHECK_NULL(out, "out");
  bool gc = true;
  auto *h = new axe_layout;
  h->L = canonicalize(l->L, &gc);
  if (gap_ok) *gap_ok = gc ? 1 : 0;
  *out = h;
  return AXE_OK;
}

axe_status axe_layout_bounds(const axe_layout *l, const char *axis, int64_t *mn, int64_t *mx) {
  CHECK_NULL(l, "layout");
  CHECK_NULL(mn, "min");
  CHECK_NULL(mx, "max");
  int a = intern_axis(axis ? axis : "m");
  if (a < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "axis name is not an identifier");
  axis_bounds(l->L, a, mn, mx);
  return AXE_OK;
}

// ------------------------------------------------------------------ copy
static axe_status plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                              const axe_storage *dst_st, int elem_size, int kernel, int max_align, CopyPlan *P,
                              int host_slabs = 0) {
  CHECK_NULL(src, "src layout");
  CHECK_NULL(dst, "dst layout");
  Storage ss, ds;
  AXE_TRY(make_storage(src_st, &ss));
  AXE_TRY(make_storage(dst_st, &ds));
  PlanRequest rq{&src->L, &dst->L, &ss, &ds, elem_size, kernel, max_align, -1};
  rq.host_slabs = host_slabs;
  return plan_copy(rq, P);
}

axe_status axe_copy_plan_create_ex(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                   const axe_storage *dst_st, int elem_size, int kernel, int host_slabs,
                                   axe_copy_plan **out) {
  CHECK_NULL(out, "out");
  *out = nullptr;
  if (host_slabs < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "host_slabs must be >= 0");
  auto *h = new axe_copy_plan;
  axe_status st = plan_create(src, src_st, dst, dst_st, elem_size, kernel, 16, &h->P, host_slabs);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *out = h;
  return AXE_OK;
}

axe_status axe_copy_plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                const axe_storage *dst_st, int elem_size, int kernel, axe_copy_plan **out) {
  CHECK_NULL(out, "out");
  *out = nullptr;
  auto *h = new axe_copy_plan;
  axe_status st = plan_create(src, src_st, dst, dst_st, elem_size, kernel, 16, &h->P);
  if (st != AXE_OK) {
    delete h;
    return st;
  }
  *out = h;
  return AXE_OK;
}

axe_status axe_copy_plan_execute(const axe_copy_plan *plan, const void *src_ptr, void *dst_ptr, void *stream) {
  CHECK_NULL(plan, "plan");
  return run_copy(plan->P, src_ptr, dst_ptr, (cudaStream_t)stream);
}

axe_status axe_copy_plan_execute_host(const axe_copy_plan *plan, const void *host_src, void *host_dst, void *dev_src,
                                      void *dev_dst, void *stream) {
  CHECK_NULL(plan, "plan");
  CHECK_NULL(host_src, "host_src");
  CHECK_NULL(host_dst, "host_dst");
  CHECK_NULL(dev_src, "dev_src");
  CHECK_NULL(dev_dst, "dev_dst");
  return run_copy_host(plan->P, host_src, host_dst, dev_src, dev_dst, (cudaStream_t)stream);
}

axe_status axe_copy_plan_sizes(const axe_copy_plan *plan, int64_t *src_bytes, int64_t *dst_bytes) {
  CHECK_NULL(plan, "plan");
  if (src_bytes) *src_bytes = plan->P.src_bytes;
  if (dst_bytes) *dst_bytes = plan->P.dst_bytes;
  return AXE_OK;
}

axe_status axe_copy_plan_describe(const axe_copy_plan *plan, char *buf, int capacity) {
  CHECK_NULL(plan, "plan");
  CHECK_NULL(buf, "buf");
  const std::string &d = plan->P.desc;
  if ((int)d.size() + 1 > capacity) AXE_FAIL(AXE_ERR_CAPACITY, "need %d bytes", (int)d.size() + 1);
  memcpy(buf, d.c_str(), d.size() + 1);
  return AXE_OK;
}

void axe_copy_plan_destroy(axe_copy_plan *plan) { delete plan; }

static std::mutex g_cache_mu;
static std::unordered_map<std::string, std::shared_ptr<CopyPlan>> g_cache;

axe_status axe_copy(const axe_layout *src, const axe_storage *src_st, const void *src_ptr, const axe_layout *dst,
                    const axe_storage *dst_st, void *dst_ptr, int elem_size, void *stream) {
  CHECK_NULL(src, "src layout");
  CHECK_NULL(dst, "dst layout");
  Storage ss, ds;
  AXE_TRY(make_storage(src_st, &ss));
  AXE_TRY(make_storage(dst_st, &ds));
  uintptr_t al = (uintptr_t)src_ptr | (uintptr_t)dst_ptr | 16;
  int align = (int)(al & (~al + 1));
  std::string key = layout_key(src->L) + "#" + storage_key(ss) + "#" + layout_key(dst->L) + "#" + storage_key(ds) +
                    "#" + std::to_string(elem_size) + "#" + std::to_string(align);
  std::shared_ptr<CopyPlan> p;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) p = it->second;
  }
  if (!p) {
    auto np = std::make_shared<CopyPlan>();
    PlanRequest rq{&src->L, &dst->L, &ss, &ds, elem_size, AXE_KERNEL_AUTO, align, -1};
    AXE_TRY(plan_copy(rq, np.get()));
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (g_cache.size() > 4096) g_cache.clear();
    g_cache[key] = np;
    p = np;
  }
  return run_copy(*p, src_ptr, dst_ptr, (cudaStream_t)stream);
}

}  // extern "C"
