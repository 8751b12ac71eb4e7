// tma_region.cpp -- executes the paper's TMA lowering (§3.4 "TMA asynchronous
// copy") on the device: the CuTensorMap comes from
// axe_tma_lower's encoding of the sliced, grouped L_G, and the shared-memory slot
// of every swizzle atom from the tiler T (L_S = T (x) atom).  Each atom is one TMA
// tensor load (hardware swizzle) into a shared ring slot, then one bulk store of
// the slot's bytes to the destination image at T(t) * |atom| -- so the
// destination holds exactly the shared-memory tensor L_S the lowering describes
// (an HBM image of it: L_S on m with the swizzle of the atom).
#include <cuda_runtime.h>

#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "handles.hpp"

#include <unordered_map>
#include <map>
#include <array>

namespace axe {
int encode_tensor_map(void *out128, void *gaddr, const uint64_t dims[5], const uint64_t strides[4],
                      const uint32_t box[5], int swizzle_bytes);
cudaError_t launch_tma_region(const void *map128, TrParams p, int store, cudaStream_t st);
void stream_forget(cudaStream_t st);
uint32_t unit_chunk(int64_t dflt);
}  // namespace axe

using namespace axe;

static bool getenv_fuse() {  // AXE_TMA_FUSE=0: one atom per box (tests compare both forms)
  const char *e = getenv("AXE_TMA_FUSE");
  return !(e && *e == '0');
}

struct axe_tma_plan {
  axe_tma_desc desc;
  int es = 1;
  uint32_t box_bytes = 0;     // one atom: 8 rows x swizzle_bytes
  int64_t image_bytes = 0;    // |T| atoms
  std::vector<TmaAtom> host;  // per box: tensor-map coordinates (byte units on dim 0) + image offset
  int fuse = 1, fuse_dim = -1;  // atoms per box along the rows (box[fuse_dim] = fuse)
  TrProg prog{};              // the table as a mixed-radix program (prog.nd < 0: use the table)
  uint32_t chunk = 0;         // units per CTA of the in-order schedule (0: the persistent ring grid)
  int pair = 0;               // units of 2 boxes with contiguous image slots (TrParams::pair)
  std::mutex mu;              // guards the caches below
  std::map<int, TmaAtom *> tables;  // device -> its copy of the table (prog.nd < 0 only)
  std::unordered_map<const void *, std::array<unsigned char, 128>> maps;  // region start -> CUtensorMap
};

// Fit the box table with a mixed-radix program (kernels.cuh TrProg): the innermost digit's step is
// box 1 - box 0, its extent the longest run of equal steps (a divisor of what is left), and so on
// outwards; the result must reproduce every box exactly, else the kernel reads the table.
static TrProg fit_program(const std::vector<TmaAtom> &A) {
  TrProg p;
  memset(&p, 0, sizeof(p));
  p.nd = -1;
  const int64_t n = (int64_t)A.size();
  if (n == 0 || n >= (int64_t(1) << 32)) return p;
  auto vec = [](const TmaAtom &a, int64_t v[6]) {
    for (int i = 0; i < 5; i++) v[i] = a.c[i];
    v[5] = a.off;
  };
  int64_t a0[6];
  vec(A[0], a0);
  int nd = 0;
  int64_t stride = 1;
  int64_t delta[TR_MAXD][6], ext[TR_MAXD];
  while (stride < n) {
    if (nd == TR_MAXD || n % stride) return p;
    int64_t d[6], v[6];
    vec(A[(size_t)stride], v);
    for (int i = 0; i < 6; i++) d[i] = v[i] - a0[i];
    int64_t e = 2;
    while (e * stride < n) {
      vec(A[(size_t)(e * stride)], v);
      bool ok = true;
      for (int i = 0; i < 6; i++) ok = ok && v[i] == a0[i] + e * d[i];
      if (!ok) break;
      e++;
    }
    const int64_t left = n / stride;
    while (e > 1 && left % e) e--;
    if (e < 2) return p;
    for (int i = 0; i < 6; i++) {
      if (i < 5 && (d[i] > INT32_MAX || d[i] < INT32_MIN)) return p;
      delta[nd][i] = d[i];
    }
    ext[nd++] = e;
    stride *= e;
  }
  // verify every box
  for (int64_t b = 0; b < n; b++) {
    int64_t r = b, v[6], w[6];
    for (int i = 0; i < 6; i++) w[i] = a0[i];
    for (int k = 0; k < nd; k++) {
      const int64_t dk = r % ext[k];
      r /= ext[k];
      for (int i = 0; i < 6; i++) w[i] += dk * delta[k][i];
    }
    vec(A[(size_t)b], v);
    for (int i = 0; i < 6; i++)
      if (v[i] != w[i]) return p;
  }
  p.nd = nd;
  for (int i = 0; i < 5; i++) p.c0[i] = (int32_t)a0[i];
  p.off0 = a0[5];
  for (int k = 0; k < nd; k++) {
    p.fd[k] = make_fastdiv((uint32_t)ext[k]);
    for (int i = 0; i < 5; i++) p.dc[k][i] = (int32_t)delta[k][i];
    p.doff[k] = delta[k][5];
  }
  return p;
}

// the atom table on device `dev` (synchronous; not allowed inside graph capture); plan->mu held
static cudaError_t upload(axe_tma_plan *plan, int dev, TmaAtom **out) {
  TmaAtom *t = nullptr;
  const size_t bytes = plan->host.size() * sizeof(TmaAtom);
  cudaError_t e = cudaMalloc(&t, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(t, plan->host.data(), bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (t) cudaFree(t);
    return e;
  }
  plan->tables[dev] = t;
  *out = t;
  return cudaSuccess;
}

// the plan's CuTensorMap for region start g (cached per pointer); plan->mu held
static axe_status map_for(axe_tma_plan *plan, const uint8_t *g, std::array<unsigned char, 128> *map) {
  auto it = plan->maps.find(g);
  if (it != plan->maps.end()) {
    *map = it->second;
    return AXE_OK;
  }
  // uint8 elements: dim 0 in bytes, the other dims as lowered (byte strides)
  uint64_t dims[5], strides[4];
  uint32_t box[5];
  const axe_tma_desc &d = plan->desc;
  for (int i = 0; i < 5; i++) {
    dims[i] = i < d.rank ? d.dims[i] : 1;
    box[i] = i < d.rank ? d.box[i] : 1;
  }
  dims[0] *= (uint64_t)plan->es;
  box[0] *= (uint32_t)plan->es;
  if (plan->fuse > 1) box[plan->fuse_dim] = (uint32_t)plan->fuse;
  uint64_t last = 16;  // unused trailing dims: extent 1, the last real stride
  for (int i = 1; i < 5; i++) {
    if (i < d.rank) last = d.strides[i];
    strides[i - 1] = last;
  }
  alignas(64) unsigned char m[128];
  const int r = encode_tensor_map(m, (void *)g, dims, strides, box, d.swizzle_bytes);
  if (r != 0) AXE_FAIL(AXE_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", r);
  memcpy(map->data(), m, 128);
  if (plan->maps.size() >= 1024) plan->maps.clear();
  plan->maps.emplace(g, *map);
  return AXE_OK;
}

// launch parameters of a plan's region (the box program, or the table on the current device); plan->mu held
static axe_status region_params(axe_tma_plan *plan, const void *s_image, cudaStream_t st, int dep, TrParams *p) {
  memset(p, 0, sizeof(*p));
  p->prog = plan->prog;
  p->img = (uint8_t *)s_image;
  p->n = (uint32_t)plan->host.size();
  p->box = plan->box_bytes;
  p->slot = (plan->box_bytes + 1023) & ~1023u;
  p->dep = dep;
  p->chunk = plan->chunk;
  p->pair = plan->pair;
  p->reps.n = 1;
  if (p->prog.nd < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaGetDevice");
    auto it = plan->tables.find(dev);
    if (it != plan->tables.end()) {
      p->atoms = it->second;
    } else {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
        AXE_FAIL(AXE_ERR_CUDA, "the atom table is not on this device yet: execute once outside graph capture");
      TmaAtom *t = nullptr;
      const cudaError_t e = upload(plan, dev, &t);
      if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "atom table: %s", cudaGetErrorString(e));
      p->atoms = t;
    }
  }
  return AXE_OK;
}

static axe_status tma_plan_run(axe_tma_plan *plan, const void *g_base, const void *s_image, void *stream, int dep,
                               int store, const TmaReps *reps = nullptr) {
  if (!plan || !g_base || !s_image) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  const uint8_t *g = (const uint8_t *)g_base + plan->desc.base_bytes;
  if ((uintptr_t)g % 16 || (uintptr_t)s_image % 16)
    AXE_FAIL(AXE_ERR_ALIGNMENT, "region start and image must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  TrParams p;
  std::array<unsigned char, 128> map;
  {
    std::lock_guard<std::mutex> lk(plan->mu);
    AXE_TRY(region_params(plan, s_image, st, dep, &p));
    if (reps) p.reps = *reps;
    AXE_TRY(map_for(plan, g, &map));
  }
  const cudaError_t e = launch_tma_region(map.data(), p, store, st);
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "tma region launch: %s", cudaGetErrorString(e));
  return AXE_OK;
}


extern "C" {

axe_status axe_tma_plan_create(const axe_tma_desc *desc, const axe_layout *tiler, axe_tma_plan **out) {
  if (!desc || !tiler || !out) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  const int n = desc->rank;
  if (n < 2 || n > 5) AXE_FAIL(AXE_ERR_INVALID_ARG, "descriptor rank %d (2..5)", n);
  const int64_t es = (int64_t)desc->strides[0];
  if (es != 1 && es != 2 && es != 4 && es != 8 && es != 16) AXE_FAIL(AXE_ERR_INVALID_ARG, "element size %lld", (long long)es);
  if (desc->swizzle_bytes != 32 && desc->swizzle_bytes != 64 && desc->swizzle_bytes != 128)
    AXE_FAIL(AXE_ERR_INVALID_ARG, "swizzle %d B", desc->swizzle_bytes);
  int rank = 0;  // logical rank
  for (int d = 0; d < n; d++) rank = std::max(rank, desc->logical_dim[d] + 1);
  if (rank < 2 || rank > 5) AXE_FAIL(AXE_ERR_INVALID_ARG, "logical rank %d", rank);
  // region extent ES_j = product of the dims of logical dimension j, atom extent Ea_j = product of its box
  std::vector<int64_t> ES(rank, 1), Ea(rank, 1), Eo(rank);
  int64_t box = es;
  for (int d = 0; d < n; d++) {
    const int j = desc->logical_dim[d];
    if (j < 0) AXE_FAIL(AXE_ERR_INVALID_ARG, "logical_dim[%d] < 0", d);
    ES[j] *= (int64_t)desc->dims[d];
    Ea[j] *= (int64_t)desc->box[d];
    box *= (int64_t)desc->box[d];
  }
  if (box != 8 * desc->swizzle_bytes) AXE_FAIL(AXE_ERR_INVALID_ARG, "box of %lld B is not one swizzle atom", (long long)box);
  int64_t atoms = 1;
  for (int j = 0; j < rank; j++) {
    if (ES[j] % Ea[j]) AXE_FAIL(AXE_ERR_INVALID_ARG, "atom does not divide the region in dimension %d", j);
    Eo[j] = ES[j] / Ea[j];
    atoms *= Eo[j];
  }
  const Layout &T = tiler->L;
  if (T.ED != atoms || !T.R.empty()) AXE_FAIL(AXE_ERR_SIZE_MISMATCH, "tiler has %lld atoms, the region %lld", (long long)T.ED, (long long)atoms);
  if (atoms >= (int64_t(1) << 31)) AXE_FAIL(AXE_ERR_UNSUPPORTED, "too many atoms");
  auto *p = new axe_tma_plan;
  p->desc = *desc;
  p->es = (int)es;
  p->box_bytes = (uint32_t)box;
  p->host.resize((size_t)atoms);
  int64_t top = 0;
  for (int64_t t = 0; t < atoms; t++) {
    // atom multi-index over E_o (row-major), its origin u_j = t_j * Ea_j, decomposed over the
    // tensor-map dims of each logical dimension (innermost first)
    std::vector<int64_t> u(rank);
    int64_t r = t;
    for (int j = rank - 1; j >= 0; j--) {
      u[j] = (r % Eo[j]) * Ea[j];
      r /= Eo[j];
    }
    TmaAtom &a = p->host[(size_t)t];
    memset(&a, 0, sizeof(a));
    for (int d = 0; d < n; d++) {
      const int j = desc->logical_dim[d];
      const int64_t dd = (int64_t)desc->dims[d];
      a.c[d] = (int32_t)((u[j] % dd) * (d == 0 ? es : 1));
      u[j] /= dd;
    }
    // slot of atom t in L_S: T(t) atom spans (P:527 -- T's strides are in atoms)
    int64_t m = 0, rem = t;
    for (int i = (int)T.D.size() - 1; i >= 0; i--) {
      m += (rem % T.D[i].e) * T.D[i].s;
      rem /= T.D[i].e;
    }
    if (m < 0) {
      delete p;
      AXE_FAIL(AXE_ERR_UNSUPPORTED, "tiler maps an atom below the base");
    }
    a.off = m * box;
    top = std::max(top, a.off + box);
  }
  p->image_bytes = top;
  // fused boxes (desc->fused_rows > 8): f atoms stacked along the rows -- the row box dim rd (8 rows)
  // continued by dim rd + 1 -- that sit in f consecutive slots become one box of f x 8 rows (one TMA
  // instruction, "multiple atoms per instruction" as far as the box limits allow).  Checked
  // against T atom by atom; any mismatch keeps one atom per box.
  const int64_t f = desc->fused_rows / 8;
  int rd = -1;
  for (int d = 0; d + 1 < n; d++)
    if (desc->logical_dim[d] == rank - 2 && desc->box[d] == 8 && desc->dims[d] == 8 &&
        desc->logical_dim[d + 1] == rank - 2 && desc->box[d + 1] == 1 &&
        desc->strides[d + 1] == desc->strides[d] * 8) {
      rd = d;
      break;
    }
  if (f > 1 && rd >= 0 && (int64_t)desc->dims[rd + 1] % f == 0 && getenv_fuse()) {
    const int64_t rstep = Eo[rank - 1];  // atom-index step of one row tile (row-major over E_o)
    bool ok = true;
    std::vector<TmaAtom> heads;
    for (int64_t t = 0; t < atoms && ok; t++) {
      const TmaAtom &a = p->host[(size_t)t];
      if (a.c[rd + 1] % f) continue;
      for (int64_t k = 1; k < f && ok; k++) {
        const int64_t u = t + k * rstep;
        ok = u < atoms && p->host[(size_t)u].off == a.off + k * box && p->host[(size_t)u].c[rd + 1] == a.c[rd + 1] + k;
      }
      heads.push_back(a);
    }
    if (ok && (int64_t)heads.size() * f == atoms) {
      p->host.swap(heads);
      p->box_bytes = (uint32_t)(box * f);
      p->fuse = (int)f;
      p->fuse_dim = rd + 1;
    }
  }
  p->prog = fit_program(p->host);
  // beyond 64 MiB of boxes, the in-order schedule with 4 boxes per CTA (kernels.cuh unit_range;
  // profiles/r02_sweep_front.log: config 2 at 16384^2 158.7 us vs 179.6, 8192^2 40.6 vs 45.0); the
  // bench's 4096^2 keeps the persistent ring, which holds the whole copy in flight (10.0 us vs 11.0)
  p->chunk = unit_chunk((int64_t)p->host.size() * p->box_bytes > (int64_t(64) << 20) ? 4 : 0);
  {  // pairs of consecutive boxes whose image slots are contiguous move as one ring unit: two TMA tensor
     // ops and ONE image-side bulk copy of both (config 2: 10.12 -> 9.81 us per dependent step, the bench
     // 6520 -> 6814 GB/s; reverse at 16384^2 162.4 -> 160.0; profiles/r02_lowered_pair.log).
     // AXE_TMA_PAIR=0: one box per unit
    const char *pe = getenv("AXE_TMA_PAIR");
    const int want = (pe && *pe) ? atoi(pe) : 2;  // boxes per unit (0 / 1: one)
    int f = want >= 4 ? 4 : want >= 2 ? 2 : 1;
    for (; f > 1; f /= 2) {
      bool ok = p->host.size() % f == 0 && p->box_bytes % 1024 == 0;
      for (size_t k = 0; ok && k < p->host.size(); k += f)
        for (int j = 1; ok && j < f; j++) ok = p->host[k + j].off == p->host[k].off + (int64_t)j * p->box_bytes;
      if (ok) break;
    }
    p->pair = f > 1 ? f : 0;
  }
  const char *force_table = getenv("AXE_TMA_REGION_TABLE");  // tests: run the table form
  if (force_table && *force_table == '1') p->prog.nd = -1;
  // a table the program does not reproduce is uploaded now when a device is current (so executes can
  // be graph-captured); on a host without a GPU the first execute would upload -- there is no execute
  int ndev = 0, dev = 0;
  if (p->prog.nd < 0 && cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0 && cudaGetDevice(&dev) == cudaSuccess) {
    TmaAtom *t = nullptr;
    upload(p, dev, &t);
  }
  cudaGetLastError();  // (clear a sticky-free error from the probe)
  *out = p;
  return AXE_OK;
}

axe_status axe_tma_plan_sizes(const axe_tma_plan *plan, int64_t *atoms, int64_t *boxes, int64_t *image_bytes) {
  if (!plan) AXE_FAIL(AXE_ERR_INVALID_ARG, "plan is NULL");
  if (atoms) *atoms = (int64_t)plan->host.size() * plan->fuse;
  if (boxes) *boxes = (int64_t)plan->host.size();
  if (image_bytes) *image_bytes = plan->image_bytes;
  return AXE_OK;
}

// The public executes wait for everything before them on the stream (dep = 1) and, since the kernel
// lets its dependents launch at entry without joining the copy planner's byte-range window, reset
// that window: the next libaxe kernel on the stream waits for this one.
axe_status axe_tma_plan_execute(axe_tma_plan *plan, const void *g_base, void *s_image, void *stream) {
  AXE_TRY(tma_plan_run(plan, g_base, s_image, stream, 1, 0));
  stream_forget((cudaStream_t)stream);
  return AXE_OK;
}

axe_status axe_tma_plan_execute_store(axe_tma_plan *plan, void *g_base, const void *s_image, void *stream) {
  AXE_TRY(tma_plan_run(plan, g_base, s_image, stream, 1, 1));
  stream_forget((cudaStream_t)stream);
  return AXE_OK;
}

void axe_tma_plan_destroy(axe_tma_plan *plan) {
  if (!plan) return;
  for (auto &t : plan->tables) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(t.first);
    cudaFree(t.second);
    cudaSetDevice(cur);
  }
  delete plan;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// The lowering as a copy schedule (AXE_KERNEL_LOWERED).  The joint digits of the copy, destination-
// outermost first, are the logical dimensions of both tensors: L_G = (e_k):(src stride_k) + the
// source base, L_S = (e_k):(dst stride_k).  When the destination storage carries a TMA swizzle and
// L_S tiles its atom, axe_tma_lower gives the tensor map and T, and every (fused) atom box is one
// TMA load + one bulk store -- config 2 is 4096 tiles x 8 atoms, fused into 64-row boxes.
namespace axe {

std::string joint_json(const std::vector<Joint> &J);

bool build_lowered(const std::vector<Joint> &J0, const Linear &ls, const Linear &ld, const Storage &sst,
                   const Storage &dstst, int es, CopyPlan *P, std::string *why) {
  auto fail = [&](const std::string &m) {
    *why = "lowered: " + m;
    return false;
  };
  auto tma_swz = [](const Storage &t) { return t.swz_b >= 1 && t.swz_b <= 3 && t.swz_m == 4 && t.swz_s == 3; };
  // load direction: unswizzled source = L_G, swizzled destination = L_S image; store direction
  // (the reverse, e.g. config 2's tiles -> row-major): swizzled source = L_S image, destination = L_G
  const bool store = !tma_swz(dstst);
  const Storage &img_st = store ? sst : dstst, &g_st = store ? dstst : sst;
  const Linear &lg = store ? ld : ls, &li = store ? ls : ld;
  if (!tma_swz(img_st)) return fail("neither side carries a TMA swizzle (Swizzle<1..3,4,3>)");
  if (g_st.swz_b) return fail("both sides swizzled");
  const int sw = 16 << img_st.swz_b;
  if ((li.base * es) % (8 * sw)) return fail("the swizzled side's base is not a whole swizzle atom");
  // destination replicas: every box leaves once per replica (load direction; a TMA store writes one place)
  std::vector<int64_t> reps{0};
  for (auto &r : ld.R) {
    std::vector<int64_t> nx;
    for (int64_t x : reps)
      for (int64_t q = 0; q < r.e; q++) nx.push_back(x + q * r.s);
    reps.swap(nx);
    if (reps.size() > 4096) break;
  }
  std::sort(reps.begin(), reps.end());
  reps.erase(std::unique(reps.begin(), reps.end()), reps.end());
  if (reps.size() > 1 && store) return fail("destination replicas with TMA stores");
  if ((int)reps.size() > K1_MAXREP) return fail("too many replicas");
  for (int64_t r : reps)
    if ((r * es) % (8 * sw)) return fail("replica offsets are not whole swizzle atoms");
  std::vector<Joint> J;
  for (auto &j : J0)
    if (j.e > 1) J.push_back(store ? Joint{j.e, j.ds, j.ss, j.ddev, j.sdev} : j);  // (ss: G side, ds: image side)
  std::stable_sort(J.begin(), J.end(), [](const Joint &a, const Joint &b) { return std::llabs(a.ds) > std::llabs(b.ds); });
  const int rank = (int)J.size();
  if (rank < 2 || rank > 5) return fail("needs 2..5 joint digits");
  const int m = axis_m();
  std::vector<Iter> DG, DS;
  std::vector<int64_t> E;
  for (auto &j : J) {
    if (j.ss <= 0 || j.ds <= 0) return fail("negative strides");
    DG.push_back(Iter{j.e, j.ss, m});
    DS.push_back(Iter{j.e, j.ds, m});
    E.push_back(j.e);
  }
  axe_layout G, S;
  std::vector<std::pair<int, int64_t>> O;
  if (lg.base) O.push_back({m, lg.base});
  if (make_layout(DG, {}, O, &G.L) != AXE_OK || make_layout(DS, {}, {}, &S.L) != AXE_OK) return fail(last_error());
  axe_tma_desc d;
  axe_layout *T = nullptr;
  if (axe_tma_lower(&G, E.data(), nullptr, nullptr, &S, E.data(), rank, es, sw, &d, &T) != AXE_OK)
    return fail(last_error());
  axe_tma_plan *tp = nullptr;
  const axe_status st = axe_tma_plan_create(&d, T, &tp);
  axe_layout_destroy(T);
  if (st != AXE_OK) return fail(last_error());
  P->lowered = std::shared_ptr<axe_tma_plan>(tp, axe_tma_plan_destroy);
  P->lowered_dst_off = li.base * es;  // byte offset of the L_S image in its buffer
  P->lowered_store = store;
  memset(&P->lowered_reps, 0, sizeof(P->lowered_reps));
  P->lowered_reps.n = (int)reps.size();
  for (size_t i = 0; i < reps.size(); i++) P->lowered_reps.r[i] = reps[i] * es;
  P->align = 16;
  int64_t total = 1;
  for (auto &j : J) total *= j.e;
  P->covers_all = total * (int64_t)reps.size() == dstst.cells;
  char b[320];
  snprintf(b, sizeof b,
           "{\"kernel\":\"lowered\",\"mode\":\"%s\",\"atoms\":%lld,\"boxes\":%lld,\"box_bytes\":%u,\"swizzle\":%d,"
           "\"replicas\":%d,\"box_program_digits\":%d,\"chunk\":%u,\"pair\":%d,\"tensor_map\":{\"dims\":[",
           store ? "bulk-load/tensor-store" : "tensor-load/bulk-store", (long long)(tp->host.size() * tp->fuse),
           (long long)tp->host.size(), tp->box_bytes, sw, (int)reps.size(), tp->prog.nd, tp->chunk, tp->pair);
  std::string s = b;
  for (int i = 0; i < d.rank; i++) s += (i ? "," : "") + std::to_string(d.dims[i]);
  s += "],\"strides\":[";
  for (int i = 0; i < d.rank; i++) s += (i ? "," : "") + std::to_string(d.strides[i]);
  s += "],\"box\":[";
  for (int i = 0; i < d.rank; i++)
    s += (i ? "," : "") + std::to_string(i == tp->fuse_dim ? (uint32_t)tp->fuse : d.box[i]);
  s += "],\"base\":" + std::to_string(d.base_bytes) + "},\"joint\":" + joint_json(J0) + "}";
  P->desc = s;
  return true;
}

uint32_t lowered_box_bytes(const CopyPlan &P) { return P.lowered ? P.lowered->box_bytes : 0; }

axe_status run_lowered(const CopyPlan &P, const void *src, void *dst, cudaStream_t st, int dep) {
  if (P.lowered_store) return tma_plan_run(P.lowered.get(), dst, (const uint8_t *)src + P.lowered_dst_off, st, dep, 1);
  return tma_plan_run(P.lowered.get(), src, (uint8_t *)dst + P.lowered_dst_off, st, dep, 0, &P.lowered_reps);
}

}  // namespace axe
