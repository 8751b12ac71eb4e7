// tma_region.cpp -- executes the paper's TMA lowering (§3.4 "TMA asynchronous
// copy") on the device: the CuTensorMap comes from
// axe_tma_lower's encoding of the sliced, grouped L_G, and the shared-memory slot
// of every swizzle atom from the tiler T (L_S = T (x) atom).  Each atom is one TMA
// tensor load (hardware swizzle) into a shared ring slot, then one bulk store of
// the slot's bytes to the destination image at T(t) * |atom| -- so the
// destination holds exactly the shared-memory tensor L_S the lowering describes
// (an HBM image of it: L_S on m with the swizzle of the atom).
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "handles.hpp"

namespace axe {
int encode_tensor_map(void *out128, void *gaddr, const uint64_t dims[5], const uint64_t strides[4],
                      const uint32_t box[5], int swizzle_bytes);
cudaError_t launch_tma_region(const void *map128, const TmaAtom *atoms, uint32_t n, uint32_t box_bytes, void *dst,
                              cudaStream_t st);
}  // namespace axe

using namespace axe;

struct axe_tma_plan {
  axe_tma_desc desc;
  int es = 1;
  uint32_t box_bytes = 0;     // one atom: 8 rows x swizzle_bytes
  int64_t image_bytes = 0;    // |T| atoms
  std::vector<TmaAtom> host;  // per atom: tensor-map coordinates (byte units on dim 0) + image offset
  std::mutex mu;
  int dev = -1;
  TmaAtom *table = nullptr;  // device copy, uploaded by the first execute
  const void *map_for = nullptr;
  alignas(64) unsigned char map[128];
};

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
  *out = p;
  return AXE_OK;
}

axe_status axe_tma_plan_sizes(const axe_tma_plan *plan, int64_t *atoms, int64_t *image_bytes) {
  if (!plan) AXE_FAIL(AXE_ERR_INVALID_ARG, "plan is NULL");
  if (atoms) *atoms = (int64_t)plan->host.size();
  if (image_bytes) *image_bytes = plan->image_bytes;
  return AXE_OK;
}

axe_status axe_tma_plan_execute(axe_tma_plan *plan, const void *g_base, void *s_image, void *stream) {
  if (!plan || !g_base || !s_image) AXE_FAIL(AXE_ERR_INVALID_ARG, "NULL argument");
  const uint8_t *g = (const uint8_t *)g_base + plan->desc.base_bytes;
  if ((uintptr_t)g % 16 || (uintptr_t)s_image % 16)
    AXE_FAIL(AXE_ERR_ALIGNMENT, "region start and image must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lk(plan->mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "cudaGetDevice");
  if (!plan->table || plan->dev != dev) {
    if (plan->table) cudaFree(plan->table);
    plan->table = nullptr;
    const size_t bytes = plan->host.size() * sizeof(TmaAtom);
    cudaError_t e = cudaMalloc(&plan->table, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(plan->table, plan->host.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "atom table: %s", cudaGetErrorString(e));
    plan->dev = dev;
    plan->map_for = nullptr;
  }
  if (plan->map_for != g) {
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
    uint64_t last = 16;  // unused trailing dims: extent 1, the last real stride
    for (int i = 1; i < 5; i++) {
      if (i < d.rank) last = d.strides[i];
      strides[i - 1] = last;
    }
    const int r = encode_tensor_map(plan->map, (void *)g, dims, strides, box, d.swizzle_bytes);
    if (r != 0) AXE_FAIL(AXE_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", r);
    plan->map_for = g;
  }
  const cudaError_t e = launch_tma_region(plan->map, plan->table, (uint32_t)plan->host.size(), plan->box_bytes,
                                          s_image, st);
  if (e != cudaSuccess) AXE_FAIL(AXE_ERR_CUDA, "tma region launch: %s", cudaGetErrorString(e));
  return AXE_OK;
}

void axe_tma_plan_destroy(axe_tma_plan *plan) {
  if (!plan) return;
  if (plan->table) cudaFree(plan->table);
  delete plan;
}

}  // extern "C"
