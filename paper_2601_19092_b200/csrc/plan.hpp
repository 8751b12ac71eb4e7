// plan.hpp -- copy planning (host) and kernel launch entry points.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <memory>
#include <mutex>
#include <string>

#include "common.hpp"
#include "kernels.cuh"

namespace axe {

enum KernelKind { KK_GENERIC = 1, KK_VECTOR = 2, KK_TMA = 3, KK_TILE = 4, KK_REGISTER = 5, KK_SHUFFLE = 7, KK_TRANSPOSE = 8, KK_LOWERED = 9, KK_DUAL = 10, KK_RAGGED = 11 };

struct CopyPlan {
  int kernel = KK_GENERIC;
  int es = 0;
  int64_t src_bytes = 0, dst_bytes = 0;
  int align = 1;         // required alignment of both device pointers (bytes)
  K0Params k0;
  K1Params k1;
  int vb = 0;            // K1 vector bytes
  unsigned blocks = 0;
  std::string desc;      // JSON
  // the composed problem (kept for describe / redistribute reuse)
  std::vector<Joint> joint;
  bool linear = false;
  bool covers_all = false;  // the destination image is every cell of the dst storage
  // K1-TMA: the tensor-map side (mode 0: src, mode 1: dst), encoded per pointer at execute
  TmaParams tma;
  uint64_t tm_dims[5] = {1, 1, 1, 1, 1}, tm_strides[4] = {16, 16, 16, 16};
  uint32_t tm_box[5] = {1, 1, 1, 1, 1};
  int tm_swizzle = 0;       // bytes: 0, 32, 64, 128
  int64_t tm_base = 0;      // byte offset of coordinate 0 from the buffer base
  std::shared_ptr<struct TmaCache> tm_cache;
  // K2 tile
  K2Params k2;
  int k2_vs = 0, k2_vd = 0, k2_gb = 0;
  double k1_sector_eff = 1.0;  // K1: useful bytes / 32-byte sectors touched by one CTA's vectors (min of both sides)
  // K3 movmatrix
  K3Params k3;
  // K6 granule transpose (warp shuffles)
  K6Params k6;
  // K7 register-block transpose
  K7Params k7;
  // K8 dual decoding (non-nested digit systems)
  K8Params k8;
  // K9 ragged transpose
  K9Params k9;
  // the paper's TMA lowering as the schedule (tma_region.cpp): plan + destination byte offset of L_S
  std::shared_ptr<axe_tma_plan> lowered;
  int64_t lowered_dst_off = 0;  // byte offset of the L_S image (the destination, or the source when storing)
  bool lowered_store = false;    // image -> G (bulk load + TMA tensor store)
  TmaReps lowered_reps{};        // destination replica byte offsets (load direction)
  // host-buffer pipeline (axe_copy_plan_execute_host): the copy splits into n_chunks
  // independent slabs (a joint digit spanning both whole buffers); each slab's
  // H2D, kernel and D2H run on three streams so PCIe traffic in both directions overlaps.
  std::shared_ptr<CopyPlan> chunk;
  int n_chunks = 0;
  std::shared_ptr<struct HostPipe> pipe;
};

struct HostPipe {
  std::mutex mu;
  int device = -1;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev;  // 3 per chunk + 2
  ~HostPipe();
};

axe_status run_copy_host(const CopyPlan &p, const void *host_src, void *host_dst, void *dev_src, void *dev_dst,
                         cudaStream_t st);

bool build_k3(const std::vector<Joint> &J, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why);
cudaError_t launch_k3(const K3Params &p, unsigned blocks, const void *src, void *dst, cudaStream_t st);
bool build_k3_bulk(CopyPlan *P, std::string *why);
bool build_k6(const std::vector<Joint> &J, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why);
cudaError_t launch_k6(const K6Params &p, unsigned blocks, const void *src, void *dst, cudaStream_t st);
bool build_k7(const std::vector<Joint> &J, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why, bool forced = false);
cudaError_t launch_k7(const K7Params &p, int es, unsigned blocks, const void *src, void *dst, cudaStream_t st);  // K3 as K1-TMA mode 2 + movmatrix in smem
bool build_k9(const std::vector<Joint> &J, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, CopyPlan *P, std::string *why);
cudaError_t launch_k9(const K9Params &p, int es, const void *src, void *dst, cudaStream_t st);
bool build_k8(const Linear &ls, const Linear &ld, const Storage &sst, const Storage &dstst, int es, int max_align,
              CopyPlan *P, std::string *why);
cudaError_t launch_k8(const K8Params &p, int vb, const void *src, void *dst, cudaStream_t st);
cudaError_t launch_k8_bulk(K8Params p, const void *src, void *dst, cudaStream_t st);

bool build_k2(const std::vector<Joint> &J, const Linear &ls, const Linear &ld, const Storage &sst,
              const Storage &dstst, int es, int max_align, CopyPlan *P, std::string *why);
cudaError_t launch_k2(const K2Params &p, int vs, int vd, int gb, unsigned blocks, const void *src, void *dst,
                      cudaStream_t st);
std::string joint_json(const std::vector<Joint> &J);
bool build_lowered(const std::vector<Joint> &J0, const Linear &ls, const Linear &ld, const Storage &sst,
                   const Storage &dstst, int es, CopyPlan *P, std::string *why);
axe_status run_lowered(const CopyPlan &P, const void *src, void *dst, cudaStream_t st, int dep);
uint32_t lowered_box_bytes(const CopyPlan &P);

struct TmaCache {
  std::mutex mu;
  std::vector<std::pair<const void *, std::array<uint64_t, 16>>> maps;  // LRU-ish, small
};

struct PlanRequest {
  const Layout *src, *dst;
  const Storage *sst, *dstst;
  int es;
  int kernel;            // AXE_KERNEL_*
  int max_align;         // pointer alignment known to hold (bytes, power of 2, <= 16)
  int skip_axis;         // -1 for copy; gpuid id for redistribute pieces
  int no_chunk = 0;      // do not build the host-pipeline slab plan
  int host_slabs = 0;    // > 0: at most this many host-pipeline slabs (else AXE_HOST_CHUNKS, default 8)
};

void stream_forget(cudaStream_t st);
axe_status plan_chunks(const PlanRequest &rq, const std::vector<Joint> &J, const Linear &ls, const Linear &ld,
                       CopyPlan *P);

axe_status plan_copy(const PlanRequest &rq, CopyPlan *out);
axe_status run_copy(const CopyPlan &p, const void *src, void *dst, cudaStream_t st);

// validation shared with redistribute
axe_status check_side(const Layout &L, const Storage &st, int skip_axis, const char *which);
axe_status check_injective(const Layout &dst, const Storage &st, int skip_axis);

// kernels.cu
cudaError_t launch_k0(const K0Params &p, const void *src, void *dst, cudaStream_t st);
cudaError_t launch_k1(const K1Params &p, int vb, unsigned blocks, const void *src, void *dst, cudaStream_t st);
int k1_unroll(int vb);
// kernels_tma.cu
int encode_tensor_map(void *out128, void *gaddr, const uint64_t dims[5], const uint64_t strides[4],
                      const uint32_t box[5], int swizzle_bytes);
cudaError_t launch_tma(const void *map128, const TmaParams &p, unsigned blocks, const void *src, void *dst,
                       cudaStream_t st);
size_t tma_smem_bytes(const TmaParams &p);
int num_sms();
// persistent-grid cap: num_sms() * per_sm CTAs (AXE_ONESHOT=1: no cap -- one CTA per work unit)
int64_t grid_cap(int64_t per_sm);
uint32_t unit_chunk(int64_t dflt);
unsigned chunk_grid(int64_t units, uint32_t chunk, unsigned persistent);
int64_t kernel_launches();
// 1 if a kernel reading [s0,s1) and writing [d0,d1) on stream st must wait for
// the previous libaxe kernel on st (records the new kernel as the previous one).
int stream_dependency(cudaStream_t st, uintptr_t s0, uintptr_t s1, uintptr_t d0, uintptr_t d1);
axe_status build_k0_side(const Layout &L, const Storage &st, int skip_axis, K0Side *S);
Swz make_swz(const Storage &st);

// ---- K4 reduction over the leading logical dimension (plan_reduce.cpp, kernels_reduce.cu)
struct ReducePlan {
  int kind = 0;          // 1: generic (k4_generic), 2: vector (k4_reduce)
  int dtype = 0, es = 0;
  int64_t K = 1;         // summands per output element
  int64_t src_bytes = 0, dst_bytes = 0;
  int align = 1, vb = 0;
  unsigned blocks = 1;
  K4Params k4;
  K4GParams k4g;
  std::string desc;
};
int dtype_size(int dtype);
axe_status plan_reduce(const Layout &src, const Storage &sst, const Layout &dst, const Storage &dstst, int dtype,
                       int max_align, ReducePlan *out);
axe_status run_reduce(const ReducePlan &p, const void *src, void *dst, cudaStream_t st);
cudaError_t launch_k4(const K4Params &p, int dtype, int vb, unsigned blocks, const void *src, void *dst,
                      cudaStream_t st);
cudaError_t launch_k4g(const K4GParams &p, int dtype, const void *src, void *dst, cudaStream_t st);
cudaError_t launch_k4_multimem(const K4Params &p, int dtype, unsigned blocks, const void *mc, void *dst,
                               cudaStream_t st);
cudaError_t launch_k4_peer(const K4Params &p, const K4Ptrs &q, int dtype, int vb, unsigned blocks, void *dst,
                           cudaStream_t st);

}  // namespace axe
