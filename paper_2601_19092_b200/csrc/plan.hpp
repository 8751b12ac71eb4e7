// plan.hpp -- copy planning (host) and kernel launch entry points.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "common.hpp"
#include "kernels.cuh"

namespace axe {

enum KernelKind { KK_GENERIC = 1, KK_VECTOR = 2, KK_TMA = 3, KK_TILE = 4 };

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
};

struct PlanRequest {
  const Layout *src, *dst;
  const Storage *sst, *dstst;
  int es;
  int kernel;            // AXE_KERNEL_*
  int max_align;         // pointer alignment known to hold (bytes, power of 2, <= 16)
  int skip_axis;         // -1 for copy; gpuid id for redistribute pieces
};

axe_status plan_copy(const PlanRequest &rq, CopyPlan *out);
axe_status run_copy(const CopyPlan &p, const void *src, void *dst, cudaStream_t st);

// validation shared with redistribute
axe_status check_side(const Layout &L, const Storage &st, int skip_axis, const char *which);
axe_status check_injective(const Layout &dst, const Storage &st, int skip_axis);

// kernels.cu
cudaError_t launch_k0(const K0Params &p, const void *src, void *dst, cudaStream_t st);
cudaError_t launch_k1(const K1Params &p, int vb, unsigned blocks, const void *src, void *dst, cudaStream_t st);
int k1_unroll(int vb);
int num_sms();
int64_t kernel_launches();

}  // namespace axe
