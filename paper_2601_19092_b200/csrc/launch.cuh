// launch.cuh -- kernel launch helper: programmatic dependent launch (PDL).
//
// Every libaxe kernel starts with griddepcontrol.wait (a full dependency on the
// previous kernel in the stream, memory included) and then lets the next
// kernel be scheduled (griddepcontrol.launch_dependents).  Launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, back-to-back copies
// overlap launch latency and CTA rasterisation with the previous kernel's
// tail.  AXE_PDL=0 turns the attribute off (plain stream order).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace axe {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

inline bool pdl_enabled() {
  static int on = [] {
    const char *e = getenv("AXE_PDL");
    return (e && *e == '0') ? 0 : 1;
  }();
  return on != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  cfg.numAttrs = 0;
  if (pdl_enabled()) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 1;
  }
  cfg.attrs = attr;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace axe
