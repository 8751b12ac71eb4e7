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
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <utility>

namespace axe {

int num_sms();

// Grid-stride kernels: a grid larger than (resident CTAs per SM) x SMs only adds a partial
// second wave that runs at low occupancy at the end (e.g. 8 CTAs/SM requested, 6 resident:
// 1.33 waves).  Cap the grid at exactly one full wave of the kernel's measured occupancy.
inline unsigned one_wave(const void *kern, int threads, size_t smem, unsigned blocks) {
  static std::mutex mu;
  static std::map<std::tuple<const void *, int, size_t>, int> occ;
  int o = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(kern, threads, smem);
    auto it = occ.find(key);
    if (it != occ.end()) {
      o = it->second;
    } else {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem) != cudaSuccess) o = 0;
      occ[key] = o;
    }
  }
  if (o <= 0) return blocks;
  const unsigned cap = (unsigned)(o * num_sms());
  return blocks > cap ? cap : blocks;
}

// Opt a kernel into more than 48 KiB of dynamic shared memory, once per (device, kernel): the
// attribute belongs to the current device's context, and several host threads may launch at once.
inline cudaError_t smem_attr(const void *kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void *>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, kern})) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({dev, kern});
  return e;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// L2 prefetch of the line holding p (a hint: no data returns, nothing to wait for; issued before
// griddepcontrol.wait it cannot observe stale data -- every SM's writes land in L2, R28)
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.L2 [%0];" ::"l"(p)); }
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
