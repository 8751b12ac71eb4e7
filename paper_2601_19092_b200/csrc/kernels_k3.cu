// kernels_k3.cu -- K3: warp-register permute through movmatrix (sm_100a).
//
// A register layout over (warp, lane, reg) (P:154-171 shows such layouts) is
// stored as a register dump (reading R17).  When the copy maps every 32-lane x
// 8-register block onto itself with an 8x8 transpose of each 32-bit register
// (the movmatrix.trans atom), each warp loads its block with one coalesced
// 16-byte load per lane, applies 4 movmatrix, and stores -- the data never
// leaves the register file.
#include <cuda_runtime.h>

#include <atomic>

#include "kernels.cuh"
#include "launch.cuh"

namespace axe {

extern std::atomic<int64_t> g_launches;

__device__ __forceinline__ uint32_t movm_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}

// One 512-byte block per warp per iteration at full occupancy (8 CTAs x 8 warps per SM, <= 32
// registers): measured on config 3b (B200) U = 1: 1422 us, U = 2: 1565 us, U = 4: 1669-1703 us.
// With U > 1 a warp's blocks lie a whole grid apart, so the loads in flight across the GPU
// scatter over U distant DRAM regions; with U = 1 they form one contiguous front.
constexpr int K3_WARPS = 8;
#ifndef AXE_K3_U
#define AXE_K3_U 1
#endif
#ifndef AXE_K3_MINB
#define AXE_K3_MINB 8
#endif
constexpr int K3_U = AXE_K3_U;

__global__ void __launch_bounds__(K3_WARPS * 32, AXE_K3_MINB) k3_movmatrix(const __grid_constant__ K3Params p,
                                                              const uint8_t *__restrict__ src,
                                                              uint8_t *__restrict__ dst) {
  if (p.dep) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * K3_WARPS + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * K3_WARPS;
  for (uint32_t b0 = warp; b0 < p.nblocks; b0 += nw * K3_U) {
    uint4 v[K3_U];
    int64_t dof[K3_U];
#pragma unroll
    for (int u = 0; u < K3_U; u++) {
      const uint32_t b = b0 + u * nw;
      if (b < p.nblocks) {
        int64_t so = p.sbase, d = p.dbase;
        uint32_t i = b;
#pragma unroll
        for (int k = K1_MAXD - 1; k >= 1; k--) {
          if (k >= p.nd) continue;
          uint32_t q = fdiv(p.fd[k], i);
          uint32_t dd = i - q * p.fd[k].d;
          i = q;
          so += (int64_t)dd * p.ss[k];
          d += (int64_t)dd * p.ds[k];
        }
        if (p.nd > 0) {
          so += (int64_t)i * p.ss[0];
          d += (int64_t)i * p.ds[0];
        }
        dof[u] = d + lane * 16;
        const uint8_t *a = src + swz(p.ssw, so + lane * 16);
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(a));
      }
    }
#pragma unroll
    for (int u = 0; u < K3_U; u++) {
      // movmatrix is warp-synchronous: every lane of the warp takes the same branch (b is warp-uniform)
      if (b0 + u * nw < p.nblocks) {
        uint4 o;
        o.x = movm_t(v[u].x);
        o.y = movm_t(v[u].y);
        o.z = movm_t(v[u].z);
        o.w = movm_t(v[u].w);
        for (int r = 0; r < p.nrep; r++) *reinterpret_cast<uint4 *>(dst + swz(p.dsw, dof[u] + p.rep[r])) = o;
      }
    }
  }
}

cudaError_t launch_k3(const K3Params &p, unsigned blocks, const void *src, void *dst, cudaStream_t st) {
  blocks = one_wave((const void *)k3_movmatrix, K3_WARPS * 32, 0, blocks);
  cudaError_t e = launch_ex(k3_movmatrix, dim3(blocks), dim3(K3_WARPS * 32), 0, st, p, (const uint8_t *)src,
                            (uint8_t *)dst);
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

}  // namespace axe
