// tma_ops.cuh -- mbarrier and cp.async.bulk helpers shared by the TMA-family kernels (sm_100a).
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace axe {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void *dst, const void *src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// TMA tensor load of a 5-D box (tensor-map coordinates c0..c4; dim 0 in bytes for the byte-element maps)
__device__ __forceinline__ void tma_load5(void *dst_smem, const void *map, uint64_t *bar, int c0, int c1, int c2,
                                          int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
      "%7}], [%2];" ::"r"(smem_u32(dst_smem)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
// L2 prefetches (no shared memory, no completion to wait for): pulling a box into L2 cannot return
// stale data -- L2 is where every SM's writes land -- so they may run before griddepcontrol.wait
__device__ __forceinline__ void tma_prefetch5(const void *map, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// box b of a lowered region (kernels.cuh TrProg / TmaAtom): tensor-map coordinates and image offset
__device__ __forceinline__ void tr_box(const TrParams &p, uint32_t b, int c[5], int64_t &off) {
  if (p.prog.nd < 0) {
    const TmaAtom a = p.atoms[b];
#pragma unroll
    for (int i = 0; i < 5; i++) c[i] = a.c[i];
    off = a.off;
    return;
  }
#pragma unroll
  for (int i = 0; i < 5; i++) c[i] = p.prog.c0[i];
  off = p.prog.off0;
#pragma unroll
  for (int k = 0; k < TR_MAXD; k++) {
    if (k >= p.prog.nd) break;
    const uint32_t q = fdiv(p.prog.fd[k], b);
    const uint32_t d = b - q * p.prog.fd[k].d;
    b = q;
#pragma unroll
    for (int i = 0; i < 5; i++) c[i] += (int)d * p.prog.dc[k][i];
    off += (int64_t)d * p.prog.doff[k];
  }
}

}  // namespace axe
