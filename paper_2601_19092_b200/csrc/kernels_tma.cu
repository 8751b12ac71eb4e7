// kernels_tma.cu -- K1-TMA: the paper's TMA copy lowering on sm_100a.
//
// One elected thread per CTA runs an S-stage ring of shared-memory boxes:
//   mode 0: cp.async.bulk.tensor (TMA, 5-D map, swizzle in smem) global->smem,
//           then cp.async.bulk smem->global for every destination replica;
//   mode 1: cp.async.bulk global->smem, then cp.async.bulk.tensor smem->global;
//   mode 2: cp.async.bulk global->smem and cp.async.bulk smem->global (a run
//           contiguous on both sides: no tensor map, no thread touches data).
// The swizzled smem image of a box is exactly the destination's swizzled bytes
// (SW128: 16-byte chunk j of row r at j ^ (r mod 8), reading R16), so no thread
// ever touches the data.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kernels.cuh"
#include "launch.cuh"
#include "tma_ops.cuh"

namespace axe {

extern std::atomic<int64_t> g_launches;

__device__ __forceinline__ void tma_store5(const CUtensorMap *map, const void *src_smem, int c0, int c1, int c2, int c3,
                                           int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(map),
      "r"(smem_u32(src_smem)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
struct BoxAddr {
  int c[5];
  int64_t boff, soff;
};

__device__ __forceinline__ BoxAddr box_addr(const TmaParams &p, uint32_t b) {
  BoxAddr a;
#pragma unroll
  for (int i = 0; i < 5; i++) a.c[i] = 0;
  a.boff = p.bbase;
  a.soff = p.sbase;
#pragma unroll
  for (int k = TMA_MAXD - 1; k >= 0; k--) {
    if (k >= p.nd) continue;
    uint32_t d;
    if (k > 0) {
      uint32_t q = fdiv(p.fd[k], b);
      d = b - q * p.fd[k].d;
      b = q;
    } else {
      d = b;
    }
#pragma unroll
    for (int i = 0; i < 5; i++)
      if (p.cdim[k] == i) a.c[i] += (int)d * p.cmul[k];
    a.boff += (int64_t)d * p.bstride[k];
    a.soff += (int64_t)d * p.sstride[k];
  }
  return a;
}

constexpr int TMA_MAX_STAGES = 16;

__device__ __forceinline__ uint32_t movm_trans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}

// p.xform == 1 (K3-TMA): between the bulk load and the bulk store the whole warp applies
// movmatrix.m8n8.trans.b16 to every 32-bit word of each 512-byte block of the box in shared memory
// (lane l owns bytes [16 l, 16 l + 16) of the block: the K3 register image), then the stores leave.
__global__ void __launch_bounds__(32) k1_tma(const __grid_constant__ CUtensorMap map, const __grid_constant__ TmaParams p,
                                             const uint8_t *__restrict__ src, uint8_t *__restrict__ dst) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[TMA_MAX_STAGES];
  const bool leader = threadIdx.x == 0;
  if (!p.xform && !leader) return;
  const UnitRange R = unit_range(p.nboxes, p.chunk);
  if (p.dep) {
    if (leader) {  // the first half-ring of boxes into L2 while the previous kernel drains (R28)
      const int np = (int)p.prefetch;
      for (int k = 0; k < np && R.lo + (uint32_t)k * R.step < R.end; k++) {
        const BoxAddr a = box_addr(p, R.lo + (uint32_t)k * R.step);
        if (p.mode == 0)
          tma_prefetch5(&map, a.c[0], a.c[1], a.c[2], a.c[3], a.c[4]);
        else
          bulk_prefetch(src + (p.mode == 2 ? a.soff : a.boff), p.box_bytes);
      }
    }
    pdl_wait();
  }
  pdl_launch_dependents();
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = p.stages;
  const uint32_t B = p.box_bytes, SL = p.slot_bytes;
  if (leader) {
    for (int s = 0; s < S; s++) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  if (p.xform) __syncwarp();

  const uint32_t first = R.lo, step = R.step;
  const uint32_t mine = first < R.end ? (R.end - first + step - 1) / step : 0;

  auto issue_load = [&](uint32_t k) {
    const int s = (int)(k % (uint32_t)S);
    BoxAddr a = box_addr(p, first + k * step);
    mbar_expect_tx(&full[s], B);
    if (p.mode == 0)
      tma_load5(smem + (size_t)s * SL, &map, &full[s], a.c[0], a.c[1], a.c[2], a.c[3], a.c[4]);
    else
      bulk_load(smem + (size_t)s * SL, src + (p.mode == 2 ? a.soff : a.boff), B, &full[s]);
  };

  const uint32_t pre = mine < (uint32_t)S ? mine : (uint32_t)S;
  if (leader)
    for (uint32_t k = 0; k < pre; k++) issue_load(k);
  for (uint32_t k = 0; k < mine; k++) {
    const int s = (int)(k % (uint32_t)S);
    mbar_wait(&full[s], (k / (uint32_t)S) & 1u);
    if (p.xform) {
      __syncwarp();  // reconverge after the per-lane barrier waits: movmatrix is .sync.aligned
      uint8_t *box = smem + (size_t)s * SL;
      for (uint32_t blk = 0; blk < B / 512; blk++) {
        uint4 *q = reinterpret_cast<uint4 *>(box + blk * 512 + threadIdx.x * 16);
        uint4 v = *q;
        v.x = movm_trans(v.x);
        v.y = movm_trans(v.y);
        v.z = movm_trans(v.z);
        v.w = movm_trans(v.w);
        *q = v;
      }
      fence_async_smem();  // the generic-proxy writes above before the async-proxy bulk store reads them
      __syncwarp();
    }
    if (!leader) continue;
    BoxAddr a = box_addr(p, first + k * step);
    if (p.mode != 1) {
      for (int r = 0; r < p.nrep; r++) bulk_store(dst + a.boff + p.rep[r], smem + (size_t)s * SL, B);
    } else {
      tma_store5(&map, smem + (size_t)s * SL, a.c[0], a.c[1], a.c[2], a.c[3], a.c[4]);
    }
    bulk_commit();
    // the stage of box k-1 is free once its store has read shared memory
    if (k >= 1 && k - 1 + S < mine) {
      bulk_wait_read<1>();
      issue_load(k - 1 + S);
    }
  }
  if (leader) bulk_wait_all();
}

// The lowered TMA region (tma_region.cpp): a persistent grid (one CTA of one issuing thread per SM by
// default), each CTA owning a contiguous range of boxes and a deep ring of 1 KiB-aligned slots that
// fills its shared memory (config 2: 28 slots of 8 KiB -- the SM's whole share of the 4096 boxes is
// in flight at once, so the first wave of loads covers the copy and no CTA waits on a ring refill).
// Load direction (G -> image): tensor load (the hardware applies the atom's swizzle), then one bulk
// store of the slot into the image at the tiler's offset.  Store direction (image -> G): bulk load
// of the slot from the image, then one tensor store (the hardware un-swizzles).  Both copies of a
// box run in the async proxy, so no proxy fence is needed.  Box coordinates come from the fitted
// mixed-radix program (no dependent global load before a TMA issue); the table is the fallback.
constexpr int TR_STAGES = 32;  // ring capacity (slots per CTA)
#ifndef AXE_TR_LAG
#define AXE_TR_LAG 1
#endif
// a slot is refilled once the store TR_LAG units back has read it (with 16 KiB two-box units, lag 1:
// config 2 9.69 us vs 9.83 with lag 2 and 9.98 with 3; profiles/r02_lowered_pair.log)
constexpr int TR_LAG = AXE_TR_LAG;

template <bool STORE>
__global__ void __launch_bounds__(32, 1) k_tma_region(const __grid_constant__ CUtensorMap map,
                                                      const __grid_constant__ TrParams p) {
  extern __shared__ __align__(1024) uint8_t raw[];
  __shared__ __align__(8) uint64_t full[TR_STAGES];
  if (threadIdx.x != 0) {
    pdl_launch_dependents();
    return;
  }
  uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  // a unit = F consecutive boxes whose image slots are contiguous (p.pair: F = 2, one bulk copy of 2 boxes
  // on the image side); a ring slot holds one unit
  const uint32_t F = p.pair > 1 ? (uint32_t)p.pair : 1u;
  const uint32_t S = p.stages, slot = p.slot, box = p.box, SL = F * slot, N = p.n / F;
  // units of this CTA: unit(k) = lo + k * bstep
  uint32_t lo, mine, bstep;
  if (p.chunk) {
    const UnitRange R = unit_range(N, p.chunk);
    lo = R.lo;
    mine = R.end > lo ? R.end - lo : 0;
    bstep = 1;
  } else if (p.strided) {
    lo = blockIdx.x;
    bstep = gridDim.x;
    mine = lo < N ? (N - lo + bstep - 1) / bstep : 0;
  } else {
    lo = (uint32_t)((uint64_t)N * blockIdx.x / gridDim.x);
    mine = (uint32_t)((uint64_t)N * (blockIdx.x + 1) / gridDim.x) - lo;
    bstep = 1;
  }
  for (uint32_t s = 0; s < S; s++) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("prefetch.tensormap [%0];" ::"l"(&map) : "memory");
  if (p.dep) {
    // while the previous kernel drains: its first p.prefetch units into L2 (harmless if that kernel
    // still writes them -- the loads after the wait read L2, which holds the latest data)
    const uint32_t np = mine < p.prefetch ? mine : p.prefetch;
    for (uint32_t k = 0; k < np; k++) {
      int c[5];
      int64_t off;
      if constexpr (STORE) {
        tr_box(p, (lo + k * bstep) * F, c, off);
        bulk_prefetch(p.img + off, F * box);
      } else {
        for (uint32_t j = 0; j < F; j++) {
          tr_box(p, (lo + k * bstep) * F + j, c, off);
          tma_prefetch5(&map, c[0], c[1], c[2], c[3], c[4]);
        }
      }
    }
    pdl_wait();
  }
  pdl_launch_dependents();
  auto issue = [&](uint32_t k) {
    const uint32_t s = k % S;
    int c[5];
    int64_t off;
    mbar_expect_tx(&full[s], F * box);
    if constexpr (STORE) {
      tr_box(p, (lo + k * bstep) * F, c, off);
      bulk_load(sm + (size_t)s * SL, p.img + off, F * box, &full[s]);
    } else {
      for (uint32_t j = 0; j < F; j++) {
        tr_box(p, (lo + k * bstep) * F + j, c, off);
        tma_load5(sm + (size_t)s * SL + j * slot, &map, &full[s], c[0], c[1], c[2], c[3], c[4]);
      }
    }
  };
  for (uint32_t k = 0; k < mine && k < S; k++) issue(k);
  for (uint32_t k = 0; k < mine; k++) {
    const uint32_t s = k % S;
    int c[5];
    int64_t off;
    mbar_wait(&full[s], (k / S) & 1u);
    if constexpr (STORE) {
      for (uint32_t j = 0; j < F; j++) {
        tr_box(p, (lo + k * bstep) * F + j, c, off);
        tma_store5(&map, sm + (size_t)s * SL + j * slot, c[0], c[1], c[2], c[3], c[4]);
      }
    } else {
      tr_box(p, (lo + k * bstep) * F, c, off);
      for (int r = 0; r < p.reps.n; r++) bulk_store(p.img + off + p.reps.r[r], sm + (size_t)s * SL, F * box);
    }
    bulk_commit();
    // refill the slot of unit k - TR_LAG once its store has read shared memory
    if (k >= (uint32_t)TR_LAG && k - TR_LAG + S < mine) {
      bulk_wait_read<TR_LAG>();
      issue(k - TR_LAG + S);
    }
  }
  // shared memory must outlive the stores' reads; their global writes complete with the grid
  bulk_wait_read<0>();
}


// ------------------------------------------------------------------ K8 bulk form
// Non-nested digit systems whose shared innermost run is contiguous on both sides (R27): every run moves as
// boxes of p.box bytes by cp.async.bulk -- global -> shared ring -> global per destination replica, one
// issuing thread per CTA, no thread touches the data -- and the run's two addresses come from the two
// independent outer decodings.  Persistent strided grid; half a ring prefetched into L2 before the wait.
__device__ __forceinline__ int64_t k8b_digits(int n, const FastDiv *fd, const int64_t *st, uint32_t i) {
  int64_t off = 0;
#pragma unroll
  for (int k = K8_MAXD - 1; k >= 1; k--) {
    if (k >= n) continue;
    const uint32_t q = fdiv(fd[k], i);
    off += (int64_t)(i - q * fd[k].d) * st[k];
    i = q;
  }
  if (n > 0) off += (int64_t)i * st[0];
  return off;
}

constexpr int K8B_STAGES = 32;

__global__ void __launch_bounds__(32, 1) k8_bulk(const __grid_constant__ K8Params p, const uint8_t *__restrict__ src,
                                                 uint8_t *__restrict__ dst) {
  extern __shared__ __align__(128) uint8_t raw[];
  __shared__ __align__(8) uint64_t full[K8B_STAGES];
  if (threadIdx.x != 0) {
    pdl_launch_dependents();
    return;
  }
  uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 127) & ~(uintptr_t)127);
  const uint32_t S = p.stages, box = p.box, slot = (box + 127) & ~127u;
  const UnitRange R = unit_range(p.nboxes, p.chunk);
  const uint32_t lo = R.lo, bstep = R.step;
  const uint32_t mine = lo < R.end ? (R.end - lo + bstep - 1) / bstep : 0;
  auto addr = [&](uint32_t b, int64_t &so, int64_t &dof) {
    const uint32_t o = fdiv(p.per_run, b);
    const int64_t r = (int64_t)(b - o * p.per_run.d) * box;
    so = p.sbase + k8b_digits(p.na, p.afd, p.as, o) + r;
    dof = p.dbase + k8b_digits(p.nb, p.bfd, p.bs, o) + r;
  };
  for (uint32_t s = 0; s < S; s++) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (p.dep) {
    const uint32_t np = mine < p.prefetch ? mine : p.prefetch;
    for (uint32_t k = 0; k < np; k++) {
      int64_t so, dof;
      addr(lo + k * bstep, so, dof);
      bulk_prefetch(src + so, box);
    }
    pdl_wait();
  }
  pdl_launch_dependents();
  auto issue = [&](uint32_t k) {
    const uint32_t s = k % S;
    int64_t so, dof;
    addr(lo + k * bstep, so, dof);
    mbar_expect_tx(&full[s], box);
    bulk_load(sm + (size_t)s * slot, src + so, box, &full[s]);
  };
  for (uint32_t k = 0; k < mine && k < S; k++) issue(k);
  for (uint32_t k = 0; k < mine; k++) {
    const uint32_t s = k % S;
    int64_t so, dof;
    addr(lo + k * bstep, so, dof);
    mbar_wait(&full[s], (k / S) & 1u);
    for (int r = 0; r < p.nrep; r++) bulk_store(dst + dof + p.rep[r], sm + (size_t)s * slot, box);
    bulk_commit();
    if (k >= 2u && k - 2 + S < mine) {
      bulk_wait_read<2>();
      issue(k - 2 + S);
    }
  }
  bulk_wait_read<0>();
}

cudaError_t launch_k8_bulk(K8Params p, const void *src, void *dst, cudaStream_t st) {
  if (p.nboxes == 0) return cudaSuccess;
  static int optin = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
  }();
  static const int per_sm = [] {
    const char *e = getenv("AXE_K8_BULK_PER_SM");
    return (e && *e) ? std::max(1, std::min(8, atoi(e))) : 2;
  }();
  const uint32_t slot = (p.box + 127) & ~127u;
  // CTAs per SM: the knob, as long as each CTA keeps a ring of >= 4 boxes
  int ps = per_sm;
  while (ps > 1 && (size_t)(233472 / ps - 1024 - 2048 - 128) < 4 * (size_t)slot) ps--;
  const size_t budget = (size_t)std::min(optin, 233472 / ps - 1024) - 2048 - 128;
  p.stages = (uint32_t)std::min<size_t>(K8B_STAGES, budget / slot);
  if (p.chunk && p.chunk <= p.stages) p.stages = p.chunk;  // in-order schedule: every box of the CTA in flight
  else if (p.stages < 3) return cudaErrorInvalidValue;     // a slot is refilled two boxes after its store
  p.prefetch = std::max<uint32_t>(1, p.stages / 2);
  const size_t smem = (size_t)p.stages * slot + 128;
  const cudaError_t attr_err = smem_attr((const void *)k8_bulk, optin - 2048);
  if (attr_err != cudaSuccess) return attr_err;
  const unsigned blocks = p.chunk ? (p.nboxes + p.chunk - 1) / p.chunk
                                  : (unsigned)std::min<int64_t>(p.nboxes, (int64_t)num_sms() * ps);
  const cudaError_t e = launch_ex(k8_bulk, dim3(blocks), dim3(32), smem, st, p, (const uint8_t *)src, (uint8_t *)dst);
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  });
  return fn;
}

// dims/strides in bytes (byte elements); rank 5; swizzle_bytes in {0, 32, 64, 128}
int encode_tensor_map(void *out128, void *gaddr, const uint64_t dims[5], const uint64_t strides[4],
                      const uint32_t box[5], int swizzle_bytes) {
  PFN_encodeTiled fn = encode_fn();
  if (!fn) return -1;
  CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  cuuint64_t gd[5], gs[4];
  cuuint32_t bd[5], es[5];
  for (int i = 0; i < 5; i++) {
    gd[i] = dims[i];
    bd[i] = box[i];
    es[i] = 1;
  }
  for (int i = 0; i < 4; i++) gs[i] = strides[i];
  CUtensorMap m;  // 64-byte aligned
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, gaddr, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  memcpy(out128, &m, sizeof(m));
  return (int)r;
}

// CTAs per SM of the lowered schedule (AXE_TMA_REGION_PER_SM, default 2).  With the half-ring L2
// prefetch before the wait, 2 and 4 rings per SM tie on config 2 (10.04 / 10.03 us per dependent step,
// bench 6512-6572 / 6508 GB/s) and 2 wins at 16384^2 (177.0 vs 183.5 us); without the prefetch 4 rings
// were needed (11.63 us with 2), profiles/r02_lowered_prefetch_sweep.log)
int tma_region_per_sm() {
  static const int v = [] {
    const char *e = getenv("AXE_TMA_REGION_PER_SM");
    return (e && *e) ? std::max(1, std::min(8, atoi(e))) : 2;
  }();
  return v;
}

cudaError_t launch_tma_region(const void *map128, TrParams p, int store, cudaStream_t st) {
  if (p.n == 0) return cudaSuccess;
  const void *kern = store ? (const void *)k_tma_region<true> : (const void *)k_tma_region<false>;
  static int optin = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
  }();
  static int per_sm_bytes = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    return v;
  }();
  // CTAs per SM: the knob, lowered until every CTA's ring holds TR_LAG + 1 slots (a slot is refilled
  // TR_LAG boxes after its store, so fewer slots would wait on a box never issued)
  int per_sm = tma_region_per_sm();
  auto ring_of = [&](int ps) { return (size_t)std::min(optin, per_sm_bytes / ps - 1024) - 4096; };
  const size_t uslot = (size_t)p.slot * (p.pair > 1 ? p.pair : 1);  // a ring slot holds one unit (1, 2 or 4 boxes)
  while (per_sm > 1 && ring_of(per_sm) / uslot < (size_t)TR_LAG + 1) per_sm--;
  if (ring_of(per_sm) / uslot < (size_t)TR_LAG + 1) return cudaErrorInvalidValue;
  // ring: the CTA's share of the SM's shared memory (1 KiB per CTA is reserved by the system, the
  // static barriers and the 1 KiB alignment pad come off the top), at most TR_STAGES slots
  static const int static_bytes = [] {  // the barriers (+ alignment) of the kernel's static shared memory
    cudaFuncAttributes a0{}, a1{};
    cudaFuncGetAttributes(&a0, (const void *)k_tma_region<false>);
    cudaFuncGetAttributes(&a1, (const void *)k_tma_region<true>);
    return (int)std::max(a0.sharedSizeBytes, a1.sharedSizeBytes);
  }();
  const int max_dyn = std::min(optin, per_sm_bytes / per_sm - 1024) - static_bytes;
  const size_t budget = (size_t)max_dyn - 1024;
  static const size_t ring_cap = [] {  // AXE_TMA_REGION_STAGE_BYTES: cap the ring (A/B only)
    const char *e = getenv("AXE_TMA_REGION_STAGE_BYTES");
    return (size_t)((e && *e) ? std::max(1024, atoi(e)) : (1 << 30));
  }();
  const size_t ring = std::min(budget, ring_cap);
  p.stages = (uint32_t)std::min<size_t>(TR_STAGES, ring / uslot);
  if (p.chunk && p.chunk <= TR_STAGES && (size_t)p.chunk * uslot + 1024 + static_bytes <= (size_t)optin)
    p.stages = p.chunk;  // in-order schedule: the CTA's units all in flight at once, no refill
  else if (p.chunk)
    p.chunk = 0;         // (units too large for a chunk-deep ring: the persistent grid)
  if (!p.chunk && p.stages < (uint32_t)TR_LAG + 1) return cudaErrorInvalidValue;
  const size_t smem = (size_t)p.stages * uslot + 1024;
  const cudaError_t attr_err = smem_attr(kern, optin - static_bytes);  // (the largest any launch asks for)
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap m;
  memcpy(&m, map128, sizeof(m));
  const uint32_t units = p.n / (p.pair > 1 ? (uint32_t)p.pair : 1u);
  const unsigned blocks = p.chunk ? (units + p.chunk - 1) / p.chunk
                                  : (unsigned)std::min<int64_t>(units, (int64_t)num_sms() * per_sm);
  static const int strided = [] {  // AXE_TMA_REGION_STRIDED: box order per CTA (A/B)
    const char *e = getenv("AXE_TMA_REGION_STRIDED");
    return (e && *e) ? atoi(e) : 1;
  }();
  p.strided = strided;
  static const int prefetch = [] {  // AXE_TMA_REGION_PREFETCH: boxes per CTA prefetched before the wait
    const char *e = getenv("AXE_TMA_REGION_PREFETCH");
    return (e && *e) ? std::max(0, atoi(e)) : -1;  // -1: half a ring
  }();
  // half the ring: config 2 (6 slots) with 3 boxes 10.04 us per steady step and 11.22 us for one cold
  // launch, against 10.40 / 12.8 with the whole ring and 10.7 / 11.2 with one box (a prefetch costs the
  // TMA unit the same request generation as a load, which a cold launch pays up front)
  p.prefetch = prefetch < 0 ? std::max<uint32_t>(1, p.stages / 2) : (uint32_t)prefetch;
  cudaError_t e = store ? launch_ex(k_tma_region<true>, dim3(blocks), dim3(32), smem, st, m, p)
                        : launch_ex(k_tma_region<false>, dim3(blocks), dim3(32), smem, st, m, p);
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

size_t tma_smem_bytes(const TmaParams &p) { return (size_t)p.stages * p.slot_bytes + 1024; }

cudaError_t launch_tma(const void *map128, const TmaParams &p, unsigned blocks, const void *src, void *dst,
                       cudaStream_t st) {
  const cudaError_t attr_err = smem_attr((const void *)k1_tma, 200 * 1024);
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap m;
  memcpy(&m, map128, sizeof(m));
  // boxes per CTA prefetched into L2 before the wait: half the ring (identity 32 MiB 9.83 us per dependent
  // step vs 10.56 with the whole ring, equal from 128 MiB -- as for the lowered schedule, a prefetch costs
  // TMA request generation up front).  AXE_TMA_PREFETCH = n boxes (A/B; -1: the whole ring)
  static const int pf = [] {
    const char *e = getenv("AXE_TMA_PREFETCH");
    return (e && *e) ? atoi(e) : -2;
  }();
  TmaParams q = p;
  q.prefetch = pf == -2 ? (uint32_t)(q.stages + 1) / 2 : pf < 0 ? (uint32_t)q.stages : (uint32_t)std::min(pf, q.stages);
  cudaError_t e = launch_ex(k1_tma, dim3(blocks), dim3(32), tma_smem_bytes(q), st, m, q, (const uint8_t *)src,
                            (uint8_t *)dst);
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

}  // namespace axe
