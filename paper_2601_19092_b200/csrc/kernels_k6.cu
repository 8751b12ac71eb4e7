// kernels_k6.cu -- K6: granule transpose across lane groups with warp shuffles (sm_100a).
//
// Config 3a (mma.sync C fragments -> tcgen05 32x32b rows) moves 4-byte pairs of
// bf16: the 16-byte destination chunk of a row takes the same 4-byte granule
// from 4 consecutive lanes' 16-byte source chunks.  Four source vectors, taken
// as a 4 x 4 matrix of granules, are exactly the transpose of four destination
// vectors.  A group of 4 threads loads them (one LDG.128 each, a group reads 64
// contiguous bytes), transposes in two butterfly stages (lane ^ 2 swaps the
// off-diagonal 2 x 2 blocks, lane ^ 1 transposes each block; 4 SHFL per
// thread), and each thread stores one STG.128.  The data never touches shared
// memory, which is what limited the smem-staged K2 on this copy (SM-bound).
#include <cuda_runtime.h>

#include <atomic>

#include "kernels.cuh"
#include "launch.cuh"

namespace axe {

extern std::atomic<int64_t> g_launches;

namespace {

constexpr int K6_THREADS = 256;

__device__ __forceinline__ uint4 ldg128(const uint8_t *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 4 x 4 transpose of 32-bit words across lanes t = 4 g + j (j = t mod 4): afterwards lane j holds
// word j of lanes 0..3 in order.
__device__ __forceinline__ uint4 transpose4(uint4 w, int j) {
  // stage A: exchange the off-diagonal 2 x 2 blocks with lane ^ 2
  const bool hi = j & 2;
  uint32_t a0 = hi ? w.x : w.z, a1 = hi ? w.y : w.w;
  uint32_t b0 = __shfl_xor_sync(0xffffffffu, a0, 2), b1 = __shfl_xor_sync(0xffffffffu, a1, 2);
  if (hi) {
    w.x = b0;
    w.y = b1;
  } else {
    w.z = b0;
    w.w = b1;
  }
  // stage B: transpose every 2 x 2 block with lane ^ 1
  const bool odd = j & 1;
  a0 = odd ? w.x : w.y;
  a1 = odd ? w.z : w.w;
  b0 = __shfl_xor_sync(0xffffffffu, a0, 1);
  b1 = __shfl_xor_sync(0xffffffffu, a1, 1);
  if (odd) {
    w.x = b0;
    w.z = b1;
  } else {
    w.y = b0;
    w.w = b1;
  }
  return w;
}

// 2 x 2 transpose of 64-bit granules with lane ^ 1
__device__ __forceinline__ uint4 transpose2(uint4 w, int j) {
  const bool odd = j & 1;
  uint32_t a0 = odd ? w.x : w.z, a1 = odd ? w.y : w.w;
  uint32_t b0 = __shfl_xor_sync(0xffffffffu, a0, 1), b1 = __shfl_xor_sync(0xffffffffu, a1, 1);
  if (odd) {
    w.x = b0;
    w.y = b1;
  } else {
    w.z = b0;
    w.w = b1;
  }
  return w;
}

__device__ __forceinline__ void k6_decode(int n, const FastDiv *fd, const int64_t *a, const int64_t *b, uint32_t i,
                                          int64_t &oa, int64_t &ob) {
#pragma unroll
  for (int k = K1_MAXD - 1; k >= 1; k--) {
    if (k >= n) continue;
    const uint32_t q = fdiv(fd[k], i);
    const uint32_t d = i - q * fd[k].d;
    i = q;
    oa += (int64_t)d * a[k];
    ob += (int64_t)d * b[k];
  }
  if (n > 0) {
    oa += (int64_t)i * a[0];
    ob += (int64_t)i * b[0];
  }
}

template <int N, bool SWZ>
__global__ void __launch_bounds__(K6_THREADS) k6_transpose(const __grid_constant__ K6Params p,
                                                           const uint8_t *__restrict__ src, uint8_t *__restrict__ dst) {
  const int j = threadIdx.x % N;
  constexpr int GPB = K6_THREADS / N;  // groups per pass of the block
  // per-thread offsets of its K6_U groups inside a tile (computed once)
  int64_t so[K6_U], dof[K6_U];
#pragma unroll
  for (int u = 0; u < K6_U; u++) {
    so[u] = j * p.sstep;
    dof[u] = p.dpos[j];
    k6_decode(p.nin, p.ifd, p.iss, p.ids, threadIdx.x / N + u * GPB, so[u], dof[u]);
  }
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const UnitRange R = unit_range(p.ntiles, p.chunk);
  for (uint32_t t = R.lo; t < R.end; t += R.step) {
    int64_t sb = p.sbase, db = p.dbase;
    k6_decode(p.nout, p.ofd, p.oss, p.ods, t, sb, db);
    uint4 w[K6_U];
#pragma unroll
    for (int u = 0; u < K6_U; u++) w[u] = ldg128(src + (SWZ ? swz(p.ssw, sb + so[u]) : sb + so[u]));
#pragma unroll
    for (int u = 0; u < K6_U; u++) {
      const uint4 v = N == 4 ? transpose4(w[u], j) : transpose2(w[u], j);
      if (!SWZ && p.nrep == 1) {
        *reinterpret_cast<uint4 *>(dst + db + dof[u] + p.rep[0]) = v;
      } else {
        for (int r = 0; r < p.nrep; r++)
          *reinterpret_cast<uint4 *>(dst + (SWZ ? swz(p.dsw, db + dof[u] + p.rep[r]) : db + dof[u] + p.rep[r])) = v;
      }
    }
  }
}

}  // namespace

cudaError_t launch_k6(const K6Params &p, unsigned blocks, const void *src, void *dst, cudaStream_t st) {
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  const bool sw = p.ssw.mask || p.dsw.mask;  // (unswizzled: no swizzle arithmetic per vector)
  cudaError_t e = p.n == 4 ? (sw ? launch_ex(k6_transpose<4, true>, dim3(blocks), dim3(K6_THREADS), 0, st, p, s, d)
                                 : launch_ex(k6_transpose<4, false>, dim3(blocks), dim3(K6_THREADS), 0, st, p, s, d))
                           : (sw ? launch_ex(k6_transpose<2, true>, dim3(blocks), dim3(K6_THREADS), 0, st, p, s, d)
                                 : launch_ex(k6_transpose<2, false>, dim3(blocks), dim3(K6_THREADS), 0, st, p, s, d));
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

}  // namespace axe
