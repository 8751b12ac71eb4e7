// kernels_reduce.cu -- K4: layout-driven reduction over the leading logical
// dimension (reading R24 of DESIGN.md):
//
//   dst(y) = sum_{k<K} src(k * E_D(dst) + y),   K = E_D(src) / E_D(dst)
//
// P:399-403 (the DTensor reduce-scatter whose (4,64,64) input "sums over 0")
// and P:628 ("invokes the sum operator").  Floating point summands are added
// in fp32 (fp64 for f64) in k order and rounded once to the element type
// (round to nearest even); integers add modulo 2^bits.
//
//   k4_reduce  : one thread per output vector (<= 16 bytes shared by both
//                layouts' contiguous run); the K summand offsets come from a
//                table (K <= 256) and are loaded 8 at a time before they are
//                added in order, so every thread keeps 8 loads in flight.
//   k4_generic : per element, both layouts evaluated with 64-bit div/mod (the
//                fallback for non-affine compositions / non-nested digits).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "kernels.cuh"
#include "launch.cuh"
#include "tma_ops.cuh"

namespace axe {

extern std::atomic<int64_t> g_launches;
int num_sms();

namespace {

template <int B>
struct RawT;
template <>
struct RawT<2> { using T = uint16_t; };
template <>
struct RawT<4> { using T = uint32_t; };
template <>
struct RawT<8> { using T = uint2; };
template <>
struct RawT<16> { using T = uint4; };

template <int B>
__device__ __forceinline__ typename RawT<B>::T ld_raw(const uint8_t *p) {
  if constexpr (B == 16) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
  } else {
    return __ldg(reinterpret_cast<const typename RawT<B>::T *>(p));
  }
}

// storage bits S, accumulator A, conversions and the (non-fused) add
template <int DT>
struct Op;
template <>
struct Op<DT_F32> {
  using S = uint32_t;
  using A = float;
  static __device__ __forceinline__ A in(S b) { return __uint_as_float(b); }
  static __device__ __forceinline__ A add(A a, A v) { return __fadd_rn(a, v); }
  static __device__ __forceinline__ S out(A a) { return __float_as_uint(a); }
};
template <>
struct Op<DT_F64> {
  using S = uint64_t;
  using A = double;
  static __device__ __forceinline__ A in(S b) { return __longlong_as_double((long long)b); }
  static __device__ __forceinline__ A add(A a, A v) { return __dadd_rn(a, v); }
  static __device__ __forceinline__ S out(A a) { return (S)__double_as_longlong(a); }
};
template <>
struct Op<DT_F16> {
  using S = uint16_t;
  using A = float;
  static __device__ __forceinline__ A in(S b) { return __half2float(__ushort_as_half(b)); }
  static __device__ __forceinline__ A add(A a, A v) { return __fadd_rn(a, v); }
  static __device__ __forceinline__ S out(A a) { return __half_as_ushort(__float2half_rn(a)); }
};
template <>
struct Op<DT_BF16> {
  using S = uint16_t;
  using A = float;
  static __device__ __forceinline__ A in(S b) { return __bfloat162float(__ushort_as_bfloat16(b)); }
  static __device__ __forceinline__ A add(A a, A v) { return __fadd_rn(a, v); }
  static __device__ __forceinline__ S out(A a) { return __bfloat16_as_ushort(__float2bfloat16_rn(a)); }
};
template <>
struct Op<DT_I32> {
  using S = uint32_t;
  using A = uint32_t;
  static __device__ __forceinline__ A in(S b) { return b; }
  static __device__ __forceinline__ A add(A a, A v) { return a + v; }
  static __device__ __forceinline__ S out(A a) { return a; }
};
template <>
struct Op<DT_I64> {
  using S = uint64_t;
  using A = uint64_t;
  static __device__ __forceinline__ A in(S b) { return b; }
  static __device__ __forceinline__ A add(A a, A v) { return a + v; }
  static __device__ __forceinline__ S out(A a) { return a; }
};

constexpr int K4_THREADS = 256;
constexpr int K4_BATCH = 8;  // summands loaded before they are added (loads in flight per thread)
// ptxas keeps k4_reduce at 32 registers (8 CTAs per SM) and interleaves each load with the adds of the
// previous one; __launch_bounds__(256, 4) gets all 8 loads issued back to back at <= 64 registers but
// measured slower on a B200 (bf16 K = 2 161.4 us vs 130.7, K = 16 84.5 vs 82.4, f32 K = 8 90.0 vs 88.4):
// resident threads matter more than loads per thread here

// PEER: summand k lives at (uint8_t *)ptrs.p[k] + swz(so + koff[k]) (a peer's buffer mapped into this
// process, read over NVLink), else at src + swz(so + koff[k]).
template <int DT, int V, bool PEER>
__device__ __forceinline__ void k4_body(const K4Params &p, const uint64_t *kp, const uint8_t *__restrict__ src,
                                        uint8_t *__restrict__ dst) {
  using O = Op<DT>;
  using S = typename O::S;
  using A = typename O::A;
  constexpr int VB = V * (int)sizeof(S);
  using R = typename RawT<VB>::T;
  const UnitRange U = unit_range((p.total + blockDim.x - 1) / blockDim.x, p.chunk);
  if (p.dep) {
    // while the previous kernel drains: this thread's first summands into L2 (R28)
    const uint32_t i0 = U.lo * blockDim.x + threadIdx.x;
    if (!PEER && p.nk > 0 && i0 < p.total) {
      int64_t so = p.sbase;
      uint32_t rem = i0;
      for (int k = p.nd - 1; k >= 0; k--) {
        const uint32_t q = fdiv(p.fd[k], rem);
        so += (int64_t)(rem - q * p.fd[k].d) * p.ss[k];
        rem = q;
      }
      for (int k = 0; k < p.nk; k++) prefetch_l2(src + swz(p.ssw, so + p.koff[k]));
    }
    pdl_wait();
  }
  pdl_launch_dependents();
  for (uint32_t t = U.lo; t < U.end; t += U.step) {
    const uint32_t i = t * blockDim.x + threadIdx.x;
    if (i >= p.total) break;
    int64_t so = p.sbase, dof = p.dbase;
    uint32_t rem = i;
    for (int k = p.nd - 1; k >= 0; k--) {
      const uint32_t q = fdiv(p.fd[k], rem);
      const uint32_t d = rem - q * p.fd[k].d;
      rem = q;
      so += (int64_t)d * p.ss[k];
      dof += (int64_t)d * p.ds[k];
    }
    A acc[V];
#pragma unroll
    for (int v = 0; v < V; v++) acc[v] = A(0);
    auto accumulate = [&](const R &raw) {
      alignas(16) S e[V];
      *reinterpret_cast<R *>(e) = raw;
#pragma unroll
      for (int v = 0; v < V; v++) acc[v] = O::add(acc[v], O::in(e[v]));
    };
    if (p.nk > 0) {
      int k = 0;
      for (; k + K4_BATCH <= p.nk; k += K4_BATCH) {
        R raw[K4_BATCH];
#pragma unroll
        for (int b = 0; b < K4_BATCH; b++)
          raw[b] = ld_raw<VB>((PEER ? (const uint8_t *)kp[k + b] : src) + swz(p.ssw, so + p.koff[k + b]));
#pragma unroll
        for (int b = 0; b < K4_BATCH; b++) accumulate(raw[b]);  // k order
      }
      for (; k < p.nk; k++)
        accumulate(ld_raw<VB>((PEER ? (const uint8_t *)kp[k] : src) + swz(p.ssw, so + p.koff[k])));
    } else {
      for (uint32_t kk = 0; kk < p.ktotal; kk++) {
        int64_t off = 0;
        uint32_t r2 = kk;
        for (int t = p.nkd - 1; t >= 0; t--) {
          const uint32_t q = fdiv(p.kfd[t], r2);
          off += (int64_t)(r2 - q * p.kfd[t].d) * p.kss[t];
          r2 = q;
        }
        accumulate(ld_raw<VB>(src + swz(p.ssw, so + off)));
      }
    }
    alignas(16) S o[V];
#pragma unroll
    for (int v = 0; v < V; v++) o[v] = O::out(acc[v]);
    const R out = *reinterpret_cast<const R *>(o);
    for (int r = 0; r < p.nrep; r++) {
      uint8_t *q = dst + swz(p.dsw, dof + p.rep[r]);
      if constexpr (VB == 16) {
        if (p.stcs) {
          asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(q), "r"(out.x), "r"(out.y), "r"(out.z),
                       "r"(out.w)
                       : "memory");
          continue;
        }
      }
      *reinterpret_cast<R *>(q) = out;
    }
  }
}

template <int DT, int V>
__global__ void __launch_bounds__(K4_THREADS) k4_reduce(const __grid_constant__ K4Params p,
                                                        const uint8_t *__restrict__ src, uint8_t *__restrict__ dst) {
  k4_body<DT, V, false>(p, nullptr, src, dst);
}

template <int DT, int V>
__global__ void __launch_bounds__(K4_THREADS) k4_reduce_peer(const __grid_constant__ K4Params p,
                                                             const __grid_constant__ K4Ptrs ptrs,
                                                             uint8_t *__restrict__ dst) {
  k4_body<DT, V, true>(p, ptrs.p, nullptr, dst);
}

// ---- generic form: the plain layout + storage evaluation per element
__device__ __forceinline__ int64_t g_storage_index(const K0Side &S, const int64_t *c) {
  int64_t idx = 0;
  for (int k = 0; k < S.nsd; k++) {
    const int64_t v = S.sax[k] >= 0 ? c[S.sax[k]] : 0;
    idx = idx * S.sext[k] + (v / S.sdiv[k]) % S.sext[k];
  }
  return idx;
}

__device__ __forceinline__ void g_fd(const K0Side &S, int64_t x, int64_t *c) {
  for (int i = 0; i < S.nax; i++) c[i] = S.off[i];
  for (int i = S.nD - 1; i >= 0; i--) {
    const int64_t d = x % S.e[i];
    x /= S.e[i];
    c[S.ax[i]] += d * S.s[i];
  }
}

template <int DT>
__global__ void __launch_bounds__(256) k4_generic(const __grid_constant__ K4GParams p, const uint8_t *__restrict__ src,
                                                  uint8_t *__restrict__ dst) {
  using O = Op<DT>;
  using S = typename O::S;
  using A = typename O::A;
  constexpr int ES = (int)sizeof(S);
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; y < (uint64_t)p.Y; y += stride) {
    int64_t c[K0_MAXAX];
    A acc = A(0);
    for (int64_t k = 0; k < p.K; k++) {
      g_fd(p.src, k * p.Y + (int64_t)y, c);  // source representative f_D(x) + O (reading R4)
      const int64_t sb = swz(p.src.sw, g_storage_index(p.src, c) * ES);
      acc = O::add(acc, O::in(*reinterpret_cast<const S *>(src + sb)));
    }
    const S v = O::out(acc);
    int64_t b[K0_MAXAX];
    g_fd(p.dst, (int64_t)y, b);
    for (int64_t r = 0; r < p.ER; r++) {
      for (int i = 0; i < p.dst.nax; i++) c[i] = b[i];
      int64_t rr = r;
      for (int t = p.dst.nR - 1; t >= 0; t--) {
        const int64_t d = rr % p.dst.re[t];
        rr /= p.dst.re[t];
        c[p.dst.rax[t]] += d * p.dst.rs[t];
      }
      *reinterpret_cast<S *>(dst + swz(p.dst.sw, g_storage_index(p.dst, c) * ES)) = v;
    }
  }
}

template <int DT>
cudaError_t launch_k4_dt(const K4Params &p, int vb, unsigned blocks, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  constexpr int ES = (int)sizeof(typename Op<DT>::S);
  const dim3 b(K4_THREADS);
  // persistent: one wave; in-order schedule (p.chunk): every block of K4_THREADS vectors covered
  auto one_wave = [&](const void *kern, int threads, size_t smem, unsigned want) -> unsigned {
    if (p.chunk) return (unsigned)(((p.total + K4_THREADS - 1) / K4_THREADS + p.chunk - 1) / p.chunk);
    return axe::one_wave(kern, threads, smem, want);
  };
  switch (vb / ES) {
    case 1: return launch_ex(k4_reduce<DT, 1>, dim3(one_wave((const void *)k4_reduce<DT, 1>, K4_THREADS, 0, blocks)), b, 0, st, p, s, d);
    case 2:
      if constexpr (2 * ES <= 16) return launch_ex(k4_reduce<DT, 2>, dim3(one_wave((const void *)k4_reduce<DT, 2>, K4_THREADS, 0, blocks)), b, 0, st, p, s, d);
      break;
    case 4:
      if constexpr (4 * ES <= 16) return launch_ex(k4_reduce<DT, 4>, dim3(one_wave((const void *)k4_reduce<DT, 4>, K4_THREADS, 0, blocks)), b, 0, st, p, s, d);
      break;
    case 8:
      if constexpr (8 * ES <= 16) return launch_ex(k4_reduce<DT, 8>, dim3(one_wave((const void *)k4_reduce<DT, 8>, K4_THREADS, 0, blocks)), b, 0, st, p, s, d);
      break;
  }
  return cudaErrorInvalidValue;
}

// NVLS form (the paper's GEMM + reduce-scatter "dispatch to multimem.ld_reduce on B200"):
// every output vector is ONE multimem.ld_reduce on the multicast address of the partials -- the
// NVSwitch reads the vector from every rank's buffer and returns the sum.  16-byte vectors.
template <int DT>
__device__ __forceinline__ uint4 mc_ld_reduce(const uint8_t *a) {
  uint4 r;
  if constexpr (DT == DT_F32)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(a)
                 : "memory");
  else if constexpr (DT == DT_BF16)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(a)
                 : "memory");
  else
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(a)
                 : "memory");
  return r;
}

template <int DT>
__global__ void __launch_bounds__(K4_THREADS) k4_multimem(const __grid_constant__ K4Params p,
                                                          const uint8_t *__restrict__ mc, uint8_t *__restrict__ dst) {
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.total; i += stride) {
    int64_t so = p.sbase + p.koff[0], dof = p.dbase;
    uint32_t rem = i;
    for (int k = p.nd - 1; k >= 0; k--) {
      const uint32_t q = fdiv(p.fd[k], rem);
      const uint32_t d = rem - q * p.fd[k].d;
      rem = q;
      so += (int64_t)d * p.ss[k];
      dof += (int64_t)d * p.ds[k];
    }
    const uint4 v = mc_ld_reduce<DT>(mc + swz(p.ssw, so));
    *reinterpret_cast<uint4 *>(dst + swz(p.dsw, dof)) = v;
  }
}

template <int DT>
cudaError_t launch_k4p_dt(const K4Params &p, const K4Ptrs &q, int vb, unsigned blocks, uint8_t *d, cudaStream_t st) {
  constexpr int ES = (int)sizeof(typename Op<DT>::S);
  const dim3 g(blocks), b(K4_THREADS);
  switch (vb / ES) {
    case 1: return launch_ex(k4_reduce_peer<DT, 1>, g, b, 0, st, p, q, d);
    case 2:
      if constexpr (2 * ES <= 16) return launch_ex(k4_reduce_peer<DT, 2>, g, b, 0, st, p, q, d);
      break;
    case 4:
      if constexpr (4 * ES <= 16) return launch_ex(k4_reduce_peer<DT, 4>, g, b, 0, st, p, q, d);
      break;
    case 8:
      if constexpr (8 * ES <= 16) return launch_ex(k4_reduce_peer<DT, 8>, g, b, 0, st, p, q, d);
      break;
  }
  return cudaErrorInvalidValue;
}


}  // namespace

cudaError_t launch_k4_peer(const K4Params &p, const K4Ptrs &q, int dtype, int vb, unsigned blocks, void *dst,
                           cudaStream_t st) {
  uint8_t *d = (uint8_t *)dst;
  cudaError_t e;
  switch (dtype) {
    case DT_F32: e = launch_k4p_dt<DT_F32>(p, q, vb, blocks, d, st); break;
    case DT_F64: e = launch_k4p_dt<DT_F64>(p, q, vb, blocks, d, st); break;
    case DT_F16: e = launch_k4p_dt<DT_F16>(p, q, vb, blocks, d, st); break;
    case DT_BF16: e = launch_k4p_dt<DT_BF16>(p, q, vb, blocks, d, st); break;
    case DT_I32: e = launch_k4p_dt<DT_I32>(p, q, vb, blocks, d, st); break;
    case DT_I64: e = launch_k4p_dt<DT_I64>(p, q, vb, blocks, d, st); break;
    default: return cudaErrorInvalidValue;
  }
  g_launches++;
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_k4_multimem(const K4Params &p, int dtype, unsigned blocks, const void *mc, void *dst,
                               cudaStream_t st) {
  const uint8_t *m = (const uint8_t *)mc;
  uint8_t *d = (uint8_t *)dst;
  const dim3 g(blocks), b(K4_THREADS);
  cudaError_t e;
  switch (dtype) {
    case DT_F32: e = launch_ex(k4_multimem<DT_F32>, g, b, 0, st, p, m, d); break;
    case DT_BF16: e = launch_ex(k4_multimem<DT_BF16>, g, b, 0, st, p, m, d); break;
    case DT_F16: e = launch_ex(k4_multimem<DT_F16>, g, b, 0, st, p, m, d); break;
    default: return cudaErrorInvalidValue;
  }
  g_launches++;
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_k4(const K4Params &p, int dtype, int vb, unsigned blocks, const void *src, void *dst,
                      cudaStream_t st) {
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  cudaError_t e;
  switch (dtype) {
    case DT_F32: e = launch_k4_dt<DT_F32>(p, vb, blocks, s, d, st); break;
    case DT_F64: e = launch_k4_dt<DT_F64>(p, vb, blocks, s, d, st); break;
    case DT_F16: e = launch_k4_dt<DT_F16>(p, vb, blocks, s, d, st); break;
    case DT_BF16: e = launch_k4_dt<DT_BF16>(p, vb, blocks, s, d, st); break;
    case DT_I32: e = launch_k4_dt<DT_I32>(p, vb, blocks, s, d, st); break;
    case DT_I64: e = launch_k4_dt<DT_I64>(p, vb, blocks, s, d, st); break;
    default: return cudaErrorInvalidValue;
  }
  g_launches++;
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_k4g(const K4GParams &p, int dtype, const void *src, void *dst, cudaStream_t st) {
  int64_t blocks = (p.Y + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  const dim3 g((unsigned)blocks), b(256);
  cudaError_t e;
  switch (dtype) {
    case DT_F32: e = launch_ex(k4_generic<DT_F32>, g, b, 0, st, p, s, d); break;
    case DT_F64: e = launch_ex(k4_generic<DT_F64>, g, b, 0, st, p, s, d); break;
    case DT_F16: e = launch_ex(k4_generic<DT_F16>, g, b, 0, st, p, s, d); break;
    case DT_BF16: e = launch_ex(k4_generic<DT_BF16>, g, b, 0, st, p, s, d); break;
    case DT_I32: e = launch_ex(k4_generic<DT_I32>, g, b, 0, st, p, s, d); break;
    case DT_I64: e = launch_ex(k4_generic<DT_I64>, g, b, 0, st, p, s, d); break;
    default: return cudaErrorInvalidValue;
  }
  g_launches++;
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace axe
