// kernels.cu -- libaxe device code for sm_100a.
//
//   K0 generic : one thread per logical element x; evaluates f_D^src(x) + O,
//                f_L^dst(x) and both storage maps per element (always
//                applicable; the fallback for non-affine storage compositions
//                and non-nested digit systems).
//   K1 vector  : joint-digit copy: one thread per 16-byte (or
//                narrower) vector shared by both layouts' contiguous run; one
//                load, one swizzled store per destination replica.
//
// "address = base pointer + memory components of the layout"; the
// copy operator's schedule is chosen from the two layouts.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>

#include "kernels.cuh"
#include "launch.cuh"

namespace axe {

std::atomic<int64_t> g_launches{0};

// ------------------------------------------------------------------ helpers
template <int B>
struct VecT;
template <>
struct VecT<1> { using T = uint8_t; };
template <>
struct VecT<2> { using T = uint16_t; };
template <>
struct VecT<4> { using T = uint32_t; };
template <>
struct VecT<8> { using T = uint2; };
template <>
struct VecT<16> { using T = uint4; };

template <int B>
__device__ __forceinline__ typename VecT<B>::T ld_stream(const uint8_t *p) {
  using T = typename VecT<B>::T;
  if constexpr (B == 16) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
  } else {
    return __ldg(reinterpret_cast<const T *>(p));
  }
}

template <int B>
__device__ __forceinline__ void st_vec(uint8_t *p, const typename VecT<B>::T &v) {
  *reinterpret_cast<typename VecT<B>::T *>(p) = v;
}

// ------------------------------------------------------------------ K0
__device__ __forceinline__ int64_t k0_storage_index(const K0Side &S, const int64_t *c) {
  int64_t idx = 0;
  for (int k = 0; k < S.nsd; k++) {
    int64_t v = S.sax[k] >= 0 ? c[S.sax[k]] : 0;
    idx = idx * S.sext[k] + (v / S.sdiv[k]) % S.sext[k];
  }
  return idx;
}

template <int ES>
__global__ void __launch_bounds__(256) k0_generic(const __grid_constant__ K0Params p, const uint8_t *__restrict__ src,
                                                  uint8_t *__restrict__ dst) {
  using T = typename VecT<ES>::T;
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < (uint64_t)p.ED; x += stride) {
    int64_t c[K0_MAXAX];
    // source representative f_D(x) + O (reading R4)
    for (int i = 0; i < p.src.nax; i++) c[i] = p.src.off[i];
    int64_t rem = (int64_t)x;
    for (int i = p.src.nD - 1; i >= 0; i--) {
      int64_t d = rem % p.src.e[i];
      rem /= p.src.e[i];
      c[p.src.ax[i]] += d * p.src.s[i];
    }
    int64_t sb = swz(p.src.sw, k0_storage_index(p.src, c) * ES);
    T v = *reinterpret_cast<const T *>(src + sb);
    // destination: every replica of f_L(x)
    int64_t b[K0_MAXAX];
    for (int i = 0; i < p.dst.nax; i++) b[i] = p.dst.off[i];
    rem = (int64_t)x;
    for (int i = p.dst.nD - 1; i >= 0; i--) {
      int64_t d = rem % p.dst.e[i];
      rem /= p.dst.e[i];
      b[p.dst.ax[i]] += d * p.dst.s[i];
    }
    for (int64_t r = 0; r < p.ER; r++) {
      for (int i = 0; i < p.dst.nax; i++) c[i] = b[i];
      int64_t rr = r;
      for (int t = p.dst.nR - 1; t >= 0; t--) {
        int64_t d = rr % p.dst.re[t];
        rr /= p.dst.re[t];
        c[p.dst.rax[t]] += d * p.dst.rs[t];
      }
      int64_t db = swz(p.dst.sw, k0_storage_index(p.dst, c) * ES);
      *reinterpret_cast<T *>(dst + db) = v;
    }
  }
}

// ------------------------------------------------------------------ K1
constexpr int K1_THREADS = 256;
// AXE_K1_MINB (dev A/B only): a minimum-CTAs-per-SM register cap.  Left undefined, the
// launch bounds carry no second argument -- an explicit 1 lets ptxas raise the register count.
#ifdef AXE_K1_MINB
#define AXE_K1_BOUNDS __launch_bounds__(K1_THREADS, AXE_K1_MINB)
#else
#define AXE_K1_BOUNDS __launch_bounds__(K1_THREADS)
#endif
#ifndef AXE_K1_U_BIG  // vectors per thread per tile, 8- and 16-byte vectors
#define AXE_K1_U_BIG 4
#endif
#ifndef AXE_K1_U_SMALL  // vectors per thread per tile, <= 4-byte vectors
#define AXE_K1_U_SMALL 8
#endif

// ND > 0: digit count known at compile time; ND == 0: runtime p.nd (<= K1_MAXD)
template <int ND>
__device__ __forceinline__ void k1_decode(const K1Params &p, uint32_t i, int64_t &so, int64_t &dof) {
  so = p.sbase;
  dof = p.dbase;
  constexpr int TOP = ND > 0 ? ND : K1_MAXD;
#pragma unroll
  for (int k = TOP - 1; k >= 1; k--) {
    if (ND == 0 && k >= p.nd) continue;
    uint32_t q = fdiv(p.fd[k], i);
    uint32_t d = i - q * p.fd[k].d;
    i = q;
    so += (int64_t)d * p.ss[k];
    dof += (int64_t)d * p.ds[k];
  }
  so += (int64_t)i * p.ss[0];
  dof += (int64_t)i * p.ds[0];
}

template <int ND, int VB, int U>
__global__ void __launch_bounds__(K1_THREADS) k1_vector(const __grid_constant__ K1Params p,
                                                        const uint8_t *__restrict__ src, uint8_t *__restrict__ dst) {
  using T = typename VecT<VB>::T;
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const uint32_t total = p.total;
  const UnitRange R = unit_range((total + K1_THREADS * U - 1) / (K1_THREADS * U), p.chunk);
  for (uint32_t ut = R.lo; ut < R.end; ut += R.step) {
    const uint32_t base = ut * (K1_THREADS * U) + threadIdx.x;
    T v[U];
    int64_t dof[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      uint32_t i = base + u * K1_THREADS;
      if (i < total) {
        int64_t so;
        k1_decode<ND>(p, i, so, dof[u]);
        v[u] = ld_stream<VB>(src + swz(p.ssw, so));
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      uint32_t i = base + u * K1_THREADS;
      if (i < total) {
        for (int r = 0; r < p.nrep; r++) st_vec<VB>(dst + swz(p.dsw, dof[u] + p.rep[r]), v[u]);
      }
    }
  }
}

// Tiled K1: the per-thread part of the digit decode (and the swizzle, when the
// tile bases are whole swizzle blocks) is done once; each tile then costs one
// uniform base decode, U loads and U * nrep stores per thread.
__device__ __forceinline__ void decode_digits(int n, const FastDiv *fd, const int64_t *a, const int64_t *b, uint32_t i,
                                              int64_t &oa, int64_t &ob) {
#pragma unroll
  for (int k = K1_MAXD - 1; k >= 1; k--) {
    if (k >= n) continue;
    uint32_t q = fdiv(fd[k], i);
    uint32_t d = i - q * fd[k].d;
    i = q;
    oa += (int64_t)d * a[k];
    ob += (int64_t)d * b[k];
  }
  if (n > 0) {
    oa += (int64_t)i * a[0];
    ob += (int64_t)i * b[0];
  }
}

template <int VB, int U>
__global__ void AXE_K1_BOUNDS k1_tiled(const __grid_constant__ K1Params p, const uint8_t *__restrict__ src,
                                                       uint8_t *__restrict__ dst) {
  using T = typename VecT<VB>::T;
  int64_t so[U], dof[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    so[u] = 0;
    dof[u] = 0;
    decode_digits(p.nin, p.ifd, p.iss, p.ids, threadIdx.x + u * K1_THREADS, so[u], dof[u]);
    if (p.pre_s) so[u] = swz(p.ssw, so[u]);
    if (p.pre_d) dof[u] = swz(p.dsw, dof[u]);
  }
  const UnitRange R = unit_range(p.ntiles, p.chunk);
  if (p.dep) {  // the per-thread decode above, and the first tile's source lines into L2 (R28), overlap
                // the previous kernel's tail
    if (R.lo < R.end) {
      int64_t sb = p.sbase, db = p.dbase;
      decode_digits(p.nout, p.ofd, p.oss, p.ods, R.lo, sb, db);
#pragma unroll
      for (int u = 0; u < U; u++) prefetch_l2(src + (p.pre_s ? sb + so[u] : swz(p.ssw, sb + so[u])));
    }
    pdl_wait();
  }
  pdl_launch_dependents();
  for (uint32_t t = R.lo; t < R.end; t += R.step) {
    int64_t sb = p.sbase, db = p.dbase;
    decode_digits(p.nout, p.ofd, p.oss, p.ods, t, sb, db);
    T v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = ld_stream<VB>(src + (p.pre_s ? sb + so[u] : swz(p.ssw, sb + so[u])));
    for (int r = 0; r < p.nrep; r++) {
      const int64_t b = db + p.rep[r];
#pragma unroll
      for (int u = 0; u < U; u++) st_vec<VB>(dst + (p.pre_d ? b + dof[u] : swz(p.dsw, b + dof[u])), v[u]);
    }
  }
}

// ------------------------------------------------------------------ launchers
static int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      g_num_sms = n;
    else
      g_num_sms = 148;
  }
  return g_num_sms;
}

cudaError_t launch_k0(const K0Params &p, const void *src, void *dst, cudaStream_t st) {
  int64_t blocks = (p.ED + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  cudaError_t e = cudaSuccess;
  switch (p.es) {
    case 1: e = launch_ex(k0_generic<1>, dim3((unsigned)blocks), dim3(256), 0, st, p, s, d); break;
    case 2: e = launch_ex(k0_generic<2>, dim3((unsigned)blocks), dim3(256), 0, st, p, s, d); break;
    case 4: e = launch_ex(k0_generic<4>, dim3((unsigned)blocks), dim3(256), 0, st, p, s, d); break;
    case 8: e = launch_ex(k0_generic<8>, dim3((unsigned)blocks), dim3(256), 0, st, p, s, d); break;
    case 16: e = launch_ex(k0_generic<16>, dim3((unsigned)blocks), dim3(256), 0, st, p, s, d); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

template <int ND, int VB>
static cudaError_t k1_launch_nd(const K1Params &p, unsigned blocks, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  constexpr int U = VB >= 8 ? AXE_K1_U_BIG : AXE_K1_U_SMALL;
  return launch_ex(k1_vector<ND, VB, U>, dim3(blocks), dim3(K1_THREADS), 0, st, p, s, d);
}


// ------------------------------------------------------------------ K8 dual decoding
template <int N>
__device__ __forceinline__ int64_t k8_digits(int n, const FastDiv *fd, const int64_t *st, uint32_t i) {
  int64_t off = 0;
#pragma unroll
  for (int k = N - 1; k >= 1; k--) {
    if (k >= n) continue;
    const uint32_t q = fdiv(fd[k], i);
    off += (int64_t)(i - q * fd[k].d) * st[k];
    i = q;
  }
  if (n > 0) off += (int64_t)i * st[0];
  return off;
}

template <int VB, int U, bool SWZ>
__global__ void __launch_bounds__(K1_THREADS) k8_dual(const __grid_constant__ K8Params p, const uint8_t *__restrict__ src,
                                                      uint8_t *__restrict__ dst) {
  auto ssw = [&](int64_t b) { return SWZ ? swz(p.ssw, b) : b; };  // (SWZ = false: no swizzle on either side)
  auto dsw = [&](int64_t b) { return SWZ ? swz(p.dsw, b) : b; };
  using T = typename VecT<VB>::T;
  if (p.dep && !p.chunked) pdl_wait();
  if (p.chunked) {
    // item = (o, c): vectors [c * CH, c * CH + CH) of block o, CH = K1_THREADS * U; the outer offsets are
    // uniform over the item (two decodings per item), the inner offset is w times the run's stride
    constexpr uint32_t CH = K1_THREADS * U;
    const uint32_t vin = p.vin.d;
    const UnitRange R = unit_range(p.nitems, p.chunk);
    if (p.dep && R.lo < R.end) {  // the first item's vectors into L2 before the wait (R28)
      const uint32_t o = fdiv(p.nchunks, R.lo);
      const uint32_t c = R.lo - o * p.nchunks.d;
      const int64_t so = p.sbase + k8_digits<K8_MAXD>(p.na, p.afd, p.as, o);
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t w = c * CH + u * K1_THREADS + threadIdx.x;
        if (w < vin && (w * VB) % 128 < VB) prefetch_l2(src + ssw(so + (int64_t)w * p.iss[0]));
      }
    }
    if (p.dep) pdl_wait();
    pdl_launch_dependents();
    for (uint32_t it = R.lo; it < R.end; it += R.step) {
      const uint32_t o = fdiv(p.nchunks, it);
      const uint32_t c = it - o * p.nchunks.d;
      const int64_t so = p.sbase + k8_digits<K8_MAXD>(p.na, p.afd, p.as, o);
      const int64_t d = p.dbase + k8_digits<K8_MAXD>(p.nb, p.bfd, p.bs, o);
      T v[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t w = c * CH + u * K1_THREADS + threadIdx.x;
        if (w < vin) v[u] = ld_stream<VB>(src + ssw(so + (int64_t)w * p.iss[0]));
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t w = c * CH + u * K1_THREADS + threadIdx.x;
        if (w < vin)
          for (int r = 0; r < p.nrep; r++) st_vec<VB>(dst + dsw(d + (int64_t)w * p.ids[0] + p.rep[r]), v[u]);
      }
    }
    return;
  }
  pdl_launch_dependents();
  const uint32_t total = p.total;
  const UnitRange R = unit_range((total + K1_THREADS * U - 1) / (K1_THREADS * U), p.chunk);
  for (uint32_t ut = R.lo; ut < R.end; ut += R.step) {
    const uint32_t base = ut * (K1_THREADS * U) + threadIdx.x;
    T v[U];
    int64_t dof[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t i = base + u * K1_THREADS;
      if (i < total) {
        const uint32_t o = fdiv(p.vin, i);
        uint32_t w = i - o * p.vin.d;
        int64_t so = p.sbase, d = p.dbase;
#pragma unroll
        for (int k = K1_MAXD - 1; k >= 1; k--) {
          if (k >= p.nin) continue;
          const uint32_t q = fdiv(p.ifd[k], w);
          const int64_t dg = (int64_t)(w - q * p.ifd[k].d);
          w = q;
          so += dg * p.iss[k];
          d += dg * p.ids[k];
        }
        if (p.nin > 0) {
          so += (int64_t)w * p.iss[0];
          d += (int64_t)w * p.ids[0];
        }
        so += k8_digits<K8_MAXD>(p.na, p.afd, p.as, o);
        d += k8_digits<K8_MAXD>(p.nb, p.bfd, p.bs, o);
        v[u] = ld_stream<VB>(src + ssw(so));
        dof[u] = d;
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t i = base + u * K1_THREADS;
      if (i < total)
        for (int r = 0; r < p.nrep; r++) st_vec<VB>(dst + dsw(dof[u] + p.rep[r]), v[u]);
    }
  }
}


// K8 odometer form: gcd-1 digit systems (no run is shared by the two sides).  Lane l of a warp takes
// x = x0 + l, x0 + l + 32, ... over a chunk of 32 K8_ODO_J elements; per side it keeps the innermost digit
// r = x mod E and the byte offset of the outer digits of q = x / E, and when r wraps it decodes q again
// (fast divisions) -- so consecutive lanes move consecutive x (coalesced wherever a side's innermost
// digit is contiguous), and an element costs a compare and two adds per side instead of two full
// decodings.  8 loads in flight per lane before their stores.
template <int ES, bool SWZ>
__global__ void __launch_bounds__(K1_THREADS) k8_odo(const __grid_constant__ K8Params p, const uint8_t *__restrict__ src,
                                                     uint8_t *__restrict__ dst) {
  using T = typename VecT<ES>::T;
  constexpr int U = 8;
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const FastDiv EA = p.afd[p.na - 1], EB = p.bfd[p.nb - 1];
  const int64_t sA = p.as[p.na - 1], sB = p.bs[p.nb - 1];
  // units of K1_THREADS / 32 consecutive chunks, warp w taking chunk w of each of its CTA's units
  constexpr uint32_t WPB = K1_THREADS / 32;
  const UnitRange R = unit_range((p.nchunk + WPB - 1) / WPB, p.chunk);
  for (uint32_t c = R.lo * WPB + (threadIdx.x >> 5), ce = min(p.nchunk, R.end * WPB); c < ce; c += R.step * WPB) {
    uint32_t x = c * (uint32_t)(K8_ODO_J * 32) + lane;
    const uint32_t xend = min(p.total, (c + 1) * (uint32_t)(K8_ODO_J * 32));
    uint32_t qa = fdiv(EA, x), ra = x - qa * EA.d;
    uint32_t qb = fdiv(EB, x), rb = x - qb * EB.d;
    int64_t oa = p.sbase + k8_digits<K8_MAXD>(p.na - 1, p.afd, p.as, qa);
    int64_t ob = p.dbase + k8_digits<K8_MAXD>(p.nb - 1, p.bfd, p.bs, qb);
    for (int j0 = 0; j0 < K8_ODO_J; j0 += U) {
      T v[U];
      int64_t d[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (x < xend) {
          const int64_t so = oa + (int64_t)ra * sA;
          v[u] = ld_stream<ES>(src + (SWZ ? swz(p.ssw, so) : so));
          d[u] = ob + (int64_t)rb * sB;
        }
        x += 32;
        ra += 32;
        rb += 32;
        if (ra >= EA.d) {  // the innermost source digit wrapped: decode the outer ones again
          qa = fdiv(EA, x);
          ra = x - qa * EA.d;
          oa = p.sbase + k8_digits<K8_MAXD>(p.na - 1, p.afd, p.as, qa);
        }
        if (rb >= EB.d) {
          qb = fdiv(EB, x);
          rb = x - qb * EB.d;
          ob = p.dbase + k8_digits<K8_MAXD>(p.nb - 1, p.bfd, p.bs, qb);
        }
      }
      if (!SWZ && p.nrep == 1) {  // (the common case: no swizzle, one destination -- no replica loop)
        const int64_t r0 = p.rep[0];
#pragma unroll
        for (int u = 0; u < U; u++)
          if (x - (uint32_t)(U - u) * 32 < xend) st_vec<ES>(dst + d[u] + r0, v[u]);
      } else {
#pragma unroll
        for (int u = 0; u < U; u++) {
          const uint32_t xu = x - (uint32_t)(U - u) * 32;
          if (xu < xend)
            for (int r = 0; r < p.nrep; r++) st_vec<ES>(dst + (SWZ ? swz(p.dsw, d[u] + p.rep[r]) : d[u] + p.rep[r]), v[u]);
        }
      }
    }
  }
}

template <int VB>
static cudaError_t k8_launch(const K8Params &p, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  constexpr int U = VB >= 8 ? 4 : 8;
  const bool sw = p.ssw.mask || p.dsw.mask;
  const void *kern = sw ? (const void *)k8_dual<VB, U, true> : (const void *)k8_dual<VB, U, false>;
  const unsigned want = p.chunked ? p.nitems
                                  : (unsigned)((p.total + (uint64_t)K1_THREADS * U - 1) / ((uint64_t)K1_THREADS * U));
  const unsigned blocks = p.chunk ? (want + p.chunk - 1) / p.chunk : one_wave(kern, K1_THREADS, 0, std::max(1u, want));
  return sw ? launch_ex(k8_dual<VB, U, true>, dim3(blocks), dim3(K1_THREADS), 0, st, p, s, d)
            : launch_ex(k8_dual<VB, U, false>, dim3(blocks), dim3(K1_THREADS), 0, st, p, s, d);
}

int k8_chunk(int vb) { return K1_THREADS * (vb >= 8 ? 4 : 8); }

cudaError_t launch_k8(const K8Params &p, int vb, const void *src, void *dst, cudaStream_t st) {
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  cudaError_t e;
  if (p.odo) {
    auto go = [&](auto kern) {
      const unsigned want = (p.nchunk + K1_THREADS / 32 - 1) / (K1_THREADS / 32);
      const unsigned blocks =
          p.chunk ? (want + p.chunk - 1) / p.chunk : one_wave((const void *)kern, K1_THREADS, 0, std::max(1u, want));
      return launch_ex(kern, dim3(blocks), dim3(K1_THREADS), 0, st, p, s, d);
    };
    const bool sw = p.ssw.mask || p.dsw.mask;
    switch (vb) {
      case 1: e = sw ? go(k8_odo<1, true>) : go(k8_odo<1, false>); break;
      case 2: e = sw ? go(k8_odo<2, true>) : go(k8_odo<2, false>); break;
      case 4: e = sw ? go(k8_odo<4, true>) : go(k8_odo<4, false>); break;
      case 8: e = sw ? go(k8_odo<8, true>) : go(k8_odo<8, false>); break;
      case 16: e = sw ? go(k8_odo<16, true>) : go(k8_odo<16, false>); break;
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    g_launches++;
    return cudaGetLastError();
  }
  switch (vb) {
    case 1: e = k8_launch<1>(p, s, d, st); break;
    case 2: e = k8_launch<2>(p, s, d, st); break;
    case 4: e = k8_launch<4>(p, s, d, st); break;
    case 8: e = k8_launch<8>(p, s, d, st); break;
    case 16: e = k8_launch<16>(p, s, d, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

template <int VB>
static cudaError_t k1_launch_vb(const K1Params &p, unsigned blocks, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  switch (p.nd) {
    case 1: return k1_launch_nd<1, VB>(p, blocks, s, d, st);
    case 2: return k1_launch_nd<2, VB>(p, blocks, s, d, st);
    case 3: return k1_launch_nd<3, VB>(p, blocks, s, d, st);
    case 4: return k1_launch_nd<4, VB>(p, blocks, s, d, st);
    case 5: return k1_launch_nd<5, VB>(p, blocks, s, d, st);
    case 6: return k1_launch_nd<6, VB>(p, blocks, s, d, st);
    case 7: return k1_launch_nd<7, VB>(p, blocks, s, d, st);
    case 8: return k1_launch_nd<8, VB>(p, blocks, s, d, st);
    default:
      if (p.nd > K1_MAXD) return cudaErrorInvalidValue;
      return k1_launch_nd<0, VB>(p, blocks, s, d, st);
  }
}

int k1_unroll(int vb) { return vb >= 8 ? AXE_K1_U_BIG : AXE_K1_U_SMALL; }

template <int VB>
static cudaError_t k1_tiled_launch(const K1Params &p, unsigned blocks, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  constexpr int U = VB >= 8 ? AXE_K1_U_BIG : AXE_K1_U_SMALL;
  return launch_ex(k1_tiled<VB, U>, dim3(blocks), dim3(K1_THREADS), 0, st, p, s, d);
}

cudaError_t launch_k1(const K1Params &p, int vb, unsigned blocks, const void *src, void *dst, cudaStream_t st) {
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  cudaError_t e = cudaSuccess;
  if (p.tile_v > 0) {
    switch (vb) {
      case 1: e = k1_tiled_launch<1>(p, blocks, s, d, st); break;
      case 2: e = k1_tiled_launch<2>(p, blocks, s, d, st); break;
      case 4: e = k1_tiled_launch<4>(p, blocks, s, d, st); break;
      case 8: e = k1_tiled_launch<8>(p, blocks, s, d, st); break;
      case 16: e = k1_tiled_launch<16>(p, blocks, s, d, st); break;
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (vb) {
      case 1: e = k1_launch_vb<1>(p, blocks, s, d, st); break;
      case 2: e = k1_launch_vb<2>(p, blocks, s, d, st); break;
      case 4: e = k1_launch_vb<4>(p, blocks, s, d, st); break;
      case 8: e = k1_launch_vb<8>(p, blocks, s, d, st); break;
      case 16: e = k1_launch_vb<16>(p, blocks, s, d, st); break;
      default: return cudaErrorInvalidValue;
    }
  }
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

}  // namespace axe
