// kernels_k2.cu -- K2: shared-memory staged tile permute (transposes, register
// layout permutes) for sm_100a.
//
// Per tile: every thread loads lj VS-byte vectors along the source-contiguous
// run (coalesced), stores them to smem in source order (XOR-swizzled on 16-byte
// chunks, swizzle chosen on the host by simulating bank conflicts), then
// gathers kg granules per VD-byte destination vector and stores it coalesced
// along the destination-contiguous run.  Offsets are host-built tables.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "kernels.cuh"
#include "launch.cuh"

namespace axe {

extern std::atomic<int64_t> g_launches;

template <int B>
struct K2Vec;
template <>
struct K2Vec<1> { using T = uint8_t; };
template <>
struct K2Vec<2> { using T = uint16_t; };
template <>
struct K2Vec<4> { using T = uint32_t; };
template <>
struct K2Vec<8> { using T = uint2; };
template <>
struct K2Vec<16> { using T = uint4; };

__device__ __forceinline__ uint32_t swz32(const Swz &s, uint32_t b) { return b ^ (((b >> s.shift) & s.mask) << s.base); }

__device__ __forceinline__ uint4 ldg16(const uint8_t *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int B>
__device__ __forceinline__ typename K2Vec<B>::T ldg(const uint8_t *p) {
  if constexpr (B == 16)
    return ldg16(p);
  else
    return __ldg(reinterpret_cast<const typename K2Vec<B>::T *>(p));
}

constexpr int K2_MAXLJ = 8;
// AXE_K2_MINB (dev A/B only): a minimum-CTAs-per-SM register cap.  Left undefined, the
// launch bounds carry no second argument -- an explicit 1 lets ptxas raise the register count.
#ifdef AXE_K2_MINB
#define AXE_K2_BOUNDS __launch_bounds__(K2_NT, AXE_K2_MINB)
#else
#define AXE_K2_BOUNDS __launch_bounds__(K2_NT)
#endif

// LJ > 0: loads per thread known at compile time (only the LJ vectors live in registers);
// LJ == 0: runtime p.lj <= K2_MAXLJ.
template <int VS, int VD, int GB, int LJ>
__global__ void AXE_K2_BOUNDS k2_tile(const __grid_constant__ K2Params p, const uint8_t *__restrict__ src,
                                                 uint8_t *__restrict__ dst) {
  extern __shared__ __align__(128) uint8_t sm[];
  using TS = typename K2Vec<VS>::T;
  using TD = typename K2Vec<VD>::T;
  using TG = typename K2Vec<GB>::T;
  constexpr int KG = VD / GB;
  const int t = threadIdx.x;
  // per-thread table entries: pinned in registers (an indexed constant load with 32 different
  // addresses per warp serialises; ptxas would otherwise re-load them inside the tile loop)
  int32_t al, as, ad;
  asm volatile("mov.b32 %0, %3;\n\tmov.b32 %1, %4;\n\tmov.b32 %2, %5;"
               : "=r"(al), "=r"(as), "=r"(ad)
               : "r"(p.A_l[t]), "r"(p.A_s[t]), "r"(p.A_d[t]));
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const UnitRange R = unit_range(p.ntiles, p.chunk);
  for (uint32_t tile = R.lo; tile < R.end; tile += R.step) {
    int64_t sb = p.sbase, db = p.dbase;
    {
      uint32_t i = tile;
#pragma unroll
      for (int k = K1_MAXD - 1; k >= 1; k--) {
        if (k >= p.nout) continue;
        uint32_t q = fdiv(p.ofd[k], i);
        uint32_t d = i - q * p.ofd[k].d;
        i = q;
        sb += (int64_t)d * p.oss[k];
        db += (int64_t)d * p.ods[k];
      }
      if (p.nout > 0) {
        sb += (int64_t)i * p.oss[0];
        db += (int64_t)i * p.ods[0];
      }
    }
    constexpr int NJ = LJ > 0 ? LJ : K2_MAXLJ;
    TS v[NJ];
#pragma unroll
    for (int j = 0; j < NJ; j++)
      if (LJ > 0 || j < p.lj) v[j] = ldg<VS>(src + swz(p.ssw, sb + p.B_l[j] + al));
    asm volatile("" ::: "memory");  // every load is in flight before the first shared store waits on one
#pragma unroll
    for (int j = 0; j < NJ; j++)
      if (LJ > 0 || j < p.lj) *reinterpret_cast<TS *>(sm + swz32(p.smsw, (uint32_t)((j * K2_NT + t) * VS))) = v[j];
    __syncthreads();
    for (int j = 0; j < p.sj; j++) {
      TD out;
      TG *o = reinterpret_cast<TG *>(&out);
      const uint32_t base = (uint32_t)(as + p.B_s[j]);
#pragma unroll
      for (int k = 0; k < KG; k++) o[k] = *reinterpret_cast<const TG *>(sm + swz32(p.smsw, base + p.C_s[k]));
      const int64_t d = db + p.B_d[j] + ad;
      for (int r = 0; r < p.nrep; r++) *reinterpret_cast<TD *>(dst + swz(p.dsw, d + p.rep[r])) = out;
    }
    __syncthreads();
  }
}

template <int VS, int VD, int GB, int LJ>
static cudaError_t k2_go_lj(const K2Params &p, unsigned blocks, size_t smem, const void *s, void *d, cudaStream_t st) {
  const cudaError_t e = smem_attr((const void *)k2_tile<VS, VD, GB, LJ>, 100 * 1024);
  if (e != cudaSuccess) return e;
  return launch_ex(k2_tile<VS, VD, GB, LJ>, dim3(blocks), dim3(K2_NT), smem, st, p, (const uint8_t *)s,
                   (uint8_t *)d);
}

template <int VS, int VD, int GB>
static cudaError_t k2_go(const K2Params &p, unsigned blocks, size_t smem, const void *s, void *d, cudaStream_t st) {
  static const bool lj_fixed = [] {
    const char *e = getenv("AXE_K2_LJ");
    return !(e && *e == '0');
  }();
  if constexpr (VS == 16 && VD == 16) {  // the transposes: fixed load counts
    if (!lj_fixed) return k2_go_lj<VS, VD, GB, 0>(p, blocks, smem, s, d, st);
    // measured (8192^2 transposes): fixed LJ = 4 (fp32, 16 KiB tiles) 121 -> 104 us; fixed LJ = 8
    // (bf16, 32 KiB tiles) 52 -> 58 us, so 8 keeps the runtime form
    if (p.lj == 4) return k2_go_lj<VS, VD, GB, 4>(p, blocks, smem, s, d, st);
  }
  return k2_go_lj<VS, VD, GB, 0>(p, blocks, smem, s, d, st);
}

template <int VS, int VD>
static cudaError_t k2_gb(int gb, const K2Params &p, unsigned blocks, size_t smem, const void *s, void *d,
                         cudaStream_t st) {
  switch (gb) {
    case 1: return k2_go<VS, VD, 1>(p, blocks, smem, s, d, st);
    case 2: return k2_go<VS, VD, 2>(p, blocks, smem, s, d, st);
    case 4: return k2_go<VS, VD, 4>(p, blocks, smem, s, d, st);
    case 8:
      if constexpr (VD >= 8) return k2_go<VS, VD, 8>(p, blocks, smem, s, d, st);
      break;
    case 16:
      if constexpr (VD >= 16) return k2_go<VS, VD, 16>(p, blocks, smem, s, d, st);
      break;
  }
  return cudaErrorInvalidValue;
}

template <int VS>
static cudaError_t k2_vd(int vd, int gb, const K2Params &p, unsigned blocks, size_t smem, const void *s, void *d,
                         cudaStream_t st) {
  switch (vd) {
    case 4: return k2_gb<VS, 4>(gb, p, blocks, smem, s, d, st);
    case 8: return k2_gb<VS, 8>(gb, p, blocks, smem, s, d, st);
    case 16: return k2_gb<VS, 16>(gb, p, blocks, smem, s, d, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_k2(const K2Params &p, int vs, int vd, int gb, unsigned blocks, const void *src, void *dst,
                      cudaStream_t st) {
  size_t smem = p.tile_bytes;
  cudaError_t e;
  switch (vs) {
    case 4: e = k2_vd<4>(vd, gb, p, blocks, smem, src, dst, st); break;
    case 8: e = k2_vd<8>(vd, gb, p, blocks, smem, src, dst, st); break;
    case 16: e = k2_vd<16>(vd, gb, p, blocks, smem, src, dst, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

}  // namespace axe
