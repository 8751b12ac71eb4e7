// kernels_k9.cu -- K9: ragged 2-D transposes (sm_100a).
//
// K7 needs whole 16-byte vectors along both pitches and whole tiles; shapes like 4095 x 4097 bf16 (rows
// that start at every 2-byte alignment) or 8000 x 8000 leave it out, and K1 then moves 2-byte vectors
// whose stores scatter one per 32-byte sector (0.13 of peak).  K9 is the classic shared-memory transpose
// with element-granular accesses: a tile of TB = 64 rows (b, destination-contiguous) x TA = 128 / es
// elements (a, source-contiguous) is loaded along the source rows (consecutive lanes, consecutive
// elements: coalesced whatever the alignment), written to shared memory with each row padded to an odd
// number of 4-byte words (the column reads that follow hit 32 distinct banks), then stored along the
// destination rows (consecutive lanes, consecutive b).  Edges are predicated; batch digits index tiles.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>

#include "kernels.cuh"
#include "launch.cuh"

namespace axe {

extern std::atomic<int64_t> g_launches;
int num_sms();

namespace {

template <int B>
struct ElemT;
template <>
struct ElemT<1> { using T = uint8_t; };
template <>
struct ElemT<2> { using T = uint16_t; };
template <>
struct ElemT<4> { using T = uint32_t; };
template <>
struct ElemT<8> { using T = uint2; };
template <>
struct ElemT<16> { using T = uint4; };

constexpr int K9_THREADS = 256;
#ifndef AXE_K9_MINB
#define AXE_K9_MINB 6
#endif

constexpr int K9_TB = 64;

template <int ES>
struct K9Geom {
  static constexpr int TA = 128 / ES;                        // elements per tile row (128 bytes)
  static constexpr int PAD = ES <= 4 ? 4 / ES : 1;           // row = 132 bytes = 33 words for es <= 4
  static constexpr int LOADS = TA * K9_TB / K9_THREADS;      // elements per thread per tile
};

template <int ES, bool SWZ>
__global__ void __launch_bounds__(K9_THREADS) k9_ragged(const __grid_constant__ K9Params p,
                                                        const uint8_t *__restrict__ src, uint8_t *__restrict__ dst) {
  using T = typename ElemT<ES>::T;
  using G = K9Geom<ES>;
  constexpr int TA = G::TA, TB = K9_TB, L = G::LOADS;
  constexpr int RS = K9_THREADS / TA;  // load phase: rows per pass (a thread keeps its column ia)
  constexpr int CS = K9_THREADS / TB;  // store phase: columns per pass (a thread keeps its row jb)
  __shared__ T tile[TB][TA + G::PAD];
  const int t = threadIdx.x;
  const int ia_l = t % TA, jb_l0 = t / TA;  // load phase: column ia_l, rows jb_l0 + u RS
  const int jb_s = t % TB, ia_s0 = t / TB;  // store phase: row jb_s, columns ia_s0 + u CS
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  // tile geometry: batch digits outermost, then a-tiles, b-tiles fastest (consecutive CTAs extend the
  // same destination rows)
  struct Tile {
    int64_t sbo, dbo, a0, b0;
    bool full;
  };
  auto tile_of = [&](uint32_t tt) {
    uint32_t r = tt;
    uint32_t q = fdiv(p.fb, r);
    const uint32_t tb = r - q * p.fb.d;
    r = q;
    q = fdiv(p.fa, r);
    const uint32_t ta = r - q * p.fa.d;
    r = q;
    Tile x;
    x.sbo = p.sbase;
    x.dbo = p.dbase;
    for (int k = p.nd - 1; k >= 0; k--) {
      uint32_t d;
      if (k > 0) {
        const uint32_t qq = fdiv(p.fd[k], r);
        d = r - qq * p.fd[k].d;
        r = qq;
      } else {
        d = r;
      }
      x.sbo += (int64_t)d * p.ss[k];
      x.dbo += (int64_t)d * p.ds[k];
    }
    x.a0 = (int64_t)ta * TA;
    x.b0 = (int64_t)tb * TB;
    x.full = x.a0 + TA <= p.ea && x.b0 + TB <= p.eb;  // an interior tile: no predicates
    return x;
  };
  // load: this thread's column ia_l of rows jb_l0 + u RS; one 64-bit add per element
  T v[L];
  auto load = [&](const Tile &x) {
    const int64_t sl = x.sbo + (x.b0 + jb_l0) * p.s_b + (x.a0 + ia_l) * ES, sstep = RS * p.s_b;
#pragma unroll
    for (int u = 0; u < L; u++) {
      const int64_t off = sl + u * sstep;
      if (x.full || (x.a0 + ia_l < p.ea && x.b0 + jb_l0 + u * RS < p.eb))
        v[u] = *reinterpret_cast<const T *>(src + (SWZ ? swz(p.ssw, off) : off));
    }
  };
  const UnitRange R = unit_range(p.ntiles, p.chunk);
  uint32_t tt = R.lo;
  Tile cur;
  if (tt < R.end) {
    cur = tile_of(tt);
    load(cur);
  }
  for (; tt < R.end; tt += R.step) {
#pragma unroll
    for (int u = 0; u < L; u++) tile[jb_l0 + u * RS][ia_l] = v[u];
    __syncthreads();
    // the next tile's loads go out before this tile's stores (register double buffering)
    const uint32_t nt = tt + R.step;
    Tile nxt;
    if (nt < R.end) {
      nxt = tile_of(nt);
      load(nxt);
    }
    // store: this thread's row jb_s of columns ia_s0 + u CS (destination rows: consecutive lanes,
    // consecutive b)
    const int64_t dl = cur.dbo + (cur.a0 + ia_s0) * p.d_a + (cur.b0 + jb_s) * ES, dstep = CS * p.d_a;
#pragma unroll
    for (int u = 0; u < L; u++) {
      if (cur.full || (cur.a0 + ia_s0 + u * CS < p.ea && cur.b0 + jb_s < p.eb)) {
        const T x = tile[jb_s][ia_s0 + u * CS];
        const int64_t off = dl + u * dstep;
        for (int rr = 0; rr < p.nrep; rr++)
          *reinterpret_cast<T *>(dst + (SWZ ? swz(p.dsw, off + p.rep[rr]) : off + p.rep[rr])) = x;
      }
    }
    __syncthreads();
    cur = nxt;
  }
}


// Vector-load form: a tile row's 128 bytes start at any alignment m (0..15) inside their first 16-byte
// chunk; the NCH = 9 chunks covering it are loaded as LDG.128 into a row buffer (144 bytes + pad), and the
// store phase reads element ia of row jb at byte m_jb + ia es of that buffer.  Loads per tile: 64 x 9
// chunks over 256 threads (3 per thread) instead of 8192 / es element loads.
constexpr int K9V_NCH = 9;
// row buffer stride: 148 bytes = 37 words (odd: column reads spread over the banks) for es <= 4; 152 for
// 8-byte elements (every element 8-byte aligned in the buffer)
template <int ES>
__host__ __device__ constexpr int k9v_row() { return ES == 8 ? 152 : 148; }

template <int ES, bool SWZ>
__device__ __forceinline__ void k9_vec_body(const K9Params &p, const uint8_t *__restrict__ src,
                                            uint8_t *__restrict__ dst) {
  using T = typename ElemT<ES>::T;
  constexpr int TA = 128 / ES, TB = K9_TB;
  constexpr int CS = K9_THREADS / TB;          // store phase: columns per pass
  constexpr int L = TA * TB / K9_THREADS;      // elements per thread per tile (store phase)
  constexpr int SLOTS = TB * K9V_NCH;          // chunk loads per tile
  constexpr int LV = (SLOTS + K9_THREADS - 1) / K9_THREADS;
  constexpr int K9V_ROW = k9v_row<ES>();
  __shared__ __align__(16) uint8_t rows[TB * K9V_ROW];  // (148 / 152-byte rows: 4-byte aligned)
  __shared__ int moff[TB];
  const int t = threadIdx.x;
  const int jb_s = t % TB, ia_s0 = t / TB;
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const UnitRange R = unit_range(p.ntiles, p.chunk);
  for (uint32_t tt = R.lo; tt < R.end; tt += R.step) {
    uint32_t r = tt;
    uint32_t q = fdiv(p.fb, r);
    const uint32_t tb = r - q * p.fb.d;
    r = q;
    q = fdiv(p.fa, r);
    const uint32_t ta = r - q * p.fa.d;
    r = q;
    int64_t sbo = p.sbase, dbo = p.dbase;
    for (int k = p.nd - 1; k >= 0; k--) {
      uint32_t d;
      if (k > 0) {
        const uint32_t qq = fdiv(p.fd[k], r);
        d = r - qq * p.fd[k].d;
        r = qq;
      } else {
        d = r;
      }
      sbo += (int64_t)d * p.ss[k];
      dbo += (int64_t)d * p.ds[k];
    }
    const int64_t a0 = (int64_t)ta * TA, b0 = (int64_t)tb * TB;
    // load: chunk slot s = (row, chunk)
    uint4 cv[LV];
#pragma unroll
    for (int u = 0; u < LV; u++) {
      const int s = t + u * K9_THREADS;
      const int jb = s / K9V_NCH, ch = s % K9V_NCH;
      if (s < SLOTS && b0 + jb < p.eb) {
        const int64_t g = sbo + (b0 + jb) * p.s_b + a0 * ES;
        const int64_t c = (g & ~int64_t(15)) + ch * 16;
        if (ch == 0) moff[jb] = (int)(g & 15);
        if (c < p.src_limit) cv[u] = *reinterpret_cast<const uint4 *>(src + (SWZ ? swz(p.ssw, c) : c));
      }
    }
#pragma unroll
    for (int u = 0; u < LV; u++) {  // (row strides are multiples of 4 bytes, not 16: four 32-bit stores)
      const int s = t + u * K9_THREADS;
      if (s < SLOTS) {
        uint32_t *w = reinterpret_cast<uint32_t *>(rows + (s / K9V_NCH) * K9V_ROW + (s % K9V_NCH) * 16);
        w[0] = cv[u].x;
        w[1] = cv[u].y;
        w[2] = cv[u].z;
        w[3] = cv[u].w;
      }
    }
    __syncthreads();
    if constexpr (ES == 1) {
      // 1-byte elements: each destination row segment (64 elements from b0) leaves as 4-byte words
      // -- word w of the segment covers its bytes [4w - m, 4w - m + 4), m = the segment's start address mod
      // 4 -- assembled from 4 / es row buffers; a word only partly inside the segment (its first and last)
      // goes out element by element.  Consecutive lanes take consecutive words of a row.  (u8 8191 x 8193:
      // 100.8 us vs 107.7 with byte stores; for bf16 the same form lost, 36.5 vs 31.2, so 2-byte
      // elements keep the element stores below)
      constexpr int EPW = 4 / ES;               // elements per word
      constexpr int WPR = TB * ES / 4 + 1;      // words per row segment (one more when misaligned)
      constexpr int TASKS = TA * WPR;
      const int nbv = (int)(p.eb - b0 < TB ? p.eb - b0 : TB), nav = (int)(p.ea - a0 < TA ? p.ea - a0 : TA);
      for (int task = t; task < TASKS; task += K9_THREADS) {
        const int ia = task / WPR, w = task - ia * WPR;
        if (ia >= nav) break;
        const int64_t rowb = dbo + (a0 + ia) * p.d_a + b0 * ES;
        for (int rr = 0; rr < p.nrep; rr++) {
          const int64_t A = rowb + p.rep[rr];
          const int m = (int)(((uintptr_t)dst + (uintptr_t)A) & 3u);
          const int o0 = 4 * w - m;             // segment byte offset of the word's first byte
          if (o0 >= TB * ES || o0 + 4 <= 0) continue;
          const int j0 = o0 >= 0 ? o0 / ES : -((-o0 + ES - 1) / ES);
          if (o0 >= 0 && j0 + EPW <= nbv) {
            uint32_t word = 0;
#pragma unroll
            for (int k = 0; k < EPW; k++) {
              const int j = j0 + k;
              const uint32_t x = *reinterpret_cast<const T *>(rows + j * K9V_ROW + moff[j] + ia * ES);
              word |= x << (8 * ES * k);
            }
            const int64_t off = A + o0;
            *reinterpret_cast<uint32_t *>(dst + (SWZ ? swz(p.dsw, off) : off)) = word;
          } else {
            for (int k = 0; k < EPW; k++) {
              const int j = j0 + k;
              if (j < 0 || j >= nbv) continue;
              const T x = *reinterpret_cast<const T *>(rows + j * K9V_ROW + moff[j] + ia * ES);
              const int64_t off = A + (int64_t)j * ES;
              *reinterpret_cast<T *>(dst + (SWZ ? swz(p.dsw, off) : off)) = x;
            }
          }
        }
      }
      __syncthreads();
      continue;
    }
    // store: this thread's row jb_s of columns ia_s0 + u CS (consecutive lanes, consecutive b; element
    // stores -- assembling 16-byte destination chunks from 16 / es row buffers measured slower: 44.9 us vs
    // 31.1 on 4095 x 4097 bf16)
    if (b0 + jb_s < p.eb) {
      const uint8_t *rb = rows + jb_s * K9V_ROW + moff[jb_s];
      const int64_t dl = dbo + (a0 + ia_s0) * p.d_a + (b0 + jb_s) * ES, dstep = CS * p.d_a;
      if (!SWZ && p.nrep == 1 && a0 + TA <= p.ea) {
        // the common case -- unswizzled, one destination, a tile of whole columns: one shared load and
        // one store per element, the address a running pointer
        uint8_t *q = dst + dl + p.rep[0];
#pragma unroll
        for (int u = 0; u < L; u++) {
          *reinterpret_cast<T *>(q) = *reinterpret_cast<const T *>(rb + (ia_s0 + u * CS) * ES);
          q += dstep;
        }
      } else {
#pragma unroll
        for (int u = 0; u < L; u++) {
          const int ia = ia_s0 + u * CS;
          if (a0 + ia < p.ea) {
            // (m_jb is a multiple of es -- elements are es-aligned in the 16-byte aligned buffer -- and so
            // is the row stride, so this read is es-aligned)
            const T x = *reinterpret_cast<const T *>(rb + ia * ES);
            const int64_t off = dl + u * dstep;
            for (int rr = 0; rr < p.nrep; rr++)
              *reinterpret_cast<T *>(dst + (SWZ ? swz(p.dsw, off + p.rep[rr]) : off + p.rep[rr])) = x;
          }
        }
      }
    }
    __syncthreads();
  }
}

// register budget: 2-8-byte elements capped for 6 CTAs per SM (4095 x 4097 bf16 18.1 us vs 30.1 with the
// compiler's choice under a 1-CTA bound; fp32 30.0 vs 53.6); the 1-byte word form keeps the compiler's
// default (91.0 us; capped at 2-5 CTAs 99-117)
template <int ES, bool SWZ>
__global__ void __launch_bounds__(K9_THREADS, AXE_K9_MINB) k9_vec(const __grid_constant__ K9Params p,
                                                                 const uint8_t *__restrict__ src,
                                                                 uint8_t *__restrict__ dst) {
  k9_vec_body<ES, SWZ>(p, src, dst);
}
template <bool SWZ>
__global__ void __launch_bounds__(K9_THREADS) k9_vec_u8(const __grid_constant__ K9Params p,
                                                        const uint8_t *__restrict__ src, uint8_t *__restrict__ dst) {
  k9_vec_body<1, SWZ>(p, src, dst);
}

template <int ES>
cudaError_t go(const K9Params &p, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  const bool sw = p.ssw.mask || p.dsw.mask;
  if (p.vec && ES == 1) {
    const void *kern = sw ? (const void *)k9_vec_u8<true> : (const void *)k9_vec_u8<false>;
    const unsigned blocks = p.chunk ? (p.ntiles + p.chunk - 1) / p.chunk : one_wave(kern, K9_THREADS, 0, std::max(1u, p.ntiles));
    return sw ? launch_ex(k9_vec_u8<true>, dim3(blocks), dim3(K9_THREADS), 0, st, p, s, d)
              : launch_ex(k9_vec_u8<false>, dim3(blocks), dim3(K9_THREADS), 0, st, p, s, d);
  }
  if (p.vec && ES <= 8) {
    const void *kern = sw ? (const void *)k9_vec<ES, true> : (const void *)k9_vec<ES, false>;
    const unsigned blocks = p.chunk ? (p.ntiles + p.chunk - 1) / p.chunk : one_wave(kern, K9_THREADS, 0, std::max(1u, p.ntiles));
    return sw ? launch_ex(k9_vec<ES, true>, dim3(blocks), dim3(K9_THREADS), 0, st, p, s, d)
              : launch_ex(k9_vec<ES, false>, dim3(blocks), dim3(K9_THREADS), 0, st, p, s, d);
  }
  const void *kern = sw ? (const void *)k9_ragged<ES, true> : (const void *)k9_ragged<ES, false>;
  const unsigned blocks = p.chunk ? (p.ntiles + p.chunk - 1) / p.chunk : one_wave(kern, K9_THREADS, 0, std::max(1u, p.ntiles));
  return sw ? launch_ex(k9_ragged<ES, true>, dim3(blocks), dim3(K9_THREADS), 0, st, p, s, d)
            : launch_ex(k9_ragged<ES, false>, dim3(blocks), dim3(K9_THREADS), 0, st, p, s, d);
}

}  // namespace

int k9_tile_a(int es) { return 128 / es; }
int k9_tile_b() { return K9_TB; }

cudaError_t launch_k9(const K9Params &p, int es, const void *src, void *dst, cudaStream_t st) {
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  cudaError_t e;
  switch (es) {
    case 1: e = go<1>(p, s, d, st); break;
    case 2: e = go<2>(p, s, d, st); break;
    case 4: e = go<4>(p, s, d, st); break;
    case 8: e = go<8>(p, s, d, st); break;
    case 16: e = go<16>(p, s, d, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

}  // namespace axe
