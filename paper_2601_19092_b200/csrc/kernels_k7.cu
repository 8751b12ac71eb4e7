// kernels_k7.cu -- K7: register-block transpose through shared memory (sm_100a).
//
// Row-major -> column-major (any 2-D transpose of 2-, 4- or 8-byte elements).
// The smem-staged K2 gathers one element per shared load (8 LDS.U16 per 16-byte
// bf16 output) and is limited by the SM, not by HBM.  K7 reads n x n element
// blocks with n LDS.128 (n = 16 / es) and transposes them in registers: for
// 4-byte elements a block is just renamed, for 2-byte elements 4 PRMT build
// each output word, for 8-byte elements the two halves swap.  Tile: 32 n source
// rows x 8 n source columns (8 chunks of 16 bytes per row); warp w owns chunk
// column w, lane l owns rows [n l, n l + n).  Chunk c of row r is stored at
// chunk c ^ ((r / n) mod 8), so the 32 lanes of every LDS.128 read 8 distinct
// chunk positions (4 wavefronts, the minimum for 512 bytes).
#include <cuda_runtime.h>

#include <atomic>

#include "kernels.cuh"
#include "launch.cuh"

namespace axe {

extern std::atomic<int64_t> g_launches;

namespace {

constexpr int K7_THREADS = 256;

__device__ __forceinline__ uint4 ldg128(const uint8_t *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t word(const uint4 &v, int m) { return m == 0 ? v.x : m == 1 ? v.y : m == 2 ? v.z : v.w; }

template <int ES, int CW, bool RG>
__device__ __forceinline__ void k7_gather(const K7Params &p, const uint8_t *sm, int64_t db, uint8_t *__restrict__ dst,
                                          int lane, int warp, uint32_t ra, uint32_t rb) {
  constexpr int N = 16 / ES;
  constexpr int CH = 8 * CW;
  // RG (ragged plans only): ra / rb = the source columns / rows of this tile that exist
  if (RG && (uint32_t)(lane * N) >= rb) return;
  // gather: lane = row block, warp (+ 8 cw) = chunk column
#pragma unroll
  for (int cw = 0; cw < CW; cw++) {
    const int cc = warp + 8 * cw;
    if (RG && (uint32_t)(cc * N) >= ra) break;
    uint4 w[N];
#pragma unroll
    for (int i = 0; i < N; i++) {
      const int r = lane * N + i;
      w[i] = *reinterpret_cast<const uint4 *>(sm + (r * CH + (cc ^ (lane & 7))) * 16);
    }
    const int64_t d0 = db + (int64_t)(cc * N) * p.dst_col + (int64_t)lane * 16;
#pragma unroll
    for (int k = 0; k < N; k++) {
      uint4 o;
      if constexpr (ES == 4) {
        o = make_uint4(word(w[0], k), word(w[1], k), word(w[2], k), word(w[3], k));
      } else if constexpr (ES == 2) {
        const uint32_t sel = (k & 1) ? 0x7632u : 0x5410u;  // high or low halves of the rows' words
        const int m = k >> 1;
        o.x = __byte_perm(word(w[0], m), word(w[1], m), sel);
        o.y = __byte_perm(word(w[2], m), word(w[3], m), sel);
        o.z = __byte_perm(word(w[4], m), word(w[5], m), sel);
        o.w = __byte_perm(word(w[6], m), word(w[7], m), sel);
      } else {  // ES == 8: element k of rows 0 and 1
        o = k == 0 ? make_uint4(w[0].x, w[0].y, w[1].x, w[1].y) : make_uint4(w[0].z, w[0].w, w[1].z, w[1].w);
      }
      const int64_t d = d0 + (int64_t)k * p.dst_col;
      for (int r = 0; r < p.nrep; r++) {
        uint8_t *q = dst + d + p.rep[r];
        if (p.stcs)
          asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(q), "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w)
                       : "memory");
        else
          *reinterpret_cast<uint4 *>(q) = o;
      }
    }
  }
}

// tile i's byte offsets, and the source columns (ra) / rows (rb) of it that exist: a ragged edge tile
// (digit ka / kb at its last value) keeps lim - d * T of its T columns / rows
template <bool RG>
__device__ __forceinline__ void tile_offsets(const K7Params &p, uint32_t i, int64_t &sb, int64_t &db, uint32_t TC,
                                             uint32_t TR, uint32_t &ra, uint32_t &rb) {
  sb = p.sbase;
  db = p.dbase;
  ra = RG ? min(TC, p.lim_a) : TC;  // (a ragged side of less than one tile has no digit)
  rb = RG ? min(TR, p.lim_b) : TR;
  for (int k = p.nd - 1; k >= 1; k--) {
    const uint32_t q = fdiv(p.fd[k], i);
    const uint32_t d = i - q * p.fd[k].d;
    i = q;
    sb += (int64_t)d * p.ss[k];
    db += (int64_t)d * p.ds[k];
    if (RG && k == p.ka) ra = min(TC, p.lim_a - d * TC);
    if (RG && k == p.kb) rb = min(TR, p.lim_b - d * TR);
  }
  if (p.nd > 0) {
    sb += (int64_t)i * p.ss[0];
    db += (int64_t)i * p.ds[0];
    if (RG && p.ka == 0) ra = min(TC, p.lim_a - i * TC);
    if (RG && p.kb == 0) rb = min(TR, p.lim_b - i * TR);
  }
}

template <int ES, int CW, bool RG>
__global__ void __launch_bounds__(K7_THREADS) k7_transpose(const __grid_constant__ K7Params p,
                                                           const uint8_t *__restrict__ src, uint8_t *__restrict__ dst) {
  constexpr int N = 16 / ES;          // elements per 16-byte vector
  constexpr int TR = 32 * N;          // tile rows (source)
  constexpr int CH = 8 * CW;          // 16-byte chunks per tile row (8 n CW columns; warp w owns w, w + 8, ..)
  constexpr int LOADS = TR * CH / K7_THREADS;  // 16-byte loads per thread per tile
  extern __shared__ __align__(128) uint8_t sm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (p.dep) pdl_wait();
  pdl_launch_dependents();
  const UnitRange R = unit_range(p.ntiles, p.chunk);
  for (uint32_t tile = R.lo; tile < R.end; tile += R.step) {
    int64_t sb, db;
    uint32_t ra, rb;
    tile_offsets<RG>(p, tile, sb, db, 8 * N * CW, TR, ra, rb);
    // load: 8 consecutive threads read one 128-byte source row
    uint4 v[LOADS];
#pragma unroll
    for (int u = 0; u < LOADS; u++) {
      const int idx = t + u * K7_THREADS, r = idx / CH, c = idx % CH;
      v[u] = !RG || ((uint32_t)r < rb && (uint32_t)(c * N) < ra) ? ldg128(src + sb + (int64_t)r * p.src_row + c * 16)
                                                                 : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < LOADS; u++) {
      const int idx = t + u * K7_THREADS, r = idx / CH, c = idx % CH;
      *reinterpret_cast<uint4 *>(sm + (r * CH + (c ^ ((r / N) & 7))) * 16) = v[u];  // XOR on the low 3 bits
    }
    __syncthreads();
    k7_gather<ES, CW, RG>(p, sm, db, dst, lane, warp, ra, rb);
    __syncthreads();
  }
}

// Double-buffered form: the next tile's 16-byte source vectors go straight to the second shared buffer
// with cp.async (no registers held) while the current tile is gathered and stored.
__device__ __forceinline__ void cp_async16(uint8_t *s, const uint8_t *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}

template <int ES, int CW, int S, bool RG>
__global__ void __launch_bounds__(K7_THREADS) k7_transpose_async(const __grid_constant__ K7Params p,
                                                                 const uint8_t *__restrict__ src,
                                                                 uint8_t *__restrict__ dst) {
  constexpr int N = 16 / ES;
  constexpr int TR = 32 * N;
  constexpr int CH = 8 * CW;
  constexpr int LOADS = TR * CH / K7_THREADS;
  constexpr int TILE = TR * CH * 16;
  extern __shared__ __align__(128) uint8_t sm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const UnitRange R = unit_range(p.ntiles, p.chunk);
  if (p.dep) {
    // while the previous kernel drains: the ring's first tiles into L2, one 128-byte line per thread and
    // pass (R28)
    for (int s = 0; s < S - 1; s++) {
      const uint32_t tt = R.lo + (uint32_t)s * R.step;
      if (tt >= R.end) break;
      int64_t sb, db;
      uint32_t ra, rb;
      tile_offsets<RG>(p, tt, sb, db, 8 * N * CW, TR, ra, rb);
      for (int idx = t; idx < TR * (CH / 8); idx += K7_THREADS)
        if (!RG || ((uint32_t)(idx / (CH / 8)) < rb && (uint32_t)((idx % (CH / 8)) * 8 * N) < ra))
          prefetch_l2(src + sb + (int64_t)(idx / (CH / 8)) * p.src_row + (idx % (CH / 8)) * 128);
    }
    pdl_wait();
  }
  pdl_launch_dependents();
  auto issue = [&](uint32_t tile, uint8_t *buf) {
    int64_t sb, db;
    uint32_t ra, rb;
    tile_offsets<RG>(p, tile, sb, db, 8 * N * CW, TR, ra, rb);
#pragma unroll
    for (int u = 0; u < LOADS; u++) {
      const int idx = t + u * K7_THREADS, r = idx / CH, c = idx % CH;
      if (!RG || ((uint32_t)r < rb && (uint32_t)(c * N) < ra))
        cp_async16(buf + (r * CH + (c ^ ((r / N) & 7))) * 16, src + sb + (int64_t)r * p.src_row + c * 16);
    }
  };
  // S-stage ring: tiles it + 1 .. it + S - 1 are in flight while tile it is gathered and stored
  uint32_t tile = R.lo;
#pragma unroll
  for (int s = 0; s < S - 1; s++) {
    const uint32_t tt = tile + (uint32_t)s * R.step;
    if (tt < R.end) issue(tt, sm + s * TILE);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; tile < R.end; tile += R.step, it++) {
    const uint32_t next = tile + (uint32_t)(S - 1) * R.step;
    if (next < R.end) issue(next, sm + ((it + S - 1) % S) * TILE);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");  // this thread's vectors of `tile` landed
    __syncthreads();                                                    // ... and every other thread's
    int64_t sb, db;
    uint32_t ra, rb;
    tile_offsets<RG>(p, tile, sb, db, 8 * N * CW, TR, ra, rb);
    k7_gather<ES, CW, RG>(p, sm + (it % S) * TILE, db, dst, lane, warp, ra, rb);
    __syncthreads();  // buffer it % S is refilled by a later iteration's issue
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int ES, int CW, int S, bool RG>
cudaError_t go_async(const K7Params &p, unsigned blocks, size_t tile, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  const cudaError_t e = smem_attr((const void *)k7_transpose_async<ES, CW, S, RG>, 200 * 1024);
  if (e != cudaSuccess) return e;
  return launch_ex(k7_transpose_async<ES, CW, S, RG>, dim3(blocks), dim3(K7_THREADS), S * tile, st, p, s, d);
}

// RG: the ragged-edge variant (masked loads and stores); whole-tile plans run the unmasked one (the masks
// cost the 1-CTA-per-SM bf16 form 17%: 8192^2 52.5 us vs 44.9)
template <int ES, int CW, bool RG>
cudaError_t go_rg(const K7Params &p, unsigned blocks, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  constexpr int N = 16 / ES;
  const size_t tile = (size_t)32 * N * 8 * CW * 16;
  if (p.async) {
    if (p.async == 4) return go_async<ES, CW, 4, RG>(p, blocks, tile, s, d, st);
    if (p.async == 3) return go_async<ES, CW, 3, RG>(p, blocks, tile, s, d, st);
    return go_async<ES, CW, 2, RG>(p, blocks, tile, s, d, st);
  }
  const cudaError_t e = smem_attr((const void *)k7_transpose<ES, CW, RG>, 100 * 1024);
  if (e != cudaSuccess) return e;
  return launch_ex(k7_transpose<ES, CW, RG>, dim3(blocks), dim3(K7_THREADS), tile, st, p, s, d);
}

template <int ES, int CW>
cudaError_t go(const K7Params &p, unsigned blocks, const uint8_t *s, uint8_t *d, cudaStream_t st) {
  constexpr int N = 16 / ES;
  const bool ragged = p.ka >= 0 || p.kb >= 0 || p.lim_a < (uint32_t)(8 * N * CW) || p.lim_b < (uint32_t)(32 * N);
  return ragged ? go_rg<ES, CW, true>(p, blocks, s, d, st) : go_rg<ES, CW, false>(p, blocks, s, d, st);
}

}  // namespace

cudaError_t launch_k7(const K7Params &p, int es, unsigned blocks, const void *src, void *dst, cudaStream_t st) {
  const uint8_t *s = (const uint8_t *)src;
  uint8_t *d = (uint8_t *)dst;
  cudaError_t e;
  switch (es) {
    case 2: e = p.cw == 2 ? go<2, 2>(p, blocks, s, d, st) : go<2, 1>(p, blocks, s, d, st); break;
    case 4:
      e = p.cw == 4 ? go<4, 4>(p, blocks, s, d, st) : p.cw == 2 ? go<4, 2>(p, blocks, s, d, st) : go<4, 1>(p, blocks, s, d, st);
      break;
    case 8:
      e = p.cw == 4 ? go<8, 4>(p, blocks, s, d, st) : p.cw == 2 ? go<8, 2>(p, blocks, s, d, st) : go<8, 1>(p, blocks, s, d, st);
      break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  g_launches++;
  return cudaGetLastError();
}

}  // namespace axe
