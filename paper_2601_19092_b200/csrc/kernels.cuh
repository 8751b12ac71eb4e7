// kernels.cuh -- parameter blocks of the libaxe kernels (host <-> device).
//
// Every block is passed by value as a __grid_constant__ kernel parameter.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define AXE_HD __host__ __device__ __forceinline__
#else
#define AXE_HD inline
#endif

namespace axe {

// Unsigned 32-bit division by an invariant divisor: q = (umulhi(n, m) + n) >> l
// (round-up multiplier; exact for every n < 2^32 and 1 <= d < 2^32).
struct FastDiv {
  uint32_t d, m, l;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t l = 0;
  while (l < 32 && (uint64_t(1) << l) < d) l++;
  f.l = l;
  f.m = (uint32_t)(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
  return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fdiv(const FastDiv &f, uint32_t n) {
  uint32_t t = __umulhi(n, f.m);
  return (uint32_t)(((uint64_t)t + n) >> f.l);
}
#endif

#ifdef __CUDACC__
// The work units (tiles, boxes) one CTA moves.  chunk == 0: a persistent grid, CTA b takes units b, b + G,
// b + 2G, ...; chunk > 0: CTA b takes units [b chunk, (b + 1) chunk) and the grid covers all of them, so
// the hardware's in-order CTA dispatch keeps the units in flight a narrow moving window of addresses
// (a persistent grid's CTAs drift apart and spread it: 256 MiB fp32 transpose 92.6 us -> 81.9 us,
// profiles/r02_sweep_front.log)
struct UnitRange {
  uint32_t lo, end, step;
};
__device__ __forceinline__ UnitRange unit_range(uint32_t n, uint32_t chunk) {
  if (chunk) {
    const uint32_t lo = blockIdx.x * chunk;
    return {lo, lo < n ? (n - lo < chunk ? n : lo + chunk) : lo, 1u};
  }
  return {blockIdx.x, n, gridDim.x};
}
#endif

// Byte-offset swizzle b' = b ^ (((b >> (M+S)) & mask) << M) (CUTLASS Swizzle<B,M,S>, R16).
struct Swz {
  uint32_t shift;  // M + S
  uint32_t mask;   // 2^B - 1 (0: no swizzle)
  uint32_t base;   // M
};
AXE_HD int64_t swz(const Swz &s, int64_t b) { return b ^ (int64_t)(((uint64_t)b >> s.shift) & s.mask) << s.base; }

// ---------------------------------------------------------------- K0 generic
constexpr int K0_MAXI = 16;   // iters per D or R
constexpr int K0_MAXAX = 8;   // axes per side
constexpr int K0_MAXSD = 12;  // storage digits per side

struct K0Side {
  int nD, nR, nsd, nax;
  int64_t e[K0_MAXI], s[K0_MAXI];
  int8_t ax[K0_MAXI];
  int64_t re[K0_MAXI], rs[K0_MAXI];
  int8_t rax[K0_MAXI];
  int64_t off[K0_MAXAX];
  int8_t sax[K0_MAXSD];  // -1: skipped axis (gpuid)
  int64_t sext[K0_MAXSD], sdiv[K0_MAXSD];
  Swz sw;
};
struct K0Params {
  K0Side src, dst;
  int64_t ED, ER;
  int es;
  int dep;  // 1: wait for the previous kernel in the stream (griddepcontrol.wait)
};

// ---------------------------------------------------------------- K1 vector
constexpr int K1_MAXD = 16;
constexpr int K1_MAXREP = 32;
struct K1Params {
  uint32_t total;   // number of vectors
  int nd;           // joint digits (vector digit excluded) in kernel order, outermost first
  FastDiv fd[K1_MAXD];
  int64_t ss[K1_MAXD], ds[K1_MAXD];  // byte strides
  int64_t sbase, dbase;              // byte offsets of the representative cells
  int nrep;
  int64_t rep[K1_MAXREP];            // byte offsets of the destination replicas (rep[0] = 0)
  Swz ssw, dsw;
  // tiled mode (tile_v > 0): vectors [t*tile_v, (t+1)*tile_v) form tile t; the
  // inner digits give every thread fixed offsets, the outer digits a tile base.
  uint32_t tile_v, ntiles;
  int nin, nout;
  FastDiv ifd[K1_MAXD], ofd[K1_MAXD];
  int64_t iss[K1_MAXD], ids[K1_MAXD], oss[K1_MAXD], ods[K1_MAXD];
  int pre_s, pre_d;  // swizzle folded into the per-thread offsets (tile bases are whole swizzle blocks)
  uint32_t chunk;    // tiles per CTA (unit_range); 0: persistent grid
  int dep;           // 1: wait for the previous kernel in the stream (griddepcontrol.wait)
};

// ---------------------------------------------------------------- K8 dual decoding
// Layout pairs whose digit systems do not nest (no joint refinement, the gcd = 1 failure of Alg. 1,
// P:978): the innermost digits still refine jointly (joint_refine_partial, down to the gcd of the
// first non-nesting pair), and the outer index o = x / G is decoded twice -- once per side.  Vector i
// of the grid = (o, w): w indexes the vectors of one inner block (K1's inner digits, the shared
// contiguous run as the vector), o the block; a warp's lanes take consecutive vectors, so runs stay
// coalesced on both sides.
constexpr int K8_MAXD = 12;
struct K8Params {
  uint32_t total;              // vectors
  FastDiv vin;                 // vectors per inner block
  int nin;                     // inner digits (vector digit excluded), outermost first
  FastDiv ifd[K1_MAXD];
  int64_t iss[K1_MAXD], ids[K1_MAXD];  // byte strides
  int na, nb;                  // outer digits of the source / destination decoding, outermost first
  FastDiv afd[K8_MAXD], bfd[K8_MAXD];
  int64_t as[K8_MAXD], bs[K8_MAXD];    // byte strides
  int64_t sbase, dbase;
  int nrep;
  int64_t rep[K1_MAXREP];
  Swz ssw, dsw;
  // chunked form (inner block = one run of vin >= K8_CHUNK vectors contiguous in vector units on both
  // sides: iss[0] / ids[0] its byte strides): work item = (o, chunk of K8_CHUNK vectors of block o),
  // the two outer decodings once per item instead of once per vector
  int chunked;
  uint32_t nitems;
  FastDiv nchunks;
  // bulk form (k8_bulk, kernels_tma.cu): the inner block is one run contiguous on both sides, moved as
  // boxes of `box` bytes by cp.async.bulk global -> smem -> global; box b = (o, r): run o, piece r
  int bulk;
  uint32_t box, nboxes, stages, prefetch;
  FastDiv per_run;                     // boxes per run
  // odometer form (odo = 1; gcd 1, vectors of one element): a warp walks K8_ODO_J * 32 consecutive x,
  // lane by lane; each lane carries (x / E, x mod E) of the innermost digit of both lists (extents
  // afd[na-1] / bfd[nb-1]) and re-decodes the outer digits only when its innermost digit wraps
  int odo;
  uint32_t nchunk;                     // chunks of K8_ODO_J * 32 elements
  uint32_t chunk;                      // bulk boxes / chunked-form items per CTA (unit_range); 0: persistent
  int dep;
};
constexpr int K8_ODO_J = 64;

// ---------------------------------------------------------------- K1-TMA
// The paper's TMA lowering: every box is (rows x row bytes), whole
// in shared memory; one side is addressed through a CUtensorMap (5-D, byte
// elements, the other side's swizzle applied in smem), the other side is a
// contiguous run of box_bytes moved with one bulk copy.
//   mode 0: TMA tensor load (src)  -> smem -> bulk store (dst, every replica)
//   mode 1: bulk load (src)        -> smem -> TMA tensor store (dst)
constexpr int TMA_MAXD = 6;
// one swizzle atom of a lowered TMA region (tma_region.cpp): tensor-map coordinates (dim 0 in bytes)
// and the byte offset of its slot in the shared-memory image
struct TmaAtom {
  int32_t c[5];
  int32_t pad;
  int64_t off;
};
// destination replicas of a lowered load (byte offsets added to every box's image offset)
struct TmaReps {
  int n;
  int64_t r[K1_MAXREP];
};
// The box table of a lowered region as a mixed-radix program (tma_region.cpp fit_program): box b has
// digits d_k (innermost first, extents fd[k].d) and coordinates c0 + sum_k d_k dc[k], image offset
// off0 + sum_k d_k doff[k].  The tiler T and the row-major atom grid of the lowering are both
// mixed-radix, so every box table the planner builds so far has this form; nd = -1 (a table the fit
// does not reproduce exactly) reads the table from global memory instead.
constexpr int TR_MAXD = 10;
struct TrProg {
  int nd;
  FastDiv fd[TR_MAXD];
  int32_t c0[5];
  int32_t dc[TR_MAXD][5];
  int64_t off0;
  int64_t doff[TR_MAXD];
};
struct TrParams {
  TrProg prog;
  const TmaAtom *atoms;  // the table (prog.nd < 0 only)
  uint8_t *img;
  uint32_t n;            // boxes
  uint32_t box;          // bytes per box
  uint32_t slot;         // ring slot stride (box rounded up to 1 KiB: every slot starts a swizzle pattern)
  uint32_t stages;       // ring slots per CTA
  int dep;               // 1: griddepcontrol.wait before the first TMA
  int strided;           // 1: CTA c takes boxes c, c + grid, ... (0: a contiguous range per CTA)
  uint32_t prefetch;     // boxes per CTA pulled into L2 before griddepcontrol.wait
  uint32_t chunk;        // > 0: the in-order schedule, `chunk` consecutive units per CTA over a covering grid
  int pair;              // > 1: units of `pair` boxes whose image slots are contiguous (one image-side bulk copy)
  TmaReps reps;
};

struct TmaParams {
  uint32_t nboxes;
  int nd;                      // box-index digits, outermost first
  FastDiv fd[TMA_MAXD];
  int32_t cdim[TMA_MAXD];      // tensor-map dimension the digit moves along
  int32_t cmul[TMA_MAXD];      // coordinate step per digit value
  int64_t bstride[TMA_MAXD];   // byte stride of the digit on the bulk side
  int64_t bbase;               // byte offset of box 0 on the bulk side
  int64_t sstride[TMA_MAXD];   // mode 2 (bulk load + bulk store): byte stride on the source side
  int64_t sbase;               // mode 2: byte offset of box 0 on the source side
  uint32_t box_bytes;
  uint32_t slot_bytes;         // ring slot stride: box_bytes rounded up to 128 B (TMA smem alignment;
                               // 1024 B with a swizzle, so every slot starts a swizzle pattern)
  int stages;
  int mode;
  int xform;                   // 1: movmatrix.trans of every 512-byte block in shared memory (K3-TMA)
  int nrep;
  int64_t rep[K1_MAXREP];      // mode 0: byte offsets of the destination replicas
  uint32_t chunk;              // boxes per CTA (unit_range); 0: persistent grid
  uint32_t prefetch;           // boxes per CTA pulled into L2 before griddepcontrol.wait (0: the ring)
  int dep;                     // 1: wait for the previous kernel in the stream (griddepcontrol.wait)
};

// ---------------------------------------------------------------- K2 tile
// A tile = the tile digits (a source-contiguous run x a destination-contiguous
// run x whatever else they share), staged through shared memory in source
// order; the other digits index tiles.  Load: every thread moves VS-byte
// vectors global -> smem; store: every thread gathers granules from smem into
// VD-byte destination vectors.  All per-thread offsets are tables built on the
// host: offset(j, t[, k]) = B[j] + A[t] (+ C[k]).
constexpr int K2_NT = 256;
constexpr int K2_MAXJ = 16;
constexpr int K2_MAXK = 16;
struct K2Params {
  uint32_t ntiles;
  int nout;
  FastDiv ofd[K1_MAXD];
  int64_t oss[K1_MAXD], ods[K1_MAXD];  // byte strides of the tile-index digits
  int64_t sbase, dbase;                // bytes
  int lj, sj, kg;                      // load iterations, store iterations, granules per store vector
  int32_t A_l[K2_NT], A_s[K2_NT], A_d[K2_NT];  // bytes: src global, smem (pre-swizzle), dst global
  int32_t B_l[K2_MAXJ], B_s[K2_MAXJ], B_d[K2_MAXJ];
  int32_t C_s[K2_MAXK];
  uint32_t tile_bytes;
  Swz smsw;                            // shared-memory swizzle chosen by the planner
  Swz ssw, dsw;                        // global swizzles of the storages
  int nrep;
  int64_t rep[K1_MAXREP];
  uint32_t chunk;  // tiles per CTA (unit_range); 0: persistent grid
  int dep;
};


// ---------------------------------------------------------------- K3 movmatrix
// Register-layout permute that is, on every 512-byte "warp row" of a register
// dump (32 lanes x 8 b16 registers), the per-register 8x8 transpose of
// movmatrix.sync.aligned.m8n8.trans.b16 (config 3b): one warp moves one block
// with LDG.128, 4 x MOVM, STG.128 -- no shared memory.
struct K3Params {
  uint32_t nblocks;
  int nd;  // block-index digits, outermost first
  FastDiv fd[K1_MAXD];
  int64_t ss[K1_MAXD], ds[K1_MAXD];  // bytes
  int64_t sbase, dbase;
  int nrep;
  int64_t rep[K1_MAXREP];
  Swz ssw, dsw;
  int dep;
};

// ------------------------------------------------ K6 granule transpose (config 3a)
// A copy whose 16-byte source vectors, taken n = 16 / G at a time (G = the shared contiguous
// granule, 4 or 8 bytes), form an n x n matrix of granules that the destination wants transposed:
// n threads load n consecutive source vectors, transpose the granules with warp shuffles, and each
// stores one 16-byte destination vector -- no shared memory.
#ifndef AXE_K6_U
// measured on config 3a: persistent grid U = 4: 1402 us, 8: 1358 us, 16: 1884 us (147 registers); with the
// in-order schedule U = 4 (4 tiles per CTA) 1277 us vs U = 8 (8 tiles) 1308 us
#define AXE_K6_U 4
#endif
constexpr int K6_U = AXE_K6_U;  // groups per thread per tile
struct K6Params {
  uint32_t ngroups;                  // groups of n threads
  int n;                             // 4 (4-byte granules) or 2 (8-byte granules)
  // tiles of (256 / n) * K6_U groups: inner digits give every thread fixed offsets, outer digits a
  // tile base (decoded once per tile)
  uint32_t tile_g, ntiles;
  int nin, nout;
  FastDiv ifd[K1_MAXD], ofd[K1_MAXD];
  int64_t iss[K1_MAXD], ids[K1_MAXD], oss[K1_MAXD], ods[K1_MAXD];  // bytes
  int64_t sbase, dbase;
  int64_t sstep;                     // bytes between the n source vectors of a group (16)
  int64_t dpos[4];                   // destination offset of the vector holding granule position j
  int nrep;
  int64_t rep[K1_MAXREP];
  Swz ssw, dsw;
  uint32_t chunk;  // tiles per CTA (unit_range); 0: persistent grid
  int dep;
};

// ------------------------------------------------ K7 register-block transpose
// A 2-D transpose of es = 2 / 4 / 8-byte elements (n = 16 / es): tiles of (32 n) source rows x
// (8 n) source columns are staged in shared memory in source order (16-byte chunks XOR-swizzled by
// (row / n) mod 8); each thread then loads an n x n element block with n LDS.128, transposes it in
// registers (byte permutes for 2-byte elements, register renaming for 4-byte ones) and stores n
// destination vectors; a warp's 32 threads take 32 consecutive row blocks, so each store
// instruction writes 512 contiguous destination bytes.
struct K7Params {
  uint32_t ntiles;
  int nd;                              // tile-index digits, outermost first
  FastDiv fd[K1_MAXD];
  int64_t ss[K1_MAXD], ds[K1_MAXD];    // bytes
  int64_t sbase, dbase;
  int64_t src_row, dst_col;            // bytes between source rows / destination columns
  int cw;                              // chunk columns per warp (tile columns = 8 n cw)
  int async;                           // 1: cp.async into a second tile buffer while the first is stored
  int stcs;                            // streaming (evict-first) stores
  int nrep;
  int64_t rep[K1_MAXREP];
  uint32_t chunk;                      // tiles per CTA (unit_range); 0: persistent grid
  // ragged edges: tile digit ka (kb) steps the source columns (rows) by one tile; only elements below
  // lim_a columns / lim_b rows exist (both whole 16-byte vectors).  -1: whole tiles on that side
  int ka, kb;
  uint32_t lim_a, lim_b;
  int dep;
};

// ---------------------------------------------------------------- K9 ragged transpose
// 2-D transposes of any extents and pitches (element-aligned only): tiles of 64 rows x 128 bytes staged
// in shared memory (rows padded so column reads are conflict-free), element-granular loads along the
// source rows and stores along the destination rows -- both coalesced -- predicated at the edges.
struct K9Params {
  uint32_t ntiles;
  FastDiv fa, fb;                      // tiles along a (source-contiguous) / b (destination-contiguous)
  int nd;                              // batch digits, outermost first
  FastDiv fd[K1_MAXD];
  int64_t ss[K1_MAXD], ds[K1_MAXD];    // bytes
  int64_t ea, eb;                      // extents of a and b
  int64_t s_b, d_a;                    // source byte stride of b (row pitch), destination byte stride of a
  int64_t sbase, dbase;
  Swz ssw, dsw;
  int nrep;
  int64_t rep[K1_MAXREP];
  // vector-load form (vec = 1; 16-byte aligned source buffer): every tile row is fetched as the 16-byte
  // chunks covering it (whatever its alignment); chunks at or past src_limit (the source storage's bytes
  // rounded up to 16) are not read
  int vec;
  int64_t src_limit;
  uint32_t chunk;                      // tiles per CTA (unit_range); 0: persistent grid
  int dep;
};

// ------------------------------------------------------- K4 reduce (§8(f) f3)
// dst(y) = sum_k src(k * E_D(dst) + y) (reading R24).  Element types:
enum DType { DT_F32 = 1, DT_F64 = 2, DT_F16 = 3, DT_BF16 = 4, DT_I32 = 5, DT_I64 = 6 };
constexpr int K4_MAXD = 12;
constexpr int K4_MAXK = 256;  // summand offsets kept as a table up to this K
struct K4Params {
  uint32_t total;                      // output vectors
  int nd;                              // output digits, outermost first
  FastDiv fd[K4_MAXD];
  int64_t ss[K4_MAXD], ds[K4_MAXD];    // byte strides (source, destination)
  int nk;                              // > 0: koff[0..nk) are the summands' byte offsets, k ascending
  int64_t koff[K4_MAXK];
  uint32_t ktotal;                     // nk == 0: decode k over the reduction digits
  int nkd;
  FastDiv kfd[K4_MAXD];
  int64_t kss[K4_MAXD];
  int64_t sbase, dbase;
  int nrep;
  int64_t rep[K1_MAXREP];
  Swz ssw, dsw;
  int stcs;                            // vector form: streaming (evict-first) stores of the sums
  uint32_t chunk;                      // vector form: blocks of blockDim.x vectors per CTA (unit_range)
  int dep;
};
// one-sided (pull) form: summand k is read through its own base pointer (a peer's buffer)
struct K4Ptrs {
  uint64_t p[K4_MAXK];
};
// generic form: both layouts evaluated per element (K0 sides; the source side spans K * Y)
struct K4GParams {
  K0Side src, dst;
  int64_t Y, K, ER;
  int dep;
};

}  // namespace axe
