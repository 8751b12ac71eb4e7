/*
 * axe.h -- C ABI of libaxe: Axe layouts (arXiv 2601.19092) and layout-driven
 * tensor data movement on B200 (sm_100a).
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line (section / definition
 * named beside it); "R<n>" = a reading listed in DESIGN.md §3.
 *
 * Conventions:
 *   - An Axe layout L = (D, R, O) (Def. Layout) maps a logical index
 *     x in [0, E_D) to the set f_L(x) = { f_D(x) + f_R(r) + O } of coordinates on
 *     named axes (Def. Induced map).  D is unflattened
 *     lexicographically, last iter fastest (R2).
 *   - Strides and offsets on memory axes are in ELEMENTS (R3); bytes appear
 *     only inside the swizzle.
 *   - A tensor = layout + pointer + element size; "address = base pointer +
 *     memory components of the layout".  Where the axes of a layout
 *     live in a buffer is given by an axe_storage descriptor (R17).
 *   - All calls are thread-safe; layout handles are immutable.
 *   - Every validation happens on the host before any launch; a failing call
 *     launches nothing and leaves every buffer untouched.
 *   - Errors: an axe_status != AXE_OK; axe_last_error() gives a thread-local
 *     message for the last failing call on this thread.
 */
#ifndef AXE_H_
#define AXE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int axe_status;
enum {
  AXE_OK = 0,
  AXE_ERR_INVALID_ARG = 1,      /* e < 1, s == 0, bad axis name, n_shard < 1, NULL pointer, bad storage */
  AXE_ERR_OVERFLOW = 2,         /* an extent product or coordinate leaves int64            */
  AXE_ERR_DOMAIN = 3,           /* x outside [0, E_D)                                                     */
  AXE_ERR_CAPACITY = 4,         /* caller's output array too small                                       */
  AXE_ERR_SIZE_MISMATCH = 5,    /* E_D(src) != E_D(dst)                                                   */
  AXE_ERR_NONINJECTIVE = 6,     /* two different x write the same destination cell (R6)                  */
  AXE_ERR_BOUNDS = 7,           /* a coordinate outside its storage box, or gpuid outside [0, nranks)     */
  AXE_ERR_UNSUPPORTED_AXIS = 8, /* axis not bound by the storage descriptor; gpuid in axe_copy           */
  AXE_ERR_ALIGNMENT = 9,        /* elem_size not in {1,2,4,8,16}; pointer misaligned for a forced plan    */
  AXE_ERR_ALIAS = 10,           /* source and destination byte ranges overlap (no in-place)               */
  AXE_ERR_CUDA = 11,            /* a CUDA runtime call failed (message has the CUDA error string)         */
  AXE_ERR_NCCL = 12,            /* an NCCL call failed                                                    */
  AXE_ERR_UNSUPPORTED = 13,     /* a forced kernel cannot run this pair of layouts                        */
  AXE_ERR_TIMEOUT = 14          /* axe_comm_wait: the stream did not finish in time (communicator aborted) */
};

/* ------------------------------------------------------------------------- */
/* Layouts (Defs. Iter, Layout, Induced map, span)                 */
/* ------------------------------------------------------------------------- */

typedef struct axe_layout axe_layout; /* opaque, immutable, shareable across threads */

/* An iter (e, s, a): extent e >= 1, stride s != 0 on axis a (Def. Iter).
 * axis == NULL means "m" ("if some stride is not paired with an axis, the axis m
 * is used by default").  Axis names are identifiers [A-Za-z_][A-Za-z0-9_]*. */
typedef struct {
  int64_t extent;
  int64_t stride;
  const char *axis;
} axe_iter;

/* One component of the offset O in ZA. */
typedef struct {
  const char *axis;
  int64_t value;
} axe_axis_coord;

/* Create L = (D, R, O).  shard: n_shard >= 1 iters, outermost first (D is an
 * ordered tuple).  replica: n_replica >= 0 iters (a multiset).  offset:
 * n_offset components; repeated axes add.  The library copies every input
 * (strings included).  Errors: AXE_ERR_INVALID_ARG, AXE_ERR_OVERFLOW (E_D or
 * E_R or an axis's coordinate range leaves int64). */
axe_status axe_layout_create(const axe_iter *shard, int n_shard, const axe_iter *replica, int n_replica,
                             const axe_axis_coord *offset, int n_offset, axe_layout **out);
void axe_layout_destroy(axe_layout *layout);

/* E_D = prod of shard extents, E_R = prod of replica extents (1 if none),
 * n_axes = number of distinct axes (first-appearance order over D, R, O). */
axe_status axe_layout_info(const axe_layout *layout, int64_t *E_D, int64_t *E_R, int *n_axes);
/* Name of axis i (0 <= i < n_axes); the string lives as long as the layout. */
axe_status axe_layout_axis_name(const axe_layout *layout, int i, const char **name);
/* Read back the iters: which = 0 for D, 1 for R.  *n receives the count; at most
 * capacity are written.  Axis strings live as long as the layout. */
axe_status axe_layout_iters(const axe_layout *layout, int which, axe_iter *out, int capacity, int *n);
/* Read back O (one entry per axis with a nonzero component). */
axe_status axe_layout_offset(const axe_layout *layout, axe_axis_coord *out, int capacity, int *n);

/* f_L(x) (Def. Induced map): writes E_R rows of n_axes int64 values,
 * row-major, replicas in lexicographic order (last replica iter fastest; R8).
 * capacity counts int64 values.  Errors: AXE_ERR_DOMAIN, AXE_ERR_CAPACITY. */
axe_status axe_layout_eval(const axe_layout *layout, int64_t x, int64_t *coords, int64_t capacity);

/* Canonical form (App. A.1): D0/D1 on D; C0/C1/C2 on (O, R).  The
 * result induces the same f_L (Prop.).  *gap_ok (may be NULL)
 * receives 1 when the canonical R satisfies the gap condition GC. */
axe_status axe_layout_canonicalize(const axe_layout *layout, axe_layout **out, int *gap_ok);

/* Signed min / max of the axis over every coordinate of every f_L(x) -- the
 * closed form of Lemma span-closed with O included (R1).  For an
 * axis the layout never names: min = max = 0 and AXE_OK. */
axe_status axe_layout_bounds(const axe_layout *layout, const char *axis, int64_t *min, int64_t *max);

/* ------------------------------------------------------------------------- */
/* Layout operators (§3.3, Apps. B-F): host-side algebra, the building blocks */
/* of the paper's TMA lowering.  Shapes are int64 arrays of `rank`  */
/* dimensions.  Algorithmic failure (the conditions are sufficient only) is   */
/* AXE_ERR_UNSUPPORTED; shape admission failure is AXE_ERR_SIZE_MISMATCH.     */
/* ------------------------------------------------------------------------- */

/* Group-By-Shape (Alg. 1): *out has D refined so that consecutive
 * blocks have extent products shape[i]; bounds (may be NULL, rank+1 ints)
 * receives the block boundaries into the refined D.  f_L is unchanged. */
axe_status axe_layout_group(const axe_layout *layout, const int64_t *shape, int rank, axe_layout **out, int *bounds);
/* span_a(f_L) in closed form (Lemma span-closed); 1 for an axis the layout never names. */
axe_status axe_layout_span(const axe_layout *layout, const char *axis, int64_t *span);
/* Tile (Alg. 2): f_T(x||y) = f_A(x) (.) span(f_B) + f_B(y), T grouped by
 * the interleaved shape (S_A[0], S_B[0], ..., S_A[r-1], S_B[r-1]). */
axe_status axe_layout_tile(const axe_layout *A, const int64_t *S_A, const axe_layout *B, const int64_t *S_B, int rank,
                           axe_layout **out);
/* TileOf_AndRecoverC (Alg. 3, with the offset / replication checks of
 * P:1332-1380): on success A = C (x) B; S_C (rank int64s) receives S_A / S_B. */
axe_status axe_layout_tile_of(const axe_layout *A, const int64_t *S_A, const axe_layout *B, const int64_t *S_B,
                              int rank, axe_layout **C, int64_t *S_C);
/* Direct sum on the tiling domain (App. F): f(x||y) = f_A(x) + f_B(y). */
axe_status axe_layout_direct_sum(const axe_layout *A, const int64_t *S_A, const axe_layout *B, const int64_t *S_B,
                                 int rank, axe_layout **out);
/* Slice L[R:S] (§3.3, Alg. 4 per block): region [begin, begin+extent) of
 * shape S; f_{L[R:S]<extent>}(u) = f_{L<S>}(u + begin). */
axe_status axe_layout_slice(const axe_layout *layout, const int64_t *shape, int rank, const int64_t *begin,
                            const int64_t *extent, axe_layout **out);

/* The paper's TMA lowering (§3.4): copy the region [begin, begin +
 * extent) of a global tensor (layout LG, logical shape EG; begin = NULL: all of
 * it) into a shared-memory tensor (layout LS, shape ES = the region's shape),
 * with the hardware swizzle of swizzle_bytes in {32, 64, 128}.  Steps: slice
 * (Alg. 4); the atom E_{d,a} = (1, .., 1, 8, swizzle_bytes / elem_size) and the
 * tiler T with LS = T (x) atom (Alg. 1 grouping + Alg. 3 matching, reading R26);
 * the atom's global counterpart as a suffix product of each group of the
 * grouped LG.  Layouts must be on the memory axis m, without replicas; strides
 * and offsets in elements.  *out receives the CuTensorMap encoding (dims and
 * byte strides innermost first, the atom box, the logical dimension of each
 * tensor-map dimension, the region's byte offset), the
 * atom count |T| and fused_rows (rows one box may cover when consecutive atoms
 * stack along rows in both memories, <= 256); *tiler (may be NULL) receives T.
 * Errors: AXE_ERR_UNSUPPORTED (no tiling / suffix product / > 5 dimensions /
 * non-contiguous innermost), AXE_ERR_SIZE_MISMATCH, AXE_ERR_ALIGNMENT. */
typedef struct {
  int rank;
  uint64_t dims[5];
  uint64_t strides[5]; /* bytes; strides[0] = elem_size */
  uint32_t box[5];
  int logical_dim[5];  /* the logical dimension (of EG) each tensor-map dimension belongs to */
  int swizzle_bytes;
  int64_t base_bytes;
  int64_t atoms;
  uint32_t fused_rows;
} axe_tma_desc;
axe_status axe_tma_lower(const axe_layout *LG, const int64_t *EG, const int64_t *begin, const int64_t *extent,
                         const axe_layout *LS, const int64_t *ES, int rank, int elem_size, int swizzle_bytes,
                         axe_tma_desc *out, axe_layout **tiler);

/* Executing a lowering on the device ("the shared memory layout is tiled by the
 * swizzle atom ... each tile issues one TMA instruction").  axe_tma_plan_create takes the
 * descriptor and tiler T that axe_tma_lower returned (the plan copies the descriptor and reads T
 * once; the caller keeps ownership of both).  axe_tma_plan_execute(plan, g_base, s_image, stream):
 * g_base is the device address of the global tensor's element m = 0 (the region's offset
 * base_bytes is added by the plan); s_image is a device buffer of image_bytes that receives the
 * shared-memory tensor L_S byte for byte -- atom t (row-major over the atom grid) at T(t) * 8 *
 * swizzle_bytes bytes, its bytes in the hardware's swizzled order (CUTLASS Swizzle<B,4,3> relative
 * to the image start, B = log2(swizzle_bytes / 16)).  One TMA tensor load per atom into a shared
 * ring slot, one bulk store per atom -- or per box of up to fused_rows / 8 atoms stacked along the
 * rows when T places them in consecutive slots (*boxes from axe_tma_plan_sizes; AXE_TMA_FUSE=0
 * keeps one atom per box); stream-ordered, asynchronous.  Both the region start and
 * s_image must be 16-byte aligned (AXE_ERR_ALIGNMENT).  The atom table is uploaded to the current
 * device at create (or by the first execute on another device -- synchronous, so that execute fails
 * with AXE_ERR_CUDA inside graph capture); the tensor map is re-encoded when g_base changes.
 * Errors: AXE_ERR_INVALID_ARG (not a lowering: box != one atom, bad rank / element size),
 * AXE_ERR_SIZE_MISMATCH (|T| != atoms), AXE_ERR_CUDA. */
typedef struct axe_tma_plan axe_tma_plan;
axe_status axe_tma_plan_create(const axe_tma_desc *desc, const axe_layout *tiler, axe_tma_plan **out);
axe_status axe_tma_plan_sizes(const axe_tma_plan *plan, int64_t *atoms, int64_t *boxes, int64_t *image_bytes);
axe_status axe_tma_plan_execute(axe_tma_plan *plan, const void *g_base, void *s_image, void *stream);
/* The reverse (the lowering's TMA store, shared -> global): every box is bulk-loaded from the image
 * and written to the region of the global tensor by one TMA tensor store (the hardware removes the
 * swizzle).  Writes exactly the region's elements of g_base; same alignment rules and errors. */
axe_status axe_tma_plan_execute_store(axe_tma_plan *plan, void *g_base, const void *s_image, void *stream);
void axe_tma_plan_destroy(axe_tma_plan *plan);

/* Textual form of the paper's matrix notation (Figures 2 and 5):
 *   layout  := shard ( "+" replica )? ( "+" offset )*
 *   shard   := "(" INT ("," INT)* "):(" stride ("," stride)* ")"
 *   stride  := INT ("@" AXIS)?          (axis m by default)
 *   replica := "[" shard "]"
 *   offset  := INT "@" AXIS             (repeated axes add)
 * Whitespace is insignificant.  Errors: AXE_ERR_INVALID_ARG with *error_pos (may
 * be NULL) = the byte offset of the syntax error, or -1 for a semantic error
 * (extent < 1, zero stride: Def. Iter); AXE_ERR_OVERFLOW. */
axe_status axe_layout_parse(const char *text, axe_layout **out, int *error_pos);
/* The layout in that grammar ("@m" omitted); parse(format(L)) is structurally L. */
axe_status axe_layout_format(const axe_layout *layout, char *buf, int capacity);
/* {"schema_version":1,"shard":[[e,s,"axis"],...],"replica":[...],"offset":{"axis":v},
 *  "E_D":..,"E_R":..,"text":"<format>"} */
axe_status axe_layout_to_json(const axe_layout *layout, char *buf, int capacity);
/* Do a and b induce the same map (§3.3 "verify if they represent the same induced
 * function")?  Both are canonicalized (App. A.1); when both canonical replica
 * sets satisfy the gap condition the canonical form is unique and
 * the answer is structural (D element-wise, R per axis as a multiset, O);
 * otherwise f_a(x) and f_b(x) are compared as sets for every x when E_D * E_R
 * <= threshold (< 0: 65536), else *result = -1 (undecidable).  *result = 1
 * equivalent, 0 not (different E_D is never equivalent). */
axe_status axe_layout_equivalent(const axe_layout *a, const axe_layout *b, int64_t threshold, int *result);

/* ------------------------------------------------------------------------- */
/* Storage descriptors (R16, R17)                                             */
/* ------------------------------------------------------------------------- */

/* One storage digit: the value (c[axis] / divisor) mod extent. */
typedef struct {
  const char *axis;
  int64_t extent;
  int64_t divisor;
} axe_storage_digit;

/* Element index of a coordinate c = sum_k ((c[a_k] / div_k) mod ext_k) * prod_{j>k} ext_j
 * (digits outermost first).  The digits of one axis must form a chain: the
 * divisor of a digit equals extent * divisor of the next (inner) digit of the
 * same axis, and the innermost digit of an axis has divisor 1; the outermost
 * digit of an axis bounds it: 0 <= c[a] < extent * divisor.  The buffer holds
 * prod_k ext_k elements of elem_size bytes.  Then the byte offset b = idx *
 * elem_size is swizzled as CUTLASS Swizzle<B, M, S> on bytes:
 *   b' = b ^ (((b >> (M + S)) & (2^B - 1)) << M)
 * (swz_bits = B, swz_base = M, swz_shift = S; B = 0 means no swizzle; SW128 =
 * (3,4,3), SW64 = (2,4,3), SW32 = (1,4,3): the TMA atom swizzles of P:527).
 * The swizzle is relative to the buffer base pointer. */
typedef struct {
  int n;
  const axe_storage_digit *digits;
  int swz_bits, swz_base, swz_shift;
} axe_storage;

/* ------------------------------------------------------------------------- */
/* Copy on one device (copy operator, schedules chosen from layouts) */
/* ------------------------------------------------------------------------- */

/* Kernel choice for plans (flags of axe_copy_plan_create); AUTO picks from the
 * layouts.  The environment variable AXE_FORCE_KERNEL
 * (generic | vector | tma | tile | register | shuffle | transpose | lowered | dual) overrides AUTO. */
enum {
  AXE_KERNEL_AUTO = 0,
  AXE_KERNEL_GENERIC = 1, /* K0: per-element evaluation of both layouts (always applicable) */
  AXE_KERNEL_VECTOR = 2,  /* K1: joint-digit vectorised LDG/STG copy                         */
  AXE_KERNEL_TMA = 3,     /* K1-TMA: TMA box load into swizzled smem + bulk store            */
  AXE_KERNEL_TILE = 4,    /* K2: smem-staged tile permute / transpose                        */
  AXE_KERNEL_REGISTER = 5, /* K3: warp-register permute through movmatrix (b16 8x8 atoms)    */
  /* 6: retired (K2T, a TMA-staged transpose AUTO never chose: K7 is faster); forcing it returns
        AXE_ERR_UNSUPPORTED */
  AXE_KERNEL_SHUFFLE = 7,  /* K6: n x n granule transpose across lanes with warp shuffles       */
  AXE_KERNEL_TRANSPOSE = 8, /* K7: smem tile + n x n register-block transpose (2-D transposes)  */
  AXE_KERNEL_LOWERED = 9,   /* the paper's TMA lowering (axe_tma_lower) as a copy schedule: the
                               destination is a tiling of the swizzle atom over the joint digits,
                               one TMA tensor op per (fused) atom box, one bulk copy per pair of
                               boxes contiguous in the image; AUTO takes it for copies into / out
                               of TMA-swizzled storage (config 2)                                 */
  AXE_KERNEL_DUAL = 10      /* K8: non-nested digit systems: the shared innermost run is
                               vectorised, the outer index decoded once per side                  */
};

typedef struct axe_copy_plan axe_copy_plan;

/* Plan a copy dst <- src (host only, no device work): validates both layouts
 * and storages, E_D(src) == E_D(dst), bounds, destination injectivity, and
 * chooses the kernel.  Copy semantics (R4, R6, R7): for every x, the bytes of
 * the source cell f_D^src(x) + O^src are written to every cell of f_L^dst(x);
 * cells of dst not in the image keep their contents; the bit pattern is moved
 * verbatim (no floating point).  elem_size in {1, 2, 4, 8, 16}.  Layouts may
 * not name the device axis "gpuid" (use axe_redistribute). */
axe_status axe_copy_plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                const axe_storage *dst_st, int elem_size, int kernel, axe_copy_plan **out);
/* Launch the planned copy on cuda_stream (a cudaStream_t; NULL = legacy default
 * stream), asynchronously.  src_ptr / dst_ptr are DEVICE pointers to buffers
 * of the storage sizes; the caller owns them.  Errors: AXE_ERR_ALIGNMENT (the
 * pointers are not aligned to the plan's vector width), AXE_ERR_ALIAS,
 * AXE_ERR_CUDA.  Launch count: 1 kernel.
 * Stream order: every libaxe kernel is launched with programmatic dependent
 * launch and waits (griddepcontrol.wait) for all work before it on the stream
 * before it touches its data; before that wait it may only prefetch its own
 * source into L2 (reading R28: a prefetch cannot observe stale data).  With
 * AXE_PDL_OVERLAP=1 (opt-in) a kernel proven disjoint from every libaxe kernel
 * in flight on its stream skips the wait -- only for streams that carry no
 * foreign kernels that trigger their dependents early. */
axe_status axe_copy_plan_execute(const axe_copy_plan *plan, const void *src_ptr, void *dst_ptr, void *cuda_stream);
/* As axe_copy_plan_create, with the host pipeline of axe_copy_plan_execute_host
 * cut into at most host_slabs slabs (0: the default, 8 or AXE_HOST_CHUNKS).
 * Fewer, larger slabs move PCIe data more efficiently when the caller overlaps
 * consecutive calls on different streams; more slabs overlap the two
 * directions within one call. */
axe_status axe_copy_plan_create_ex(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                   const axe_storage *dst_st, int elem_size, int kernel, int host_slabs,
                                   axe_copy_plan **out);
/* End-to-end variant: src/dst are HOST buffers (pinned for async overlap),
 * staged through the caller's device buffers dev_src / dev_dst (storage sizes)
 * with cudaMemcpyAsync: H2D, copy kernel, D2H, all on cuda_stream.  Asynchronous
 * with respect to the host. */
axe_status axe_copy_plan_execute_host(const axe_copy_plan *plan, const void *host_src, void *host_dst,
                                      void *dev_src, void *dev_dst, void *cuda_stream);
/* Byte sizes of the source and destination storages. */
axe_status axe_copy_plan_sizes(const axe_copy_plan *plan, int64_t *src_bytes, int64_t *dst_bytes);
/* A JSON description of the plan (kernel, joint digits, vector width, grid). */
axe_status axe_copy_plan_describe(const axe_copy_plan *plan, char *buf, int capacity);
void axe_copy_plan_destroy(axe_copy_plan *plan);

/* One-shot copy through an internal plan cache keyed by (layouts, storages,
 * elem_size, pointer alignment).  Same semantics and errors as plan_create +
 * plan_execute. */
axe_status axe_copy(const axe_layout *src, const axe_storage *src_st, const void *src_ptr, const axe_layout *dst,
                    const axe_storage *dst_st, void *dst_ptr, int elem_size, void *cuda_stream);

/* ------------------------------------------------------------------------- */
/* Redistribution across the device axis "gpuid"       */
/* ------------------------------------------------------------------------- */

typedef struct axe_comm axe_comm;

/* 128-byte NCCL unique id, created on one rank and broadcast by the caller. */
axe_status axe_get_unique_id(uint8_t out[128]);
/* Collective over nranks processes, one device each (cuda_device). */
axe_status axe_comm_create(const uint8_t id[128], int nranks, int rank, int cuda_device, axe_comm **out);
void axe_comm_destroy(axe_comm *comm);
/* Wait on the host until every operation enqueued on cuda_stream so far has finished, polling the
 * communicator's asynchronous NCCL error state (ncclCommGetAsyncError) every 50 us.  On an
 * asynchronous error (AXE_ERR_NCCL) or when timeout_ms (< 0: no limit) passes first
 * (AXE_ERR_TIMEOUT), the communicator is aborted (ncclCommAbort: the NCCL kernels waiting on a
 * failed peer return) and every later call on it fails with AXE_ERR_NCCL; destroy it and create a
 * new one.  Every execute on a communicator also checks the asynchronous error before and after its
 * enqueue.  Executes of one plan are serialised: on the host, and on the device each waits for the
 * previous execute of the same plan (they share its staging buffers). */
axe_status axe_comm_wait(axe_comm *comm, void *cuda_stream, int timeout_ms);

/* CUDA IPC for the one-sided forms (axe_redist_plan_execute_peers / _peers_reduce) between processes
 * of one node: export writes a 128-byte handle for the device allocation holding dev_ptr (the
 * cudaIpcMemHandle_t of the allocation + dev_ptr's byte offset in it, so sub-allocated framework
 * tensors work); import maps a handle exported by ANOTHER process (same or another GPU; peer access
 * is enabled lazily) and returns the pointer to use in dst_peers / src_peers; close unmaps it.
 * Errors: AXE_ERR_INVALID_ARG (not a device allocation / not an imported pointer), AXE_ERR_CUDA
 * (the driver refused, e.g. importing a handle of the same process). */
axe_status axe_ipc_export(const void *dev_ptr, uint8_t handle[128]);
axe_status axe_ipc_import(const uint8_t handle[128], void **dev_ptr);
axe_status axe_ipc_close(void *dev_ptr);

typedef struct axe_redist_plan axe_redist_plan;

/* Plan rank `rank`'s part of a redistribution (host only): the layouts describe
 * the global tensor; their "gpuid" coordinate names the rank, and the storages
 * describe the non-gpuid axes of each rank's local buffer.  Every rank must
 * plan with identical arguments (except rank).  For each destination cell the
 * source owner is the local rank when it holds the element, else one owner
 * chosen to balance egress (R5). */
axe_status axe_redist_plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                  const axe_storage *dst_st, int elem_size, int nranks, int rank,
                                  axe_redist_plan **out);
/* Collective launch: pack kernels, NCCL exchange over the comm, unpack kernels
 * and the local copy, all ordered on cuda_stream. src_local/dst_local are this
 * rank's device buffers. */
axe_status axe_redist_plan_execute(const axe_redist_plan *plan, axe_comm *comm, const void *src_local,
                                   void *dst_local, void *cuda_stream);
/* One-sided form: every block this rank sends is ONE copy kernel reading
 * src_local and writing straight into the receiver's destination buffer
 * dst_peers[receiver] (peer memory mapped into this process, e.g. CUDA IPC or
 * torch symmetric memory; dst_peers[rank] is this rank's own dst_local) -- the
 * pack, the NVLink transfer and the unpack fused.  The caller orders it across
 * ranks: every peer's dst buffer must be ready before (a barrier) and is
 * complete only after every rank's launches finished (a barrier after). */
axe_status axe_redist_plan_execute_peers(const axe_redist_plan *plan, const void *src_local, void *const *dst_peers,
                                         void *cuda_stream);
/* JSON description: pattern (allgather / exchange / local), per-peer element
 * counts and the kernels used. */
axe_status axe_redist_plan_describe(const axe_redist_plan *plan, char *buf, int capacity);
/* Host-side view of the plan for tests: for peer p, *send = elements this rank
 * sends to p, *recv = elements it receives from p (p == rank: both are the
 * number of elements copied locally). */
axe_status axe_redist_plan_counts(const axe_redist_plan *plan, int peer, int64_t *send, int64_t *recv);
/* Host-side view for tests, element k in wire order:
 *   kind 0 (send to peer, k < send count): *a = source element index in this
 *          rank's src_local storage (before the storage swizzle), *b = -1;
 *   kind 1 (receive from peer, k < recv count): *a = destination element index
 *          in this rank's dst_local (the first destination replica), *b = -1;
 *   kind 2 (local copy, k < counts(rank)): *a = source element, *b = destination
 *          element (first replica).
 * A sender's k-th element to p is the receiver's k-th element from the sender. */
axe_status axe_redist_plan_map(const axe_redist_plan *plan, int kind, int peer, int64_t k, int64_t *a, int64_t *b);
void axe_redist_plan_destroy(axe_redist_plan *plan);

/* One-shot collective redistribute (plans through an internal cache). */
axe_status axe_redistribute(const axe_layout *src, const axe_storage *src_st, const void *src_local,
                            const axe_layout *dst, const axe_storage *dst_st, void *dst_local, int elem_size,
                            axe_comm *comm, void *cuda_stream);

/* Single-device emulation of a whole redistribution for tests: runs every
 * rank's plan (plans[g] planned with rank g) on the current device, with the
 * NCCL exchange replaced by device-to-device copies between the ranks'
 * staging buffers.  src_locals[g] / dst_locals[g] are device buffers. */
axe_status axe_redist_emulate(const axe_redist_plan *const *plans, int nranks, const void *const *src_locals,
                              void *const *dst_locals, void *cuda_stream);

/* ------------------------------------------------------------------------- */
/* Reduction over the leading logical dimension              */
/* ------------------------------------------------------------------------- */
/* a reduce-scatter "accepts a DTensor with shape (4, 64, 64) that
 * shards over the first dimension, and sums over 0, generating an output
 * DTensor with shape (64, 64)"; "invokes the sum operator".  Reading R24
 * (DESIGN.md): with K = E_D(src) / E_D(dst) (an integer, else
 * AXE_ERR_SIZE_MISMATCH),
 *     dst(y) = sum_{k=0}^{K-1} src(k * E_D(dst) + y)   for every y in [0, E_D(dst)),
 * the source element of x read at its representative f_D(x) + O (R4) and the
 * sum written to every cell of f_L^dst(y); other dst cells are untouched.
 * Floating point: summed in fp32 (fp64 for AXE_DTYPE_F64) in k order and
 * rounded once to the element type (round to nearest even); integers add
 * modulo 2^bits.  Elements are dtype-sized; storages as for copies. */
enum {
  AXE_DTYPE_F32 = 1,
  AXE_DTYPE_F64 = 2,
  AXE_DTYPE_F16 = 3,
  AXE_DTYPE_BF16 = 4,
  AXE_DTYPE_I32 = 5,
  AXE_DTYPE_I64 = 6
};

typedef struct axe_reduce_plan axe_reduce_plan;

/* Plan a one-device reduction (host only).  Errors: AXE_ERR_INVALID_ARG (unknown
 * dtype), AXE_ERR_SIZE_MISMATCH, AXE_ERR_BOUNDS, AXE_ERR_NONINJECTIVE,
 * AXE_ERR_UNSUPPORTED_AXIS (gpuid: use axe_redist_reduce_plan_create). */
axe_status axe_reduce_plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                  const axe_storage *dst_st, int dtype, axe_reduce_plan **out);
/* Launch on cuda_stream (asynchronous, 1 kernel).  src_ptr / dst_ptr: DEVICE
 * buffers of the storage sizes, owned by the caller, not overlapping
 * (AXE_ERR_ALIAS); aligned to the plan's vector width (AXE_ERR_ALIGNMENT). */
axe_status axe_reduce_plan_execute(const axe_reduce_plan *plan, const void *src_ptr, void *dst_ptr, void *cuda_stream);
axe_status axe_reduce_plan_sizes(const axe_reduce_plan *plan, int64_t *src_bytes, int64_t *dst_bytes);
/* JSON: kernel (reduce | reduce_generic), K, vector bytes, output / reduction digits. */
axe_status axe_reduce_plan_describe(const axe_reduce_plan *plan, char *buf, int capacity);
void axe_reduce_plan_destroy(axe_reduce_plan *plan);
/* One-shot form through an internal plan cache. */
axe_status axe_reduce(const axe_layout *src, const axe_storage *src_st, const void *src_ptr, const axe_layout *dst,
                      const axe_storage *dst_st, void *dst_ptr, int dtype, void *cuda_stream);

/* Distributed form (Partial -> Shard = reduce-scatter, Partial -> Replicate =
 * all-reduce): the layouts name "gpuid" as for axe_redist_plan_create, and the
 * source's summed dimension is typically sharded over gpuid (one partial per
 * rank).  Executed as an exchange of the partials into a library-owned stage
 * buffer (K slabs shaped like this rank's dst storage; pack / NCCL / unpack as
 * axe_redist_plan_execute) followed by one K4 sum of the slabs into dst_local.
 * Every rank's destination image must be its whole dst storage
 * (AXE_ERR_UNSUPPORTED otherwise).  A destination replicated over >= 3 ranks
 * is planned in two phases instead: a reduce-scatter (as above) into an even
 * shard (nranks, E_D(dst)/nranks):(1@gpuid, 1@m), then a plain redistribution
 * of that shard into the destination (an all-gather for a row-major replicated
 * destination) -- describe() says "reduce_scatter_allgather" and
 * axe_redist_plan_phase returns the two sub-plans.  The returned plan is used
 * with axe_redist_plan_execute / _describe / _counts / _map (stage element
 * indices; two-phase plans: query the phases) / _destroy and
 * axe_redist_emulate; not with _execute_peers. */
axe_status axe_redist_reduce_plan_create(const axe_layout *src, const axe_storage *src_st, const axe_layout *dst,
                                         const axe_storage *dst_st, int dtype, int nranks, int rank,
                                         axe_redist_plan **out);
/* One-sided pull form of a single-phase reduction plan (SURVEY §8(f) f2 + f3):
 * src_peers[r] is rank r's source buffer mapped into this process (peer memory
 * over NVLink: torch symmetric memory / CUDA IPC; src_peers[rank] = this rank's
 * own).  Each destination region is ONE kernel that reads its K partials
 * straight from the owners' buffers and writes the sum into dst_local -- the
 * exchange, the staging and the sum fused.  The caller orders it across ranks
 * (every src ready before: a barrier; no src reuse until every rank finished:
 * a barrier after).  AXE_ERR_UNSUPPORTED for two-phase plans, more than 256
 * summands, destination memory replicas, or blocks that straddle stage slabs
 * (describe(): "pull_regions" = 0). */
axe_status axe_redist_plan_execute_peers_reduce(const axe_redist_plan *plan, const void *const *src_peers,
                                                void *dst_local, void *cuda_stream);
/* NVLS form of the same (the paper's reduce-scatter "dispatch[es] to
 * multimem.ld_reduce on B200"): src_multicast is the multicast address of the
 * ranks' source buffers (an NVSwitch multicast object bound to every rank's
 * src, e.g. torch symmetric memory's multicast_ptr).  Every 16-byte output
 * vector is one multimem.ld_reduce -- the switch sums the vector over all
 * ranks -- stored into dst_local.  Requires each region to take exactly one
 * partial from every rank at the same offset (describe(): "multicast": true),
 * f32 / bf16 / f16 (bf16 / f16 accumulate in f32 inside the switch; the
 * summation order is the hardware's).  Same cross-rank ordering contract as
 * axe_redist_plan_execute_peers_reduce. */
axe_status axe_redist_plan_execute_multicast_reduce(const axe_redist_plan *plan, const void *src_multicast,
                                                    void *dst_local, void *cuda_stream);
/* Phase i (0: reduce-scatter, 1: gather) of a two-phase reduction plan; the
 * sub-plan is owned by `plan` (do not destroy it).  AXE_ERR_UNSUPPORTED for
 * any other plan. */
axe_status axe_redist_plan_phase(const axe_redist_plan *plan, int i, const axe_redist_plan **out);
/* One-shot collective form (plans through an internal cache). */
axe_status axe_redistribute_reduce(const axe_layout *src, const axe_storage *src_st, const void *src_local,
                                   const axe_layout *dst, const axe_storage *dst_st, void *dst_local, int dtype,
                                   axe_comm *comm, void *cuda_stream);

/* ------------------------------------------------------------------------- */
const char *axe_last_error(void);
/* Number of kernels this library has launched in this process (all threads). */
int64_t axe_kernel_launch_count(void);
const char *axe_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AXE_H_ */
