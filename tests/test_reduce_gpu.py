"""GPU parity of the reduction row (reading R24): K4 on one device
(axe_reduce / ReducePlan) and the distributed reduce-redistribute (emulated on one
B200, and through a 1-rank NCCL communicator), against oracle.reduce.

Inputs (synth.numbers "wide"): random signs, exponents over the whole range of the type
(binary16: subnormals up to 65504; bf16 / f32: subnormals up to 2^110; f64: up to 2^900),
so sums mix terms hundreds of binades apart, cancel, and overflow binary16.

Tolerance (DESIGN.md §3 R24), element by element: the kernel adds the K summands in k
order in fp32 (fp64 for f64) and rounds once to the type; the oracle sums in fp64 and
rounds once.  With A = sum_k |x_k| (the oracle's fp64 sum of the absolute values, on the
same layouts), u_a the accumulator's unit roundoff (2^-24, 2^-53 for f64), gamma =
(K-1) u_a / (1 - (K-1) u_a) (Higham's bound for K-1 sequential additions), u_T the output
type's unit roundoff and eta_T half its smallest subnormal:

    |got - exp| <= gamma A + K 2^-53 A + u_T (1 + 2 u_T) (|got| + |exp|) + 2 eta_T

(the fp32 sum is within gamma A of the exact sum, the oracle's fp64 sum within K 2^-53 A,
and each side's final rounding moves its value by at most u_T of it or eta_T in the
subnormal range).  No accumulator overflow is possible on these inputs (K <= 256 terms
below 2^111 in fp32), so the only infinities are binary16 overflows: where one side is
+-inf the other must be the same infinity or the largest finite value of that sign (the
exact sum lies within the bound of the overflow threshold 65520).  Integers, and
bf16 / f16 sums whose fp32 partial sums are exact ("narrow" inputs), are bit-exact."""
import os

import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage, storage

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
NT = os.cpu_count() or 4
FLOAT = {"f16": (np.float16, np.uint16), "bf16": (None, np.uint16), "f32": (np.float32, np.uint32),
         "f64": (np.float64, np.uint64)}
U_ACC = {"f16": 2.0 ** -24, "bf16": 2.0 ** -24, "f32": 2.0 ** -24, "f64": 2.0 ** -53}
U_OUT = {"f16": 2.0 ** -11, "bf16": 2.0 ** -8, "f32": 2.0 ** -24, "f64": 2.0 ** -53}
ETA = {"f16": 2.0 ** -25, "bf16": 2.0 ** -134, "f32": 2.0 ** -150, "f64": 0.0}
MAXF = {"f16": 65504.0}


def to_f64(b, dtype):
    """Raw bytes of `dtype` -> float64 values (exact conversions)."""
    if dtype == "bf16":
        return (b.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return b.view(FLOAT[dtype][0]).astype(np.float64)


def abs_sums(cfg, vals, dtype, nranks=None):
    """A = sum_k |x_k| per destination cell (f64; NaN in cells outside the image), from the LOGICAL
    summands vals (x = k * E_D(dst) + y, R24) -- only the tolerance's magnitude, not an expected value.
    Placing A[y] on the destination storage needs the cell of every y: the oracle scatters the index y
    itself (in es-byte pieces, so the storage swizzle sees the same element size as the data) into the
    destination layout; a never-written cell keeps the all-ones fill."""
    es = synth.DTYPE_SIZE[dtype]
    ed, _ = oracle.sizes(cfg["dst"])
    K = len(vals) // es // ed
    Al = np.abs(to_f64(vals, dtype)).reshape(K, ed).sum(axis=0)
    y = np.arange(ed, dtype=np.uint64)
    cells = synth.storage_cells(cfg["dst_st"])
    fill = np.full(cells * es, 0xFF, np.uint8)
    pieces = 1 if es >= 4 else 2   # 16-bit pieces of y for 2-byte elements
    ut = {2: np.uint16, 4: np.uint32, 8: np.uint64}[es]
    idx = None
    for p in range(pieces):
        part = ((y >> np.uint64(16 * p)) & np.uint64(0xFFFF)) if pieces == 2 else y
        vb = part.astype(ut).view(np.uint8)
        if nranks is None:
            got = [oracle.scatter_logical(cfg["dst"], cfg["dst_st"], vb, es, fill, NT)]
        else:
            got = oracle.scatter_ranks(cfg["dst"], cfg["dst_st"], vb, es, nranks, fill, NT)
        got = [g.view(ut).astype(np.uint64) for g in got]
        idx = got if idx is None else [i | (g << np.uint64(16)) for i, g in zip(idx, got)]
    allones = np.uint64(0xFFFFFFFF) if pieces == 2 else np.uint64(np.iinfo(ut).max)
    out = []
    for i in idx:
        a = np.full(cells, np.nan)
        w = i != allones
        a[w] = Al[i[w].astype(np.int64)]
        out.append(a)
    return out[0] if nranks is None else out


def compare(got, exp, fill, dtype, K, A=None):
    """got (kernel) against exp (oracle), R24's bound per element; exact for integers or A is None."""
    if dtype not in FLOAT or A is None:
        assert np.array_equal(got, exp)
        return
    ut = FLOAT[dtype][1]
    untouched = np.isnan(A)
    assert np.array_equal(exp.view(ut)[untouched], fill.view(ut)[untouched]), "oracle wrote outside the image"
    assert np.array_equal(got.view(ut)[untouched], exp.view(ut)[untouched]), "cells outside the image changed"
    g, e, a = to_f64(got, dtype)[~untouched], to_f64(exp, dtype)[~untouched], A[~untouched]
    assert not np.isnan(g).any() and not np.isnan(e).any(), "NaN in a sum of finite summands"
    inf = np.isinf(g) | np.isinf(e)
    if inf.any():
        assert dtype in MAXF, "only binary16 sums can overflow on these inputs"
        gi, ei = g[inf], e[inf]
        same = gi == ei
        edge = (np.isinf(gi) & (ei == np.sign(gi) * MAXF[dtype])) | (np.isinf(ei) & (gi == np.sign(ei) * MAXF[dtype]))
        assert np.all(same | edge), f"{(~(same | edge)).sum()} overflows disagree"
    g, e, a = g[~inf], e[~inf], a[~inf]
    ua = U_ACC[dtype]
    gamma = (K - 1) * ua / (1 - (K - 1) * ua)
    uo = U_OUT[dtype]
    tol = gamma * a + K * 2.0 ** -53 * a + uo * (1 + 2 * uo) * (np.abs(g) + np.abs(e)) + 2 * ETA[dtype]
    bad = np.abs(g - e) > tol
    assert not bad.any(), (f"{bad.sum()} of {len(g)} elements outside the bound, worst excess "
                           f"{(np.abs(g - e) - tol).max()}")


@pytest.fixture(scope="module")
def axe():
    assert torch.cuda.is_available()
    import paper_2601_19092_b200 as m
    return m


def guard(nbytes, seed):
    """Device buffer with 4 KiB sentinel guards on both sides (compute-sanitizer is closed on the pool)."""
    g = 4096
    buf = torch.from_numpy(synth.sentinel(nbytes + 2 * g, seed)).cuda()
    return buf, buf[g:g + nbytes]


def check_guards(buf, nbytes, seed):
    g = 4096
    ref = synth.sentinel(nbytes + 2 * g, seed)
    h = buf.cpu().numpy()
    assert np.array_equal(h[:g], ref[:g]) and np.array_equal(h[g + nbytes:], ref[g + nbytes:]), "guard overwritten"


def run_local(axe, cfg, dtype, seed=7, one_shot=False, dist="wide", vals=None):
    """dist "narrow" (exact fp32 partial sums) is compared bit for bit, everything else with R24's bound."""
    es = synth.DTYPE_SIZE[dtype]
    ed, _ = oracle.sizes(cfg["src"])
    edd, _ = oracle.sizes(cfg["dst"])
    K = ed // edd
    if vals is None:
        vals = synth.numbers(ed, dtype, seed, dist)
    sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, seed + 1)
    sbuf = oracle.scatter_logical(cfg["src"], cfg["src_st"], vals, es, sfill, NT)
    dbytes = synth.storage_cells(cfg["dst_st"]) * es
    dfill = synth.sentinel(dbytes, seed + 2)
    exp = dfill.copy()
    oracle.reduce(cfg["src"], cfg["src_st"], sbuf, cfg["dst"], cfg["dst_st"], exp, dtype, nthreads=NT)
    s_dev = torch.from_numpy(sbuf).cuda()
    gbuf, d_dev = guard(dbytes, seed + 2 - 1)
    d_dev.copy_(torch.from_numpy(dfill))
    n0 = axe.kernel_launch_count()
    if one_shot:
        axe.axe_reduce(cfg["src"], cfg["src_st"], s_dev, cfg["dst"], cfg["dst_st"], d_dev, dtype)
        desc = None
    else:
        plan = axe.ReducePlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], dtype)
        assert plan.sizes() == (sbuf.nbytes, dbytes)
        plan.execute(s_dev, d_dev)
        desc = plan.describe()
    torch.cuda.synchronize()
    assert axe.kernel_launch_count() - n0 == 1
    check_guards(gbuf, dbytes, seed + 1)
    A = None if dist == "narrow" or dtype not in FLOAT else abs_sums(cfg, vals, dtype)
    compare(d_dev.cpu().numpy(), exp, dfill, dtype, K, A)
    return desc


@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32", "f64", "i32", "i64"])
def test_leading_dim_sum_row_major(axe, dtype):
    d = run_local(axe, synth.reduce_local(8, 96, 200, dtype), dtype)
    assert d["kernel"] == "reduce" and d["K"] == 8


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_sum_into_swizzled_tiles(axe, dtype):
    """The reduction fused with config 2's re-tiling: 64x64 tiles + SW128 destination."""
    d = run_local(axe, synth.reduce_local(4, 256, 512, dtype, tiled=True), dtype)
    assert d["kernel"] == "reduce" and d["vec_bytes"] == 16


def tiled_reduce_cfg(K, rows, cols, dtype, reps=1):
    """(K, rows, cols) row-major -> (rows, cols) in t x t tiles with the 128-byte swizzle, t = 128 bytes of
    elements (one SW128 atom row per tile row), optionally `reps` destination replicas."""
    es = synth.DTYPE_SIZE[dtype]
    t = 128 // es
    src = layout([(K, rows * cols), (rows, cols), (cols, 1)])
    R = [(reps, rows * cols)] if reps > 1 else []
    dst = layout([(rows // t, t * cols), (t, t), (cols // t, t * t), (t, 1)], R)
    return dict(src=src, src_st=linear_storage(K * rows * cols), dst=dst,
                dst_st=linear_storage(reps * rows * cols, synth.SW128))


@pytest.mark.parametrize("K,dtype,reps", [(2, "bf16", 1), (3, "f16", 1), (5, "f32", 1), (8, "bf16", 2), (8, "f64", 1),
                                          (4, "i32", 1), (6, "i64", 1), (7, "bf16", 1)])
def test_sum_into_swizzled_tiles(axe, K, dtype, reps):
    """The reduction fused with config 2's re-tiling: the sums land in 64-row SW128 tiles (the swizzle folded
    into the per-thread destination offsets), one store per replica."""
    es = synth.DTYPE_SIZE[dtype]
    rows, cols = 128 * (2 if es <= 4 else 1), 128 // es * 6
    d = run_local(axe, tiled_reduce_cfg(K, rows, cols, dtype, reps), dtype, seed=K * 3 + es)
    assert d["kernel"] == "reduce" and d["mode"] == "vector", d


@pytest.mark.parametrize("K,dtype,rows,cols,ld,reps", [
    (2, "bf16", 64, 512, 512, 1), (3, "f32", 48, 1024, 1040, 1), (8, "f16", 32, 2048, 2048, 2), (5, "f64", 16, 256, 264, 1),
    (4, "i32", 40, 1024, 1028, 1), (8, "bf16", 96, 4096, 4096, 1), (7, "i64", 8, 512, 512, 3)])
@pytest.mark.parametrize("chunk", ["", "3"])
def test_padded_rows_and_replicas(axe, K, dtype, rows, cols, ld, reps, chunk, monkeypatch):
    """Whole or padded rows (ld > cols) summed into a replicated destination, with the persistent grid or the
    in-order schedule forced to 3 blocks per CTA (a ragged last CTA)."""
    monkeypatch.setenv("AXE_CHUNK", chunk)
    src = layout([(K, rows * ld), (rows, ld), (cols, 1)])
    dst = layout([(rows, cols), (cols, 1)], [(reps, rows * cols)] if reps > 1 else [])
    cfg = dict(src=src, src_st=linear_storage(K * rows * ld), dst=dst, dst_st=linear_storage(reps * rows * cols))
    d = run_local(axe, cfg, dtype, seed=K * 5 + rows)
    assert d["kernel"] == "reduce" and d["mode"] == "vector" and d["replicas"] == reps, d


@pytest.mark.parametrize("K,dtype,tiled", [(8, "f32", False), (2, "bf16", False), (8, "bf16", True)])
def test_in_order_schedule_matches_persistent_bitwise(axe, K, dtype, tiled, monkeypatch):
    """The in-order schedule (max(1, 8 / K) blocks of 256 vectors per CTA over a covering grid) changes which
    CTA sums which outputs, never the arithmetic: bit for bit the persistent grid's result, at a size where
    AUTO takes it (4096+ blocks)."""
    rows, cols = (2048, 2048) if dtype == "f32" else (2048, 4096)
    cfg = synth.reduce_local(K, rows, cols, dtype, tiled=tiled)
    vals = synth.numbers(K * rows * cols, dtype, 78 + K)
    s = torch.from_numpy(vals.copy()).cuda()
    outs = []
    for chunk in ("", "0"):
        monkeypatch.setenv("AXE_CHUNK", chunk)
        p = axe.ReducePlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], dtype)
        o = torch.zeros(rows * cols * synth.DTYPE_SIZE[dtype] // 2, dtype=torch.int16, device="cuda")
        p.execute(s, o)
        torch.cuda.synchronize()
        outs.append(o.cpu().numpy())
        assert p.describe()["chunk"] == (max(1, 8 // K) if chunk == "" else 0)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("K", [1, 2, 3, 17, 300])
def test_k_values(axe, K):
    """K = 1 (a copy), odd K (tail of the 8-wide load batch), K > 256 (decoded summand offsets)."""
    dtype = "f16" if K <= 32 else "i32"
    d = run_local(axe, synth.reduce_local(K, 8, 96, dtype), dtype)
    assert d["table"] == (K <= 256)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_exact_when_partial_sums_are_exact(axe, dtype):
    """On "narrow" summands (|x| in [2^-8, 1), every fp32 partial sum of K <= 32 exact) the kernel's one
    rounding and the oracle's one rounding see the same exact value: bit-exact."""
    run_local(axe, synth.reduce_local(16, 64, 256, dtype), dtype, dist="narrow")


@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32", "f64"])
def test_cancellation(axe, dtype):
    """Summand 1 = -summand 0 in every output (synth.cancelling): the result is small against A."""
    K, R, C = 6, 64, 128
    run_local(axe, synth.reduce_local(K, R, C, dtype), dtype,
              vals=synth.cancelling(K, R * C, dtype, 61))


@pytest.mark.parametrize("K", [2, 4, 8])
def test_f16_sums_around_the_largest_finite(axe, K):
    """Summands from the top 4 binades of binary16 (4096 .. 65504), mixed signs: sums straddle 65504 and
    overflow to +-inf on both sides (R24's overflow rule at the threshold 65520)."""
    cfg = synth.reduce_local(K, 64, 512, "f16")
    run_local(axe, cfg, "f16", vals=synth.numbers(K * 64 * 512, "f16", 62 + K, "top"))


def test_interleaved_summands_and_transposed_destination(axe):
    """Summands innermost in memory (src (Y, K) storage order) into a column-major padded destination."""
    K, R, C, ld = 6, 40, 24, 48
    src = layout([(K, 1), (R, C * K), (C, K)])
    dst = layout([(R, 1), (C, ld)])
    cfg = dict(src=src, src_st=linear_storage(K * R * C), dst=dst, dst_st=linear_storage(C * ld))
    run_local(axe, cfg, "bf16")


def test_replicas_and_offsets(axe):
    """Source replicas (read at the representative) and destination replicas + offset on named axes."""
    K, N = 4, 256
    src = layout([(K, N), (N, 1)], [(2, K * N)])
    dst = layout([(N // 32, 1, "warp"), (32, 1, "lane")], [(2, 8, "warp")], {"warp": 1})
    cfg = dict(src=src, src_st=linear_storage(2 * K * N), dst=dst, dst_st=storage([("warp", 17), ("lane", 32)]))
    d = run_local(axe, cfg, "f32")
    assert d["replicas"] == 2


def test_generic_fallback(axe):
    """Digit systems that do not nest: the source is a column-major 30x7 matrix (K = 6 blocks of 35), the
    destination a 7x5 matrix with rows padded to 8 -- innermost extents 7 and 5 share no divisor -> k4_generic."""
    src = layout([(30, 1), (7, 30)])
    dst = layout([(7, 8), (5, 1)])
    cfg = dict(src=src, src_st=linear_storage(210), dst=dst, dst_st=linear_storage(56))
    d = run_local(axe, cfg, "f32")
    assert d["kernel"] == "reduce_generic"


def test_one_shot_cached(axe):
    cfg = synth.reduce_local(3, 32, 64, "bf16")
    run_local(axe, cfg, "bf16", one_shot=True)
    run_local(axe, cfg, "bf16", seed=9, one_shot=True)


def test_bench_workload_full_size(axe):
    """bench.py's reduce row at full size: (8, 8192, 4096) bf16 -> (8192, 4096), every element."""
    d = run_local(axe, synth.reduce_local(8, 8192, 4096, "bf16"), "bf16")
    assert d["vec_bytes"] == 16


def test_errors(axe):
    with pytest.raises(axe.AxeError) as e:
        axe.ReducePlan(layout([(30, 1)]), linear_storage(30), layout([(7, 1)]), linear_storage(7), "f32")
    assert e.value.name == "AXE_ERR_SIZE_MISMATCH"
    x = torch.zeros(64, dtype=torch.float32, device="cuda")
    plan = axe.ReducePlan(layout([(2, 32), (32, 1)]), linear_storage(64), layout([(32, 1)]), linear_storage(32), "f32")
    with pytest.raises(axe.AxeError) as e:
        plan.execute(x, x[8:])
    assert e.value.name == "AXE_ERR_ALIAS"


# ------------------------------------------------------------------ distributed


def run_dist(axe, cfg, dtype, seed=21):
    n, es = cfg["nranks"], synth.DTYPE_SIZE[dtype]
    ed, _ = oracle.sizes(cfg["src"])
    edd, _ = oracle.sizes(cfg["dst"])
    K = ed // edd
    vals = synth.numbers(ed, dtype, seed, "wide")
    sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, seed + 1)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], vals, es, n, sfill, NT)
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, seed + 2)
    exp = [dfill.copy() for _ in range(n)]
    oracle.reduce(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, dtype, nranks=n, nthreads=NT)
    plans = [axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, n, r, reduce_dtype=dtype)
             for r in range(n)]
    s_dev = [torch.from_numpy(s).cuda() for s in src]
    d_dev = [torch.from_numpy(dfill).cuda() for _ in range(n)]
    axe.redist_emulate(plans, s_dev, d_dev)
    torch.cuda.synchronize()
    A = abs_sums(cfg, vals, dtype, n) if dtype in FLOAT else [None] * n
    for r in range(n):
        compare(d_dev[r].cpu().numpy(), exp[r], dfill, dtype, K, A[r])
    return plans[0].describe()


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_reduce_scatter_emulated(axe, P, dtype):
    """The DTensor reduce-scatter of P:399-403 ((P, 64, 64) partials summed over dim 0, rows sharded)."""
    d = run_dist(axe, synth.reduce_scatter(P, 64, 64, dtype), dtype)
    assert d["pattern"] == "reduce" and d["K"] == P


def test_reduce_scatter_emulated_large(axe):
    d = run_dist(axe, synth.reduce_scatter(8, 1024, 2048, "bf16"), "bf16")
    assert d["exchange"]["packs"] == 0


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_all_reduce_emulated(axe, P, dtype):
    """Partial -> Replicate: one exchange at P = 2, reduce-scatter + all-gather (two phases) at P >= 3."""
    d = run_dist(axe, synth.all_reduce(P, 32, 128, dtype), dtype)
    assert d["pattern"] == ("reduce" if P == 2 else "reduce_scatter_allgather")


def test_mesh_partial_over_one_axis(axe):
    """2x2 mesh (gpuid = 2a + b): partials over a, replicated over b -> summed, sharded by rows over b,
    replicated over a."""
    R, C = 64, 32
    src = layout([(2, 2, "gpuid"), (R, C), (C, 1)], [(2, 1, "gpuid")])
    dst = layout([(2, 1, "gpuid"), (R // 2, C), (C, 1)], [(2, 2, "gpuid")])
    cfg = dict(nranks=4, src=src, src_st=linear_storage(R * C), dst=dst, dst_st=linear_storage(R // 2 * C))
    run_dist(axe, cfg, "f32")


def test_transposed_shard_emulated(axe):
    """Partials row-major, destination column shards stored column-major (pack + unpack kernels)."""
    P, R, C = 4, 32, 64
    src = layout([(P, 1, "gpuid"), (R, C), (C, 1)])
    dst = layout([(R, 1), (P, 1, "gpuid"), (C // P, R)])
    cfg = dict(nranks=P, src=src, src_st=linear_storage(R * C), dst=dst, dst_st=linear_storage(R * C // P))
    run_dist(axe, cfg, "bf16")


def test_nccl_single_rank_reduce(axe):
    """The NCCL path on one GPU: both partials on rank 0 (K = 2), axe_redistribute_reduce through a 1-rank
    communicator, against the oracle."""
    comm = axe.Comm(axe.get_unique_id(), 1, 0, torch.cuda.current_device())
    K, R, C = 2, 64, 96
    src = layout([(K, R * C), (R, C), (C, 1)])
    dst = layout([(R, C), (C, 1)], [(1, 1, "gpuid")])
    vals = synth.numbers(K * R * C, "bf16", 3, "narrow")   # exact: compared bit for bit
    x = torch.from_numpy(vals.copy()).cuda()
    y = torch.zeros(R * C * 2, dtype=torch.uint8, device="cuda")
    axe.axe_redistribute_reduce(src, linear_storage(K * R * C), x, dst, linear_storage(R * C), y, "bf16", comm)
    torch.cuda.synchronize()
    exp = np.zeros(R * C * 2, np.uint8)
    oracle.reduce(src, linear_storage(K * R * C), [vals], dst, linear_storage(R * C), [exp], "bf16", nranks=1)
    assert np.array_equal(y.cpu().numpy(), exp)


# ------------------------------------------------------------------ one-sided pull form
def run_pull(axe, cfg, dtype, seed=31):
    """Every rank's pull plan on one device: the 'peer' table holds the ranks' separate source buffers (on a
    multi-GPU box these are NVLink-mapped peer buffers; the kernel only sees pointers)."""
    n, es = cfg["nranks"], synth.DTYPE_SIZE[dtype]
    ed, _ = oracle.sizes(cfg["src"])
    edd, _ = oracle.sizes(cfg["dst"])
    K = ed // edd
    vals = synth.numbers(ed, dtype, seed, "wide")
    sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, seed + 1)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], vals, es, n, sfill, NT)
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, seed + 2)
    exp = [dfill.copy() for _ in range(n)]
    oracle.reduce(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, dtype, nranks=n, nthreads=NT)
    A = abs_sums(cfg, vals, dtype, n) if dtype in FLOAT else [None] * n
    s_dev = [torch.from_numpy(s).cuda() for s in src]
    d_dev = [torch.from_numpy(dfill).cuda() for _ in range(n)]
    n0 = axe.kernel_launch_count()
    descs = []
    for r in range(n):
        p = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, n, r, reduce_dtype=dtype)
        d = p.describe()
        descs.append(d)
        p.execute_peers_reduce(s_dev, d_dev[r])
    torch.cuda.synchronize()
    assert axe.kernel_launch_count() - n0 == sum(d["pull_regions"] for d in descs)
    for r in range(n):
        compare(d_dev[r].cpu().numpy(), exp[r], dfill, dtype, K, A[r])
    return descs[0]


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["bf16", "f32", "i32"])
def test_pull_reduce_scatter(axe, P, dtype):
    """P:399-403 reduce-scatter as one kernel per rank reading every partial from its owner."""
    d = run_pull(axe, synth.reduce_scatter(P, 128, 256, dtype), dtype)
    assert d["pull_regions"] == 1 and d["pull_vec_bytes"] == 16


def test_pull_transposed_shard(axe):
    """Column shards stored column-major: one region per rank, 2-byte vectors (no shared contiguous run)."""
    P, R, C = 4, 32, 64
    src = layout([(P, 1, "gpuid"), (R, C), (C, 1)])
    dst = layout([(R, 1), (P, 1, "gpuid"), (C // P, R)])
    cfg = dict(nranks=P, src=src, src_st=linear_storage(R * C), dst=dst, dst_st=linear_storage(R * C // P))
    run_pull(axe, cfg, "bf16")


def test_pull_mesh_partial_over_one_axis(axe):
    R, C = 64, 32
    src = layout([(2, 2, "gpuid"), (R, C), (C, 1)], [(2, 1, "gpuid")])
    dst = layout([(2, 1, "gpuid"), (R // 2, C), (C, 1)], [(2, 2, "gpuid")])
    cfg = dict(nranks=4, src=src, src_st=linear_storage(R * C), dst=dst, dst_st=linear_storage(R // 2 * C))
    run_pull(axe, cfg, "f32")


def test_pull_rejects_two_phase_plans(axe):
    cfg = synth.all_reduce(4, 32, 64, "bf16")
    p = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, 4, 0, reduce_dtype="bf16")
    x = torch.zeros(32 * 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(axe.AxeError) as e:
        p.execute_peers_reduce([x] * 4, x.clone())
    assert e.value.name == "AXE_ERR_UNSUPPORTED"
