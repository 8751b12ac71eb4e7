"""Pins for the oracle's reduction (oracle.reduce, reading R24).

Reading R24 (the DTensor reduce-scatter whose (4, 64, 64) input "sums
over 0" into a (64, 64) output): dst(y) = sum_k src(k * E_D(dst) + y), summed in
fp64 and rounded once to the element type; integers wrap.  Every expected value
here comes from numpy / torch CPU routines or from the IEEE-754 formats
themselves, never from the CUDA path.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import layout, linear_storage

NP = {"f16": np.float16, "f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64}


def as_float64(b: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return torch.from_numpy(b.view(np.int16).copy()).view(torch.bfloat16).double().numpy()
    return b.view(NP[dtype]).astype(np.float64)


def to_dtype_bytes(v: np.ndarray, dtype: str) -> np.ndarray:
    """float64 -> dtype with numpy's / torch's own conversion (round to nearest even)."""
    if dtype == "bf16":
        return torch.from_numpy(v).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint8)
    return v.astype(NP[dtype]).view(np.uint8)


def run_local(cfg, sbytes):
    es = synth.DTYPE_SIZE[cfg["dtype"]]
    out = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, 99)
    oracle.reduce(cfg["src"], cfg["src_st"], sbytes, cfg["dst"], cfg["dst_st"], out, cfg["dtype"])
    return out


@pytest.mark.parametrize("dtype", ["f16", "bf16", "f32", "f64"])
def test_sum_over_leading_dim_is_numpy_sum(dtype):
    """Row-major (K, R, C) -> (R, C): numpy's sum over axis 0 (sequential over the leading axis),
    cast once.  For f16 / bf16 / f32 summands in [2^-8, 1) the fp64 sums of K = 5 terms are exact,
    so the only rounding is the final cast, which numpy / torch perform independently."""
    K, R, Cc = 5, 24, 40
    cfg = synth.reduce_local(K, R, Cc, dtype)
    s = synth.numbers(K * R * Cc, dtype, 11, "narrow")
    got = run_local(cfg, s)
    exp = to_dtype_bytes(as_float64(s, dtype).reshape(K, R * Cc).sum(axis=0), dtype)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("dtype", ["i32", "i64"])
def test_integer_sums_wrap_like_numpy(dtype):
    K, R, Cc = 7, 16, 16
    cfg = synth.reduce_local(K, R, Cc, dtype)
    s = synth.numbers(K * R * Cc, dtype, 12)
    got = run_local(cfg, s)
    a = s.view(NP[dtype]).reshape(K, R * Cc)
    exp = a.sum(axis=0, dtype=NP[dtype])  # two's complement wrap-around
    assert np.array_equal(got.view(NP[dtype]), exp)


def test_f16_rounding_edges():
    """Final rounding to binary16 (IEEE-754): ties to even at 1 + 2^-11, overflow at 65520,
    the largest finite 65504, subnormal sums -- numpy's float16 cast decides each."""
    pairs = [(1.0, 2.0 ** -11), (1.0, 3 * 2.0 ** -11), (65504.0, 8.0), (65504.0, 16.0), (65504.0, 15.0 / 16 * 16),
             (2.0 ** -24, 2.0 ** -24), (2.0 ** -14, -2.0 ** -24), (-1.0, 1.0), (2048.0, 1.0), (2048.0, 3.0),
             (-65504.0, -32.0), (0.5, 2.0 ** -12)]
    a = np.array([p[0] for p in pairs], dtype=np.float16)
    b = np.array([p[1] for p in pairs], dtype=np.float16)
    assert np.all(a.astype(np.float64) == [p[0] for p in pairs]) and np.all(np.isfinite(b))
    n = len(pairs)
    cfg = synth.reduce_local(2, 1, n, "f16")
    s = np.concatenate([a, b]).view(np.uint8)
    got = run_local(cfg, s).view(np.float16)
    with np.errstate(over="ignore"):
        exp = (a.astype(np.float64) + b.astype(np.float64)).astype(np.float16)
    assert np.array_equal(got.view(np.uint16), exp.view(np.uint16))
    assert np.isinf(got[3]) and got[2] == 65504.0 and got[0] == 1.0


def test_bf16_rounding_edges():
    """Final rounding to bfloat16: ties to even, overflow past (2 - 2^-8) 2^127, subnormals;
    torch's float32 -> bfloat16 conversion decides (exact float32 sums)."""
    big = float(torch.finfo(torch.bfloat16).max)
    tiny = float(torch.finfo(torch.bfloat16).smallest_normal)
    pairs = [(1.0, 2.0 ** -8), (1.0, 3 * 2.0 ** -8), (big, 2.0 ** 118), (big, 2.0 ** 120), (tiny, -tiny / 2),
             (tiny / 128, tiny / 128), (-1.5, -2.0 ** -7), (3.0, 2.0 ** -7), (big, 2.0 ** 119)]
    a = torch.tensor([p[0] for p in pairs], dtype=torch.bfloat16)
    b = torch.tensor([p[1] for p in pairs], dtype=torch.bfloat16)
    assert a.double().tolist() == [p[0] for p in pairs] and b.double().tolist() == [p[1] for p in pairs]
    cfg = synth.reduce_local(2, 1, len(pairs), "bf16")
    s = torch.cat([a, b]).view(torch.int16).numpy().view(np.uint8)
    got = run_local(cfg, s)
    exp = (a.float() + b.float()).to(torch.bfloat16)  # the float32 sums are exact here
    assert np.array_equal(got.view(np.int16), exp.view(torch.int16).numpy())
    assert torch.isinf(exp[3]) and not torch.isinf(exp[2]) and torch.isinf(exp[8])  # 8: tie -> even = 2^128


def test_dtensor_reduce_scatter_example():
    """a (4, 64, 64) DTensor sharded over dim 0 on 4 devices, summed over dim 0 into a
    (64, 64) output sharded by rows: rank g holds rows [16 g, 16 g + 16) of numpy's sum."""
    P = 4
    cfg = synth.reduce_scatter(P, 64, 64, "f32")
    parts = [synth.numbers(64 * 64, "f32", 20 + g, "narrow") for g in range(P)]
    outs = [synth.sentinel(16 * 64 * 4, g) for g in range(P)]
    oracle.reduce(cfg["src"], cfg["src_st"], parts, cfg["dst"], cfg["dst_st"], outs, "f32", nranks=P)
    tot = np.stack([p.view(np.float32).astype(np.float64) for p in parts]).sum(axis=0).astype(np.float32)
    tot = tot.reshape(64, 64)
    for g in range(P):
        assert np.array_equal(outs[g].view(np.float32).reshape(16, 64), tot[16 * g:16 * g + 16])


def test_all_reduce_every_rank_holds_the_sum():
    P = 3
    cfg = synth.all_reduce(P, 8, 32, "bf16")
    parts = [synth.numbers(8 * 32, "bf16", 30 + g, "narrow") for g in range(P)]
    outs = [synth.sentinel(8 * 32 * 2, g) for g in range(P)]
    oracle.reduce(cfg["src"], cfg["src_st"], parts, cfg["dst"], cfg["dst_st"], outs, "bf16", nranks=P)
    tot = to_dtype_bytes(np.stack([as_float64(p, "bf16") for p in parts]).sum(axis=0), "bf16")
    for g in range(P):
        assert np.array_equal(outs[g], tot)


def test_transposed_destination_and_untouched_cells():
    """Sum into a column-major destination with a padded leading dimension: numpy's sum, transposed;
    the padding keeps its sentinel (reading R7)."""
    K, R, Cc, ld = 3, 8, 12, 10
    src = layout([(K, R * Cc), (R, Cc), (Cc, 1)])
    dst = layout([(R, 1), (Cc, ld)])
    cfg = dict(dtype="f32", src=src, src_st=linear_storage(K * R * Cc), dst=dst, dst_st=linear_storage(Cc * ld))
    s = synth.numbers(K * R * Cc, "f32", 40, "narrow")
    got = run_local(cfg, s)
    tot = s.view(np.float32).astype(np.float64).reshape(K, R, Cc).sum(axis=0).astype(np.float32)
    g = got.view(np.float32).reshape(Cc, ld)
    assert np.array_equal(g[:, :R], tot.T)
    assert np.array_equal(got.view(np.uint32).reshape(Cc, ld)[:, R:], synth.sentinel(Cc * ld * 4, 99).view(np.uint32).reshape(Cc, ld)[:, R:])


def test_source_replicas_and_destination_replicas():
    """A source replica (consistent copies) does not change the sum; a destination replica writes the
    same sum twice (P:122 replicas are copies)."""
    K, N = 4, 32
    src = layout([(K, N), (N, 1)], [(2, K * N)])
    dst = layout([(N, 1)], [(2, N)])
    s = synth.numbers(K * N, "f32", 41, "narrow")
    sbuf = np.concatenate([s, s])
    cfg = dict(dtype="f32", src=src, src_st=linear_storage(2 * K * N), dst=dst, dst_st=linear_storage(2 * N))
    got = run_local(cfg, sbuf).view(np.float32)
    tot = s.view(np.float32).astype(np.float64).reshape(K, N).sum(axis=0).astype(np.float32)
    assert np.array_equal(got[:N], tot) and np.array_equal(got[N:], tot)


def test_k_equals_one_is_a_copy():
    """K = 1: the sum of one term is the term (for every float format, no rounding)."""
    for dtype in ("f16", "bf16", "f32", "f64"):
        cfg = synth.reduce_local(1, 4, 16, dtype)
        s = synth.numbers(64, dtype, 42)
        assert np.array_equal(run_local(cfg, s), s)


def test_errors():
    s = synth.numbers(30, "f32", 1)
    with pytest.raises(oracle.OracleError) as e:  # E_D(src) not a multiple of E_D(dst)
        oracle.reduce(layout([(30, 1)]), linear_storage(30), s, layout([(7, 1)]), linear_storage(7),
                      np.zeros(28, np.uint8), "f32")
    assert e.value.status == "size"
    with pytest.raises(oracle.OracleError) as e:  # two y write one cell
        oracle.reduce(layout([(30, 1)]), linear_storage(30), s, layout([(3, 0 + 1), (5, 1)]), linear_storage(8),
                      np.zeros(32, np.uint8), "f32")
    assert e.value.status == "collide"


@pytest.mark.parametrize("dtype", ["f16", "bf16", "f32"])
def test_wide_range_sums_are_the_correctly_rounded_sum(dtype):
    """Summands spanning the whole exponent range (subnormals, cancellation, f16 overflow): the oracle's
    fp64 sum rounded once equals math.fsum (the exactly rounded sum) cast to the type -- except where the
    two roundings of fp64-then-type differ from one rounding, which leaves at most one unit in the last
    place (and never changes the result's sign or overflow)."""
    import math
    K, R, Cc = 6, 16, 64
    cfg = synth.reduce_local(K, R, Cc, dtype)
    s = synth.numbers(K * R * Cc, dtype, 51)
    got = run_local(cfg, s)
    x = as_float64(s, dtype).reshape(K, R * Cc)
    exact = np.array([math.fsum(x[:, j]) for j in range(R * Cc)])
    exp = to_dtype_bytes(exact, dtype)
    ut = np.uint16 if dtype in ("f16", "bf16") else np.uint32
    g, e = got.view(ut).astype(np.int64), exp.view(ut).astype(np.int64)
    assert (g == e).mean() > 0.99
    assert np.all(np.abs(g - e) <= 1)


def test_cancelling_pairs_sum_to_the_rest():
    """synth.cancelling: summand 1 is summand 0 negated, so the sum is exactly that of summands 2..K-1."""
    K, Y = 4, 256
    s = synth.cancelling(K, Y, "f32", 52)
    cfg = synth.reduce_local(K, 1, Y, "f32")
    got = run_local(cfg, s).view(np.float32)
    x = s.view(np.float32).astype(np.float64).reshape(K, Y)
    assert np.array_equal(x[0], -x[1])
    assert np.array_equal(got, (x[2] + x[3]).astype(np.float32))
