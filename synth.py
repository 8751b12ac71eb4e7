"""Seeded synthetic inputs and workload descriptions shared by tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no layout evaluation, storage
indexing, swizzling or copying).  It only provides

  * the value generator v(x) (splitmix64, SURVEY.md §8(c) "Data generator"),
  * the untouched-cell sentinel generator,
  * the BASELINE.json workload descriptions as plain data: every layout is a
    dict {"D": [(extent, stride, axis)], "R": [...], "O": {axis: value}} and
    every storage descriptor is a dict {"digits": [(axis, extent, divisor)],
    "swizzle": (B, M, S)}.

Both the oracle (oracle/) and the product binding (paper_2601_19092_b200/)
consume these plain tuples; neither imports the other.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
SEED_BASE = 2601190920  # seed = SEED_BASE + config number

_DT = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}


def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def values(n: int, es: int, seed: int) -> np.ndarray:
    """Logical tensor values v(x), x in [0, n): low 8*es bits of splitmix64(seed ^ x*phi).

    Returned as a flat uint8 array of n*es bytes (raw bit patterns: random bf16/fp32
    words include NaN/Inf/denormal encodings, so compare as integers, never floats).
    """
    out = np.empty(n * es, dtype=np.uint8)
    chunk = 1 << 22
    words = max(1, es // 8)

    def fill(s):
        e = min(n, s + chunk)
        x = np.arange(s, e, dtype=np.uint64)
        if es <= 8:
            with np.errstate(over="ignore"):
                h = _splitmix64(np.uint64(seed) ^ (x * GOLDEN))
            out[s * es:e * es] = h.astype(_DT[es]).view(np.uint8)
        else:  # 16-byte elements: two consecutive 64-bit draws
            parts = []
            for w in range(words):
                with np.errstate(over="ignore"):
                    parts.append(_splitmix64(np.uint64(seed) ^ ((x * np.uint64(words) + np.uint64(w)) * GOLDEN)))
            out[s * es:e * es] = np.stack(parts, axis=1).reshape(-1).view(np.uint8)

    starts = range(0, n, chunk)
    if n > 4 * chunk:  # numpy releases the GIL inside these ufuncs: chunks in parallel, same values
        from concurrent.futures import ThreadPoolExecutor
        import os
        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
            list(ex.map(fill, starts))
    else:
        for s in starts:
            fill(s)
    return out


def sentinel(nbytes: int, seed: int) -> np.ndarray:
    """Untouched-cell sentinel bytes s(i) = splitmix64(~seed ^ i)."""
    n8 = (nbytes + 7) // 8
    h = np.empty(n8, dtype=np.uint64)
    chunk = 1 << 22

    def fill(s):
        e = min(n8, s + chunk)
        with np.errstate(over="ignore"):
            h[s:e] = _splitmix64(np.uint64(~np.uint64(seed)) ^ (np.arange(s, e, dtype=np.uint64) * GOLDEN))

    starts = range(0, n8, chunk)
    if n8 > 4 * chunk:  # chunks in parallel (numpy releases the GIL), same bytes
        from concurrent.futures import ThreadPoolExecutor
        import os
        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
            list(ex.map(fill, starts))
    else:
        for s in starts:
            fill(s)
    return h.view(np.uint8)[:nbytes]


# ----------------------------------------------------------------------------
# Plain-data helpers
# ----------------------------------------------------------------------------

def layout(D, R=(), O=None):
    """A layout as plain data. Iters are (extent, stride, axis); axis None means "m"."""
    fix = lambda it: (int(it[0]), int(it[1]), it[2] if len(it) > 2 and it[2] is not None else "m")
    return {"D": [fix(i) for i in D], "R": [fix(i) for i in R], "O": dict(O or {})}


def storage(digits, swizzle=(0, 0, 0)):
    fix = lambda d: (d[0], int(d[1]), int(d[2]) if len(d) > 2 else 1)
    return {"digits": [fix(d) for d in digits], "swizzle": tuple(int(v) for v in swizzle)}


def linear_storage(n: int, swizzle=(0, 0, 0), axis="m"):
    return storage([(axis, n, 1)], swizzle)


def storage_cells(st) -> int:
    n = 1
    for _, e, _ in st["digits"]:
        n *= e
    return n


SW128 = (3, 4, 3)
SW64 = (2, 4, 3)
SW32 = (1, 4, 3)

# ----------------------------------------------------------------------------
# BASELINE.json configs; sizes are parameters so tests can
# scale them down while keeping their structure.
# ----------------------------------------------------------------------------


def config1():
    """8x8 fp32 row-major -> (lane, warp, m) layout with replica + offset."""
    src = layout([(8, 8), (8, 1)])
    dst = layout([(8, 4, "lane"), (2, 1, "warp"), (2, 1, "lane"), (2, 1, "m")],
                 [(2, 4, "warp")], {"warp": 5})
    return dict(name="config1", es=4, src=src, src_st=linear_storage(64),
                dst=dst, dst_st=storage([("warp", 11), ("lane", 32), ("m", 2)]), seed=SEED_BASE + 1)


def config1_tc():
    """The exact §2.2 tensor-core tile layout on an 8x16 fp32 tile."""
    src = layout([(8, 16), (16, 1)])
    dst = layout([(8, 4, "lane"), (2, 1, "warp"), (4, 1, "lane"), (2, 1, "reg")],
                 [(2, 4, "warp")], {"warp": 5})
    return dict(name="config1_tc", es=4, src=src, src_st=linear_storage(128),
                dst=dst, dst_st=storage([("warp", 11), ("lane", 32), ("reg", 2)]), seed=SEED_BASE + 1)


def config2(n: int = 4096, tile: int = 64, es: int = 2, swizzle=SW128, reverse: bool = False):
    """n x n row-major -> (n/t, t, n/t, t):(t*n, t, t*t, 1) tiles, 128B swizzle."""
    b = n // tile
    rm = layout([(n, n), (n, 1)])
    tl = layout([(b, tile * n), (tile, tile), (b, tile * tile), (tile, 1)])
    st_rm = linear_storage(n * n)
    st_tl = linear_storage(n * n, swizzle)
    if reverse:
        return dict(name="config2r", es=es, src=tl, src_st=st_tl, dst=rm, dst_st=st_rm, seed=SEED_BASE + 2)
    return dict(name="config2", es=es, src=rm, src_st=st_rm, dst=tl, dst_st=st_tl, seed=SEED_BASE + 2)


def _regdump_storage(tiles: int):
    return storage([("cta", tiles), ("warp", 8), ("reg", 16, 8), ("lane", 32), ("reg", 8)])


def config3_src(tiles: int):
    """mma.sync m16n8k16 C-fragments of a 128x256 tile over 8 warps (2x4), warp tile 64x64."""
    return layout([(tiles, 1, "cta"), (2, 4, "warp"), (4, 32, "reg"), (2, 2, "reg"), (8, 4, "lane"),
                   (4, 1, "warp"), (8, 4, "reg"), (4, 1, "lane"), (2, 1, "reg")])


def config3a_dst(tiles: int):
    """tcgen05.ld 32x32b row-per-thread: warp = 4*wg + wq, lane = row mod 32, reg = column."""
    return layout([(tiles, 1, "cta"), (4, 1, "warp"), (32, 1, "lane"), (2, 4, "warp"), (128, 1, "reg")])


def config3b_dst(tiles: int):
    """Per-8x8 transposed fragment (movmatrix.trans of every 32-bit register)."""
    return layout([(tiles, 1, "cta"), (2, 4, "warp"), (4, 32, "reg"), (2, 2, "reg"), (4, 1, "lane"),
                   (2, 1, "reg"), (4, 1, "warp"), (8, 4, "reg"), (4, 8, "lane"), (2, 4, "lane")])


def config3(tiles: int = 65536, variant: str = "a"):
    dst = config3a_dst(tiles) if variant == "a" else config3b_dst(tiles)
    st = _regdump_storage(tiles)
    return dict(name="config3" + variant, es=2, src=config3_src(tiles), src_st=st, dst=dst, dst_st=st,
                seed=SEED_BASE + 3)


def config4(P: int, n: int = 16384):
    """n x n on a 1-D mesh: shard(dim0) -> replicate (all-gather)."""
    src = layout([(P, 1, "gpuid"), (n // P, n), (n, 1)])
    dst = layout([(n, n), (n, 1)], [(P, 1, "gpuid")])
    return dict(name="config4", es=2, nranks=P, src=src, src_st=linear_storage(n // P * n),
                dst=dst, dst_st=linear_storage(n * n), seed=SEED_BASE + 4)


def config5(rows: int = 32768, cols: int = 8192, A: int = 2, B: int = 4):
    """A x B mesh (gpuid = B*a + b): [S(0)@a, R@b] -> [R@a, S(1)@b]."""
    src = layout([(A, B, "gpuid"), (rows // A, cols), (cols, 1)], [(B, 1, "gpuid")])
    dst = layout([(rows, cols // B), (B, 1, "gpuid"), (cols // B, 1)], [(A, B, "gpuid")])
    return dict(name="config5", es=2, nranks=A * B, src=src, src_st=linear_storage(rows // A * cols),
                dst=dst, dst_st=linear_storage(rows * cols // B), seed=SEED_BASE + 5)


# ----------------------------------------------------------------------------
# Reduction rows.  Summands are finite numbers
# whose bit patterns are assembled directly from the splitmix64 draws (no
# rounding, no arithmetic of the method).
# ----------------------------------------------------------------------------

# name -> (sign bit, exponent shift, exponent bias, fraction bits, storage dtype)
_FLOAT_FORMATS = {
    "f16": (15, 10, 15, 10, np.uint16),
    "bf16": (15, 7, 127, 7, np.uint16),
    "f32": (31, 23, 127, 23, np.uint32),
    "f64": (63, 52, 1023, 52, np.uint64),
}
DTYPE_SIZE = {"f16": 2, "bf16": 2, "f32": 4, "f64": 8, "i32": 4, "i64": 8}


# exponent-field ranges of the "wide" summands: the whole range of binary16 (subnormals up to 65504, so
# f16 sums overflow and straddle the largest finite value); for bf16 / f32 / f64 everything from the
# subnormals up to bias + 110 (bias + 900 for f64), so no fp32 (fp64) partial sum of K <= 256 terms
# can overflow the accumulator -- 237 binades of bf16 / f32 in one sum
_WIDE_EXP = {"f16": (0, 30), "bf16": (0, 127 + 110), "f32": (0, 127 + 110), "f64": (0, 1023 + 900)}


def numbers(n: int, dtype: str, seed: int, dist: str = "wide") -> np.ndarray:
    """n summands of `dtype` as raw bytes.  Floats: random sign and fraction; the exponent field
    uniform over `dist`'s range -- "wide": _WIDE_EXP (subnormals, cancellation between terms of
    similar size, sums of terms hundreds of binades apart, f16 overflow); "narrow": bias-8 .. bias-1
    (|v| in [2^-8, 1): every partial sum of K <= 32 bf16 / f16 terms is exact in fp32, used where a
    test needs exact sums); "top": the top 4 binades of f16 (sums land around 65504).  Integers: the
    raw draws (sums wrap modulo 2^bits)."""
    with np.errstate(over="ignore"):
        h = _splitmix64(np.uint64(seed) ^ (np.arange(n, dtype=np.uint64) * GOLDEN))
    if dtype == "i32":
        return h.astype(np.uint32).view(np.uint8)
    if dtype == "i64":
        return h.view(np.uint8)
    sbit, eshift, bias, fbits, st = _FLOAT_FORMATS[dtype]
    sign = (h >> np.uint64(63)) << np.uint64(sbit)
    frac = h & np.uint64((1 << fbits) - 1)
    if dist == "narrow":
        efield = np.uint64(bias - 8) + ((h >> np.uint64(56)) & np.uint64(7))
    elif dist == "wide" or dist == "top":
        lo, hi = _WIDE_EXP[dtype] if dist == "wide" else (27, 30)
        if dist == "top" and dtype != "f16":
            raise ValueError("'top' is the f16 overflow range")
        efield = np.uint64(lo) + (h >> np.uint64(40)) % np.uint64(hi - lo + 1)
    else:
        raise ValueError(dist)
    return (sign | (efield << np.uint64(eshift)) | frac).astype(st).view(np.uint8)


def cancelling(K: int, Y: int, dtype: str, seed: int) -> np.ndarray:
    """(K, Y) summands (logical order k * Y + y) where summand 1 of every output is summand 0 with its
    sign bit flipped (exact cancellation when K >= 2) and the rest are "wide" numbers: whenever the
    pair is the largest term the result is small against sum |x_k|."""
    es = DTYPE_SIZE[dtype]
    a = numbers(K * Y, dtype, seed, "wide").copy()
    if K < 2:
        return a
    sbit = _FLOAT_FORMATS[dtype][0]
    st = _FLOAT_FORMATS[dtype][4]
    v = a.view(st)
    v[Y:2 * Y] = v[:Y] ^ st(1 << sbit)
    return v.view(np.uint8)[:K * Y * es]


def reduce_local(K: int = 8, rows: int = 8192, cols: int = 4096, dtype: str = "bf16", tiled: bool = False):
    """One-GPU sum over the leading dimension: (K, rows, cols) row-major -> (rows, cols), row-major
    or (tiled) 64x64 tiles with SW128 (the reduction fused with the re-tiling of config 2)."""
    src = layout([(K, rows * cols), (rows, cols), (cols, 1)])
    if tiled:
        t = 64
        dst = layout([(rows // t, t * cols), (t, t), (cols // t, t * t), (t, 1)])
        dst_st = linear_storage(rows * cols, SW128)
    else:
        dst = layout([(rows, cols), (cols, 1)])
        dst_st = linear_storage(rows * cols)
    return dict(name="reduce_local" + ("_tiled" if tiled else ""), dtype=dtype, K=K, src=src,
                src_st=linear_storage(K * rows * cols), dst=dst, dst_st=dst_st, seed=SEED_BASE + 6)


def reduce_scatter(P: int, rows: int = 64, cols: int = 64, dtype: str = "bf16"):
    """The DTensor reduce-scatter of P:399-403: a (P, rows, cols) tensor whose dim 0 is sharded over
    P devices (each holds one partial), summed over dim 0 into (rows, cols) sharded by rows."""
    src = layout([(P, 1, "gpuid"), (rows, cols), (cols, 1)])
    dst = layout([(P, 1, "gpuid"), (rows // P, cols), (cols, 1)])
    return dict(name="reduce_scatter", dtype=dtype, nranks=P, src=src, src_st=linear_storage(rows * cols),
                dst=dst, dst_st=linear_storage(rows // P * cols), seed=SEED_BASE + 7)


def all_reduce(P: int, rows: int = 64, cols: int = 64, dtype: str = "bf16"):
    """Partial -> Replicate: every device ends with the full sum."""
    src = layout([(P, 1, "gpuid"), (rows, cols), (cols, 1)])
    dst = layout([(rows, cols), (cols, 1)], [(P, 1, "gpuid")])
    return dict(name="all_reduce", dtype=dtype, nranks=P, src=src, src_st=linear_storage(rows * cols),
                dst=dst, dst_st=linear_storage(rows * cols), seed=SEED_BASE + 8)
