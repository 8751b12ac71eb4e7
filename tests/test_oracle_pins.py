"""Pins for the CPU oracle (oracle/), checked against things other than itself.

Each test names the PAPER.md passage ("P:<line>", section) whose printed value,
closed form or stated property it checks, or the library routine / invariant
that the special case reduces to.  No value here comes from the CUDA path.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth
from synth import layout, storage, linear_storage

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def coords(L, x):
    """f_L(x) as a sorted list of tuples over the layout's axes, zeros included."""
    return sorted(tuple(sorted(c.items())) for c in oracle.eval(L, x))


def flat(S, u):
    x = 0
    for s, v in zip(S, u):
        x = x * s + v
    return x


# ---------------------------------------------------------------------------
# §2.2 worked examples
# ---------------------------------------------------------------------------

TC = layout([(8, 4, "lane"), (2, 1, "warp"), (4, 1, "lane"), (2, 1, "reg")], [(2, 4, "warp")], {"warp": 5})


def test_tensor_core_tile_prose():
    """rows -> lane (stride 4); columns split 2x4x2 over warp, lane, reg (stride 1 each);
    replicated twice 4 warps apart; offset 5 warps => warps {5,6} and {9,10} hold the 8x16 tile."""
    S = (8, 16)
    warps = set()
    for i in range(8):
        for j in range(16):
            got = coords(TC, flat(S, (i, j)))
            exp = sorted(tuple(sorted({"lane": 4 * i + (j // 2) % 4, "warp": 5 + j // 8 + 4 * r,
                                       "reg": j % 2}.items())) for r in range(2))
            assert got == exp, (i, j)
            warps |= {dict(c)["warp"] for c in got}
    assert warps == {5, 6, 9, 10}
    assert coords(TC, 0) == sorted([(("lane", 0), ("reg", 0), ("warp", 5)), (("lane", 0), ("reg", 0), ("warp", 9))])


def test_tensor_core_tile_cells_hit_once():
    """Bijection modulo replicas: 128 elements x 2 replicas = 256 distinct (warp, lane, reg) cells."""
    cells = [c for x in range(128) for c in coords(TC, x)]
    assert len(cells) == 256 and len(set(cells)) == 256


def test_tensor_core_tile_span():
    """SPEC S:125 (span example) from the closed form of App. C: 1 + sum |s|(e-1)."""
    assert oracle.bounds(TC, "lane") == (0, 31)
    assert oracle.bounds(TC, "warp") == (5, 10)       # span 6
    assert oracle.bounds(TC, "reg") == (0, 1)


MESH_SS = layout([(2, 1, "gpuid"), (32, 128), (2, 2, "gpuid"), (64, 1)])
MESH_SR = layout([(2, 1, "gpuid"), (32, 128), (128, 1)], [(2, 2, "gpuid")])


def test_mesh_fully_sharded():
    """64x128 over the 2x2 mesh [[GPU0, GPU2], [GPU1, GPU3]]: rows split across mesh rows,
    columns across mesh columns; local offset 128*(i mod 32) + (j mod 64) (taken as printed, R15)."""
    S = (64, 128)
    for i in range(64):
        for j in range(128):
            (c,) = oracle.eval(MESH_SS, flat(S, (i, j)))
            assert c["gpuid"] == (i // 32) + 2 * (j // 64)
            assert c["m"] == 128 * (i % 32) + j % 64
    assert oracle.eval(MESH_SS, flat(S, (63, 127)))[0] == {"gpuid": 3, "m": 4031}


def test_mesh_shard_replicate():
    """rows split over the two mesh-row groups, each row shard replicated on both GPUs
    of its group (Alpa S^0 R)."""
    S = (64, 128)
    for i in range(0, 64, 3):
        for j in range(0, 128, 5):
            got = oracle.eval(MESH_SR, flat(S, (i, j)))
            assert sorted(c["gpuid"] for c in got) == sorted([i // 32, i // 32 + 2])
            assert all(c["m"] == 128 * (i % 32) + j for c in got)


def test_sbuf_layout():
    """(2,128,512):(512@F,1@P,1@F) for a logical 256x512 tensor over 128 partitions:
    (i, j) -> P = i mod 128, F = 512*floor(i/128) + j."""
    L = layout([(2, 512, "F"), (128, 1, "P"), (512, 1, "F")])
    for i in range(0, 256, 7):
        for j in range(0, 512, 13):
            (c,) = oracle.eval(L, flat((256, 512), (i, j)))
            assert c == {"F": 512 * (i // 128) + j, "P": i % 128}


# ---------------------------------------------------------------------------
# §3.1 motivating example: CuTe partition and Triton CTA layout
# ---------------------------------------------------------------------------

CUTE = layout([(16, 128), (8, 8), (2, 4), (4, 1)], O={"m": 2112})


def test_cute_partition():
    """thread i loads the [1,8] region starting at [16 + i//8, 64 + (i mod 8)*8] of a row-major
    fp32 (32,128) tensor C; the partition (16,8,2,4):(128,8,4,1)+2112 enumerates (tx//8, tx%8, k)."""
    for tx in range(128):
        for k in range(8):
            x = flat((16, 8, 8), (tx // 8, tx % 8, k))
            (c,) = oracle.eval(CUTE, x)
            row, col = 16 + tx // 8, 64 + (tx % 8) * 8 + k
            assert c == {"m": row * 128 + col}


def test_cute_thread_binding_residual():
    """binding the first two loops to tx//8, tx%8 leaves (2,4):(4,1) +
    ((tx//8)*128 + (tx%8)*8 + 2112)@m for each thread."""
    for tx in range(128):
        res = layout([(2, 4), (4, 1)], O={"m": (tx // 8) * 128 + (tx % 8) * 8 + 2112})
        for k in range(8):
            assert oracle.eval(res, k) == oracle.eval(CUTE, tx * 8 + k)


def test_triton_register_layout_matches_cute_partition():
    """C_local:(16,8,8):(8@tx,1@tx,1@reg) = C[16:32, 64:128] describes the same copy as the
    CuTe partition: element (i, j) of the region lives in thread tx at register reg,
    where the CuTe thread tx loads C[16+i, 64+j] as its reg-th element."""
    T = layout([(16, 8, "tx"), (8, 1, "tx"), (8, 1, "reg")])
    owner = {}
    for tx in range(128):
        for k in range(8):
            (c,) = oracle.eval(CUTE, tx * 8 + k)
            owner[c["m"]] = (tx, k)
    for i in range(16):
        for j in range(64):
            (c,) = oracle.eval(T, flat((16, 64), (i, j)))
            assert (c["tx"], c.get("reg", 0)) == owner[(16 + i) * 128 + 64 + j]
    assert oracle.eval(T, flat((16, 64), (0, 9)))[0] == {"tx": 1, "reg": 1}


# ---------------------------------------------------------------------------
# §3.3 tile and slice examples, App. F, App. G
# ---------------------------------------------------------------------------

def test_tile_example_formula():
    """P:440-444 + P:451-457: (2,3):(3,1) (x) (8,8):(8,1) = (2,8,3,8):(192,8,64,1) satisfies
    f_T(x||y) = f_A(x) * span(f_B) + f_B(y), span(f_B) = 64 (reading R10: the formula decides)."""
    A = layout([(2, 3), (3, 1)])
    B = layout([(8, 8), (8, 1)])
    T = layout([(2, 192), (8, 8), (3, 64), (8, 1)])
    lo, hi = oracle.bounds(B, "m")
    span = hi - lo + 1
    assert span == 64
    for p, i, q, j in itertools.product(range(2), range(8), range(3), range(8)):
        x = flat((2, 8, 3, 8), (p, i, q, j))
        fa = oracle.eval(A, flat((2, 3), (p, q)))[0]["m"]
        fb = oracle.eval(B, flat((8, 8), (i, j)))[0]["m"]
        assert oracle.eval(T, x)[0]["m"] == fa * span + fb


def test_tile_example_block_layout():
    """the tiled layout is a 16x24 matrix made of 8x8 blocks with 64 contiguous elements each,
    blocks arranged as a 2x3 grid in row-major order (reading R10)."""
    T = layout([(2, 192), (8, 8), (3, 64), (8, 1)])
    for r in range(16):
        for c in range(24):
            blk = (r // 8) * 3 + c // 8
            assert oracle.eval(T, flat((16, 24), (r, c)))[0]["m"] == blk * 64 + (r % 8) * 8 + c % 8


def test_slice_example():
    """L = (2,8,3,8):(192,8,64,1), S = (16,24), R = [0:8) x [8:24)
    => L[R:S] = (1,8,2,8):(192,8,64,1) + 64, i.e. f_{L[R:S]<T>}(u) = f_{L<S>}(u + b)."""
    L = layout([(2, 192), (8, 8), (3, 64), (8, 1)])
    Ls = layout([(1, 192), (8, 8), (2, 64), (8, 1)], O={"m": 64})
    for u0 in range(8):
        for u1 in range(16):
            assert oracle.eval(Ls, flat((8, 16), (u0, u1))) == oracle.eval(L, flat((16, 24), (u0, u1 + 8)))


def test_direct_sum_example_values():
    """f_B = {0,1,4,5} for B = (2,2):(4,1); f_A = {0,2,8,10} for A = (2,2):(8,2);
    span(f_B) = 6; the A+B digit list (2,2,2,2):(8,4,2,1) enumerates {0..15}."""
    B = layout([(2, 4), (2, 1)])
    A = layout([(2, 8), (2, 2)])
    assert sorted(oracle.eval(B, x)[0]["m"] for x in range(4)) == [0, 1, 4, 5]
    assert sorted(oracle.eval(A, x)[0]["m"] for x in range(4)) == [0, 2, 8, 10]
    lo, hi = oracle.bounds(B, "m")
    assert hi - lo + 1 == 6
    AB = layout([(2, 8), (2, 4), (2, 2), (2, 1)])
    assert [oracle.eval(AB, x)[0]["m"] for x in range(16)] == list(range(16))


def test_non_bit_linear_example():
    """column-major 24x24, f(i) = floor(i/24) + (i mod 24)*24: f(1) = 24, f(2) = 48,
    f(3) = 72 and f(1) xor f(2) = 40 != f(1 xor 2)."""
    L = layout([(24, 1), (24, 24)])
    f = lambda x: oracle.eval(L, x)[0]["m"]
    assert (f(1), f(2), f(3)) == (24, 48, 72)
    assert f(1) ^ f(2) == 40 != f(1 ^ 2)
    for i in range(0, 576, 17):
        assert f(i) == i // 24 + (i % 24) * 24


def test_golden_files():
    """Every fixture under tests/golden/ carries its own citation; each lists (layout, x, expected)."""
    files = sorted(f for f in os.listdir(GOLD) if f.endswith(".json"))
    assert files
    for fn in files:
        with open(os.path.join(GOLD, fn)) as fh:
            g = json.load(fh)
        assert g.get("cite"), fn
        L = layout(g["layout"]["D"], g["layout"].get("R", []), g["layout"].get("O", {}))
        shape = g.get("shape")
        for case in g["cases"]:
            x = flat(shape, case["u"]) if shape else case["x"]
            got = sorted(sorted((a, v) for a, v in c.items() if v != 0) for c in oracle.eval(L, x))
            exp = sorted(sorted((a, v) for a, v in c.items() if v != 0) for c in case["expect"])
            assert got == exp, (fn, case)


# ---------------------------------------------------------------------------
# Properties of f_L
# ---------------------------------------------------------------------------

def rand_layout(rng, axes=("m", "lane", "warp")):
    nD = rng.integers(1, 5)
    D = [(int(rng.integers(1, 7)), int(rng.choice([-1, 1]) * rng.integers(1, 24)), str(rng.choice(axes)))
         for _ in range(nD)]
    R = [(int(rng.integers(1, 4)), int(rng.choice([-1, 1]) * rng.integers(1, 24)), str(rng.choice(axes)))
         for _ in range(rng.integers(0, 3))]
    O = {str(a): int(rng.integers(-5, 6)) for a in rng.choice(axes, size=rng.integers(0, 3))}
    return layout(D, R, O)


def test_eval_cardinality_and_replica_permutation():
    """|f_L(x)| = E_R and f_L is invariant under permutation of R (a multiset)."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        L = rand_layout(rng)
        ed, er = oracle.sizes(L)
        Lp = dict(L, R=list(reversed(L["R"])))
        for x in range(0, ed, max(1, ed // 7)):
            assert len(oracle.eval(L, x)) == er
            assert oracle.eval_set(L, x) == oracle.eval_set(Lp, x)


def test_bounds_closed_form():
    """App. C Lemma span-closed, signed form: per axis, min = O_a + sum min(0,(e-1)s),
    max = O_a + sum max(0,(e-1)s) over the iters of D and R on that axis."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        L = rand_layout(rng)
        for a in ("m", "lane", "warp"):
            its = [it for it in L["D"] + L["R"] if it[2] == a]
            b = oracle.bounds(L, a)
            if not its and a not in L["O"]:
                assert b is None
                continue
            o = L["O"].get(a, 0)
            assert b == (o + sum(min(0, (e - 1) * s) for e, s, _ in its),
                         o + sum(max(0, (e - 1) * s) for e, s, _ in its))


def test_eval_domain_error():
    with pytest.raises(oracle.OracleError) as ei:
        oracle.eval(TC, 128)
    assert ei.value.status == "domain"
    with pytest.raises(oracle.OracleError):
        oracle.eval(layout([(4, 0)]), 0)        # s != 0 (Def. Iter)
    with pytest.raises(oracle.OracleError):
        oracle.eval(layout([(0, 1)]), 0)        # e > 0


# ---------------------------------------------------------------------------
# Copy: special cases that reduce to library routines (numpy), no shared code
# ---------------------------------------------------------------------------

def _vals(n, es, seed=1):
    return synth.values(n, es, seed)


@pytest.mark.parametrize("es", [1, 2, 4, 8, 16])
def test_copy_identity_is_memcpy(es):
    n = 1000
    v = _vals(n, es)
    out = synth.sentinel(n * es, 3)
    L = layout([(n, 1)])
    oracle.copy(L, linear_storage(n), v, L, linear_storage(n), out, es)
    assert np.array_equal(out, v)


@pytest.mark.parametrize("R,Cn,es", [(64, 32, 2), (7, 13, 4), (24, 24, 8)])
def test_copy_transpose_is_numpy_transpose(R, Cn, es):
    v = _vals(R * Cn, es)
    src = layout([(R, Cn), (Cn, 1)])
    dst = layout([(R, 1), (Cn, R)])          # column-major
    out = np.zeros(R * Cn * es, np.uint8)
    oracle.copy(src, linear_storage(R * Cn), v, dst, linear_storage(R * Cn), out, es)
    a = v.view(synth._DT[es]).reshape(R, Cn)
    assert np.array_equal(out.view(synth._DT[es]), np.ascontiguousarray(a.T).reshape(-1))


def test_copy_tiling_is_numpy_block_permute():
    """Config-2 structure without swizzle: row-major -> 64x64 tiles == view(b,t,b,t).permute(0,2,1,3)."""
    n, t = 512, 64
    cfg = synth.config2(n, t, 2, swizzle=(0, 0, 0))
    v = _vals(n * n, 2)
    out = np.zeros_like(v)
    oracle.copy(cfg["src"], cfg["src_st"], v, cfg["dst"], cfg["dst_st"], out, 2)
    a = v.view(np.uint16).reshape(n // t, t, n // t, t)
    assert np.array_equal(out.view(np.uint16), np.ascontiguousarray(a.transpose(0, 2, 1, 3)).reshape(-1))


def _sw128_numpy(tiles_u16: np.ndarray) -> np.ndarray:
    """128-byte swizzle as the TMA/CUTLASS docs describe it for 128-byte rows: in every 1024-byte
    block, the 16-byte chunk j of row r (r = 0..7) is stored at chunk position j ^ r."""
    b = tiles_u16.view(np.uint8).reshape(-1, 8, 8, 16)        # [block][row][chunk][16 bytes]
    out = np.empty_like(b)
    for r in range(8):
        for j in range(8):
            out[:, r, j ^ r, :] = b[:, r, j, :]
    return out.reshape(-1)


def test_copy_config2_small_swizzled_matches_numpy():
    n, t = 256, 64
    cfg = synth.config2(n, t)
    v = _vals(n * n, 2)
    out = np.zeros_like(v)
    oracle.copy(cfg["src"], cfg["src_st"], v, cfg["dst"], cfg["dst_st"], out, 2)
    a = v.view(np.uint16).reshape(n // t, t, n // t, t)
    tiled = np.ascontiguousarray(a.transpose(0, 2, 1, 3)).reshape(-1)
    assert np.array_equal(out, _sw128_numpy(tiled))


def test_config2_goldens():
    """SURVEY §8(c) config-2 goldens: logical (r,c) -> dst element offset under
    (64,64,64,64):(262144,64,4096,1) + SW128 (bf16)."""
    cfg = synth.config2()
    table = {(0, 0): 0, (0, 8): 8, (1, 0): 72, (1, 8): 64, (3, 17): 201, (7, 63): 455, (8, 0): 512,
             (0, 64): 4096, (64, 0): 262144, (4095, 4095): 16777159}
    for (r, c), off in table.items():
        (co,) = oracle.eval(cfg["dst"], r * 4096 + c)
        assert oracle.storage_byte(cfg["dst_st"], co, 2) == 2 * off


def test_swizzle_involution_and_block_bijection():
    st = linear_storage(1 << 12, synth.SW128)
    offs = [oracle.storage_byte(st, {"m": i}, 2) for i in range(1 << 12)]
    assert sorted(offs) == list(range(0, 1 << 13, 2))
    for i in range(0, 1 << 12, 37):           # blocks of 1024 B map onto themselves
        assert offs[i] // 1024 == (2 * i) // 1024


def test_copy_replica_offset_config1():
    """Config 1 (SURVEY §8(c) goldens): 128 cells written, warps {5,6,9,10}, lanes within [0,29];
    x = 63 lands at storage indices {443, 699}; the other 576 cells keep the sentinel."""
    cfg = synth.config1()
    v = _vals(64, 4)
    fill = synth.sentinel(704 * 4, 5)
    out = fill.copy()
    oracle.copy(cfg["src"], cfg["src_st"], v, cfg["dst"], cfg["dst_st"], out, 4)
    w = out.view(np.uint32)
    changed = np.nonzero(w != fill.view(np.uint32))[0]
    assert len(changed) == 128
    warps = set(int(i) // 64 for i in changed)
    lanes = set((int(i) // 2) % 32 for i in changed)
    assert warps == {5, 6, 9, 10} and max(lanes) <= 29
    assert w[443] == v.view(np.uint32)[63] and w[699] == v.view(np.uint32)[63]


def test_copy_round_trip_and_composition():
    """copy(A->B) then copy(B->A) restores A's covered cells; copy(A->B) o copy(B->C) = copy(A->C)."""
    n, t = 128, 16
    A = layout([(n, n), (n, 1)])
    Bl = layout([(n // t, t * n), (t, t), (n // t, t * t), (t, 1)])
    Cl = layout([(n, 1), (n, n)])
    st = linear_storage(n * n)
    stB = linear_storage(n * n, synth.SW64)
    v = _vals(n * n, 4)
    b = np.zeros_like(v); c1 = np.zeros_like(v); c2 = np.zeros_like(v); back = np.zeros_like(v)
    oracle.copy(A, st, v, Bl, stB, b, 4)
    oracle.copy(Bl, stB, b, A, st, back, 4)
    assert np.array_equal(back, v)
    oracle.copy(Bl, stB, b, Cl, st, c1, 4)
    oracle.copy(A, st, v, Cl, st, c2, 4)
    assert np.array_equal(c1, c2)


def test_copy_errors():
    st = linear_storage(16)
    v = _vals(16, 4)
    out = np.zeros_like(v)
    with pytest.raises(oracle.OracleError) as e:           # E_D mismatch
        oracle.copy(layout([(16, 1)]), st, v, layout([(8, 1)]), st, out, 4)
    assert e.value.status == "size"
    with pytest.raises(oracle.OracleError) as e:           # two x to one cell (reading R6)
        oracle.copy(layout([(16, 1)]), st, v, layout([(4, 1), (4, 1)]), st, out, 4)
    assert e.value.status == "collide"
    with pytest.raises(oracle.OracleError) as e:           # outside the storage box
        oracle.copy(layout([(16, 1)]), st, v, layout([(16, 1)], O={"m": 1}), st, out, 4)
    assert e.value.status == "bounds"
    with pytest.raises(oracle.OracleError) as e:           # axis not bound by the storage
        oracle.copy(layout([(16, 1)]), st, v, layout([(16, 1, "lane")]), st, out, 4)
    assert e.value.status == "bounds"
    # aliasing replicas of the same x collapse (set semantics): R = [(2, 0)] is not legal
    # (s != 0) but [(2,1),(2,1)] on an axis of extent... same-x duplicates: (2,1)+(2,1) hits 0,1,1,2
    dst = layout([(4, 4)], [(2, 1), (2, 1)])
    out2 = np.zeros(16 * 4, np.uint8)
    oracle.copy(layout([(4, 1)]), linear_storage(4), v[:16], dst, st, out2, 4)


@pytest.mark.parametrize("es", [2, 4])
def test_storage_divisor_chain_is_numpy_blocking(es):
    """A storage axis split over two digits (S:O6: idx = sum_k ((c[a_k] / div_k) mod ext_k) prod_{j>k} ext_j):
    m = 32 rows stored as (m / 8, n, m mod 8) -- the digit chain ("m", 4, 8), ("n", 3), ("m", 8, 1) -- is
    numpy's blocking of a (32, 3) row-major array: reshape (4, 8, 3), transpose (0, 2, 1), flatten; a
    three-digit chain ("m", 2, 16), ("n", 3), ("m", 4, 4), ("m", 4, 1) is the (2, 16) blocking; with both m
    digits outside n, ("m", 4, 8), ("m", 8, 1), ("n", 3), the chain recomposes m: plain row-major."""
    v = _vals(96, es, 5)
    src = layout([(32, 3), (3, 1)])
    dst = layout([(32, 1, "m"), (3, 1, "n")])
    a = v.view(synth._DT[es]).reshape(32, 3)
    out = np.zeros(96 * es, np.uint8)
    oracle.copy(src, linear_storage(96), v, dst, storage([("m", 4, 8), ("n", 3), ("m", 8, 1)]), out, es)
    assert np.array_equal(out.view(synth._DT[es]), np.ascontiguousarray(a.reshape(4, 8, 3).transpose(0, 2, 1)).reshape(-1))
    out = np.zeros(96 * es, np.uint8)
    oracle.copy(src, linear_storage(96), v, dst, storage([("m", 2, 16), ("n", 3), ("m", 4, 4), ("m", 4, 1)]), out, es)
    assert np.array_equal(out.view(synth._DT[es]), np.ascontiguousarray(a.reshape(2, 16, 3).transpose(0, 2, 1)).reshape(-1))
    out = np.zeros(96 * es, np.uint8)
    oracle.copy(src, linear_storage(96), v, dst, storage([("m", 4, 8), ("m", 8, 1), ("n", 3)]), out, es)
    assert np.array_equal(out, v)


def test_storage_chain_validation():
    assert oracle.storage_check(storage([("reg", 16, 8), ("lane", 32), ("reg", 8)])) == 0
    assert oracle.storage_check(storage([("reg", 16, 4), ("lane", 32), ("reg", 8)])) != 0
    assert oracle.storage_check(storage([("m", 8, 2)])) != 0


# ---------------------------------------------------------------------------
# Config 3 register-dump layouts: structural pins
# ---------------------------------------------------------------------------

def _frag_owner_mma_c(row, col):
    """PTX ISA mma.m16n8k16 (f32/f16 accumulator) C-fragment ownership for a 16x8 tile:
    thread (lane) = 4*(row mod 8) + (col mod 8)//2, element c = 2*(row//8) + col mod 2."""
    return 4 * (row % 8) + (col % 8) // 2, 2 * (row // 8) + col % 2


def test_config3_src_is_mma_c_fragment():
    L = synth.config3_src(1)
    for row in range(0, 128, 3):
        for col in range(0, 256, 5):
            (c,) = oracle.eval(L, row * 256 + col)
            wm, wn = row // 64, col // 64
            mi, ni = (row % 64) // 16, (col % 64) // 8
            lane, e = _frag_owner_mma_c(row % 16, col % 8)
            assert c["warp"] == 4 * wm + wn and c["lane"] == lane
            assert c["reg"] == 32 * mi + 4 * ni + e


def test_config3_dst_bijective():
    st = synth._regdump_storage(1)
    for L in (synth.config3_src(1), synth.config3a_dst(1), synth.config3b_dst(1)):
        seen = set()
        for x in range(128 * 256):
            (c,) = oracle.eval(L, x)
            seen.add(oracle.storage_byte(st, c, 2))
        assert len(seen) == 128 * 256


def test_config3b_is_8x8_transpose_of_each_register():
    """3b holds, for every 8x8 block of each 16x8 fragment, the transposed block (movmatrix.trans
    semantics): element (i, j) of a block sits where element (j, i) sits in the C-fragment."""
    A, Bt = synth.config3_src(1), synth.config3b_dst(1)
    for row in range(128):
        for col in range(0, 256, 3):
            (cb,) = oracle.eval(Bt, row * 256 + col)
            r0, c0 = row - row % 8, col - col % 8
            i, j = row % 8, col % 8
            (ca,) = oracle.eval(A, (r0 + j) * 256 + c0 + i)
            assert cb == ca


# ---------------------------------------------------------------------------
# Redistribute: special cases (all-gather == concatenation; shard change == numpy slicing)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("P", [2, 4])
def test_redistribute_allgather_is_concatenation(P):
    n = 64
    cfg = synth.config4(P, n)
    v = _vals(n * n, 2)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], v, 2, P, np.zeros(n * n // P * 2, np.uint8))
    a = v.view(np.uint16).reshape(n, n)
    for g in range(P):   # shard g holds rows [g*n/P, (g+1)*n/P) (S(0) over gpuid)
        assert np.array_equal(src[g].view(np.uint16).reshape(n // P, n), a[g * n // P:(g + 1) * n // P])
    dst = [np.zeros(n * n * 2, np.uint8) for _ in range(P)]
    oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], dst, 2)
    cat = np.concatenate([s.view(np.uint16) for s in src])
    for g in range(P):
        assert np.array_equal(dst[g].view(np.uint16), cat)


def test_redistribute_config5_is_numpy_slicing():
    rows, cols = 64, 32
    cfg = synth.config5(rows, cols)
    v = _vals(rows * cols, 2)
    a = v.view(np.uint16).reshape(rows, cols)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], v, 2, 8, np.zeros(rows // 2 * cols * 2, np.uint8))
    for g in range(8):
        ga = g // 4
        assert np.array_equal(src[g].view(np.uint16).reshape(rows // 2, cols), a[ga * rows // 2:(ga + 1) * rows // 2])
    dst = [np.zeros(rows * cols // 4 * 2, np.uint8) for _ in range(8)]
    oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], dst, 2)
    for g in range(8):
        gb = g % 4
        assert np.array_equal(dst[g].view(np.uint16).reshape(rows, cols // 4), a[:, gb * cols // 4:(gb + 1) * cols // 4])


def test_redistribute_only_rank_and_bounds():
    cfg = synth.config4(2, 16)
    v = _vals(256, 2)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], v, 2, 2, np.zeros(256, np.uint8))
    d1 = np.zeros(512, np.uint8)
    oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], [None, d1], 2, only_rank=1)
    assert np.array_equal(d1.view(np.uint16), v.view(np.uint16))
    bad = synth.config4(4, 16)        # gpuid reaches 3 but only 2 ranks exist
    with pytest.raises(oracle.OracleError) as e:
        oracle.redistribute(bad["src"], bad["src_st"], src, bad["dst"], bad["dst_st"],
                            [np.zeros(512, np.uint8)] * 2, 2)
    assert e.value.status == "bounds"


def test_threads_agree():
    cfg = synth.config2(256, 64)
    v = _vals(256 * 256, 2)
    o1 = np.zeros_like(v); o4 = np.zeros_like(v)
    oracle.copy(cfg["src"], cfg["src_st"], v, cfg["dst"], cfg["dst_st"], o1, 2, nthreads=1)
    oracle.copy(cfg["src"], cfg["src_st"], v, cfg["dst"], cfg["dst_st"], o4, 2, nthreads=4)
    assert np.array_equal(o1, o4)
