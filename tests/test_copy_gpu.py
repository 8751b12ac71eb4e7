"""GPU parity of axe_copy against the CPU oracle (bit-exact, every byte of the
destination buffer including cells that must stay untouched)."""
import os

import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage, storage

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NT = os.cpu_count() or 4


@pytest.fixture(scope="module")
def axe():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2601_19092_b200 as m
    return m


def to_dev(a: np.ndarray):
    return torch.from_numpy(a).cuda()


def prepare(cfg):
    es = cfg["es"]
    ed, _ = oracle.sizes(cfg["src"])
    v = synth.values(ed, es, cfg["seed"])
    s_fill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, cfg["seed"] + 17)
    src = oracle.scatter_logical(cfg["src"], cfg["src_st"], v, es, s_fill, NT)
    d_fill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, cfg["seed"])
    exp = d_fill.copy()
    oracle.copy(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, es, NT)
    return src, d_fill, exp


GUARD = 4096  # bytes of sentinel on both sides of every device buffer (compute-sanitizer is closed on this pool)


def run_gpu(axe, cfg, src, d_fill, kernel="auto"):
    plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["es"], kernel)
    g = synth.sentinel(2 * GUARD, 99)
    s = to_dev(np.concatenate([g[:GUARD], src, g[GUARD:]]))
    d = to_dev(np.concatenate([g[:GUARD], d_fill, g[GUARD:]]))
    plan.execute(s[GUARD:GUARD + src.nbytes], d[GUARD:GUARD + d_fill.nbytes])
    torch.cuda.synchronize()
    out = d.cpu().numpy()
    assert np.array_equal(out[:GUARD], g[:GUARD]) and np.array_equal(out[-GUARD:], g[GUARD:]), \
        f"{cfg['name']}: write outside the destination buffer"
    return out[GUARD:GUARD + d_fill.nbytes], plan.describe()


def check(axe, cfg, kernel="auto", expect_kernel=None):
    src, d_fill, exp = prepare(cfg)
    got, desc = run_gpu(axe, cfg, src, d_fill, kernel)
    if expect_kernel:
        assert desc["kernel"] == expect_kernel, desc
    if not np.array_equal(got, exp):
        bad = np.nonzero(got != exp)[0]
        raise AssertionError(f"{cfg['name']} [{desc['kernel']}]: {len(bad)} bytes differ, first at {bad[:8]}")
    return desc


@pytest.mark.parametrize("kernel", ["auto", "generic"])
@pytest.mark.parametrize("mk", [synth.config1, synth.config1_tc])
def test_config1_exhaustive(axe, mk, kernel):
    check(axe, mk(), kernel)


@pytest.mark.parametrize("kernel", ["auto", "generic", "vector"])
@pytest.mark.parametrize("n,es,sw,rev", [(256, 2, synth.SW128, False), (256, 2, synth.SW128, True),
                                        (512, 4, synth.SW64, False), (192, 8, synth.SW32, True),
                                        (128, 1, (0, 0, 0), False)])
def test_config2_small(axe, n, es, sw, rev, kernel):
    check(axe, synth.config2(n, 64, es, sw, rev), kernel)


@pytest.mark.parametrize("rev", [False, True])
@pytest.mark.parametrize("kernel", ["auto", "vector", "tma"])
def test_config2_full(axe, rev, kernel):
    """BASELINE config 2 at full size (4096^2 bf16); "auto" is the launch configuration bench.py times."""
    desc = check(axe, synth.config2(reverse=rev), kernel)
    assert desc["kernel"] == ("lowered" if kernel == "auto" else kernel)


@pytest.mark.parametrize("rev", [False, True])
@pytest.mark.parametrize("tr,tc,es", [(256, 64, 2), (128, 128, 1), (256, 32, 4), (64, 64, 2)])
def test_lowered_large_boxes(axe, rev, tr, tc, es):
    """Tall tiles: the lowered schedule fuses up to 256 atom rows into one box (32 KiB); the launch lowers the
    CTAs per SM until every ring holds the 3 slots its refill lag needs, both directions."""
    R, C = 2 * tr * 2, tc * 8
    rm = layout([(R, C), (C, 1)])
    tiles = layout([(R // tr, tr * C), (tr, tc), (C // tc, tr * tc), (tc, 1)])
    st_rm, st_t = linear_storage(R * C), linear_storage(R * C, synth.SW128)
    cfg = dict(name=f"tall{tr}x{tc}x{es}", es=es, src=tiles if rev else rm, src_st=st_t if rev else st_rm,
               dst=rm if rev else tiles, dst_st=st_rm if rev else st_t, seed=tr + tc + es)
    d = check(axe, cfg)
    assert d["kernel"] == "lowered" and d["box_bytes"] == tr * tc * es, d


@pytest.mark.parametrize("R,Cn,es,pad_s,pad_d,B,reps", [
    (4095, 4097, 2, 0, 0, 1, 1), (8000, 8000, 2, 0, 0, 1, 1), (333, 777, 1, 5, 3, 2, 1), (130, 70, 4, 1, 0, 3, 2),
    (65, 129, 8, 0, 7, 1, 1), (31, 33, 16, 2, 2, 2, 3), (1, 1000, 2, 0, 0, 1, 1), (1000, 2, 4, 3, 0, 1, 1),
    (4096, 4097, 4, 0, 0, 1, 1)])
@pytest.mark.parametrize("vec", ["1", "0"])
def test_ragged_transposes(axe, R, Cn, es, pad_s, pad_d, B, reps, vec, monkeypatch):
    """K9 (the fallback of K7 and K2): 2-D transposes with ragged extents and pitches that are not whole
    16-byte vectors (rows starting at any element alignment), padded pitches, a batch digit, destination
    replicas, 1..16-byte elements -- against the oracle, through AUTO and forced; the vector-load form
    (16-byte chunks covering each tile row at any alignment) and the element form."""
    monkeypatch.setenv("AXE_K9_VEC", vec)
    lds, ldd = Cn + pad_s, R + pad_d
    src = layout([(B, R * lds), (R, lds), (Cn, 1)])
    dst = layout([(B, Cn * ldd), (R, 1), (Cn, ldd)], [(reps, B * Cn * ldd)] if reps > 1 else [])
    cfg = dict(name=f"rag{R}x{Cn}x{es}", es=es, src=src, src_st=linear_storage(B * R * lds), dst=dst,
               dst_st=linear_storage(reps * B * Cn * ldd), seed=R * 7 + Cn + es)
    check(axe, cfg)                      # AUTO: K7 (ragged edges masked) / K2 where legal, else K9
    if R > 1 and Cn > 1:                 # (a single row is a plain copy)
        d = check(axe, cfg, "transpose")  # forced transpose: K7 where the extents and pitches are whole
        n = 16 // es                      # 16-byte vectors, else K9
        k7 = es in (2, 4, 8) and R % n == 0 and Cn % n == 0 and lds * es % 16 == 0 and ldd * es % 16 == 0
        assert d["kernel"] == "transpose" and d.get("mode") == (None if k7 else "ragged"), d


@pytest.mark.parametrize("es", [2, 4, 8])
@pytest.mark.parametrize("R,Cn,B,asyn,chunk", [(8000, 8000, 1, 2, ""), (136, 72, 3, 3, "3"), (40, 24, 2, 0, ""),
                                                (264, 520, 1, 2, "1"), (8, 8, 1, 2, "")])
def test_k7_ragged_edges(axe, monkeypatch, es, R, Cn, B, asyn, chunk):
    """K7 with ragged edges: extents of whole 16-byte vectors that are not whole tiles (last tile row and / or
    column partly outside, or a side shorter than one tile), batched, padded pitches, a destination replica;
    register-staged and cp.async forms, persistent and in-order grids -- every byte against the oracle, the
    cells past the extents untouched."""
    n = 16 // es
    R, Cn = R // n * n, Cn // n * n
    monkeypatch.setenv("AXE_K7_ASYNC", str(asyn))
    monkeypatch.setenv("AXE_CHUNK", chunk)
    lds, ldd = Cn + n, R + 2 * n
    src = layout([(B, R * lds), (R, lds), (Cn, 1)])
    dst = layout([(B, Cn * ldd), (R, 1), (Cn, ldd)], [(2, B * Cn * ldd)])
    cfg = dict(name=f"k7r{R}x{Cn}x{es}", es=es, src=src, src_st=linear_storage(B * R * lds), dst=dst,
               dst_st=linear_storage(2 * B * Cn * ldd), seed=R + Cn + es)
    d = check(axe, cfg, "transpose", "transpose")   # (AUTO takes K7 while half of each tile is inside)
    assert "mode" not in d and d["replicas"] == 2, d
    if R * Cn >= 1 << 20:
        assert check(axe, cfg)["kernel"] == "transpose"


@pytest.mark.parametrize("R,Cn,es", [(8192, 8192, 2), (8192, 8192, 4), (8192, 4096, 8)])
def test_bench_transposes_full_size(axe, R, Cn, es):
    """bench.py's transpose rows at the size it times (K7, the AUTO plan), every byte against the oracle."""
    cfg = dict(name=f"T{R}x{Cn}x{es}", es=es, src=layout([(R, Cn), (Cn, 1)]), src_st=linear_storage(R * Cn),
               dst=layout([(R, 1), (Cn, R)]), dst_st=linear_storage(R * Cn), seed=R + Cn + es)
    d = check(axe, cfg)
    assert d["kernel"] == "transpose", d
    torch.cuda.empty_cache()


def test_bench_nonnested_row_full_size(axe):
    """bench.py's non-nested row at the size it times ((3*2^13, 2*2^13) -> (2*2^13, 3*2^13) bf16, padded, 768
    MiB each side): K8's bulk form, every byte against the oracle (the source storage filled with synth.values
    cell by cell -- padding included -- so the oracle's copy is the only pass over 2^28.6 elements)."""
    g = 1 << 13
    cfg = nonnested_pair(3, 2, g, g, 64, 128, 2)
    cells = synth.storage_cells(cfg["src_st"])
    src = synth.values(cells, 2, cfg["seed"])
    d_fill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * 2, cfg["seed"])
    exp = d_fill.copy()
    oracle.copy(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, 2, NT)
    got, d = run_gpu(axe, cfg, src, d_fill)
    assert d["kernel"] == "dual" and d["bulk"] == 1, d
    if not np.array_equal(got, exp):
        bad = np.nonzero(got != exp)[0]
        raise AssertionError(f"{len(bad)} bytes differ, first at {bad[:8]}")
    del got, exp, src, d_fill
    torch.cuda.empty_cache()


@pytest.mark.parametrize("fuse", ["1", "0"])
@pytest.mark.parametrize("n,t,es,sw", [(4096, 64, 2, synth.SW128), (1024, 64, 2, synth.SW128),
                                       (512, 32, 4, synth.SW128), (512, 64, 1, synth.SW64), (256, 16, 4, synth.SW64),
                                       (256, 8, 4, synth.SW32), (128, 16, 8, synth.SW128)])
def test_lowered_schedule(axe, monkeypatch, n, t, es, sw, fuse):
    """The paper's TMA lowering as the copy schedule (AXE_KERNEL_LOWERED): config-2 re-tilings through
    axe_tma_lower's tensor map and tiler, one TMA load + bulk store per atom (fuse=0) or per fused box."""
    monkeypatch.setenv("AXE_TMA_FUSE", fuse)
    cfg = synth.config2(n, t, es, sw)
    desc = check(axe, cfg, "lowered", "lowered")
    atom = 8 * (16 << sw[0])
    assert desc["atoms"] * atom == n * n * es
    assert desc["box_bytes"] == (atom if fuse == "0" else atom * desc["atoms"] // desc["boxes"])


@pytest.mark.parametrize("n,t,es,sw", [(4096, 64, 2, synth.SW128), (512, 32, 4, synth.SW128), (256, 16, 4, synth.SW64),
                                       (256, 8, 4, synth.SW32)])
def test_lowered_schedule_reverse(axe, n, t, es, sw):
    """Config 2 reversed (swizzled tiles -> row-major) through the lowering's TMA stores."""
    desc = check(axe, synth.config2(n, t, es, sw, True), "lowered", "lowered")
    assert desc["mode"] == "bulk-load/tensor-store"


@pytest.mark.parametrize("pair", ["2", "4", "0"])
@pytest.mark.parametrize("rev", [False, True])
@pytest.mark.parametrize("chunk", ["", "0", "3"])
@pytest.mark.parametrize("n,t,es,sw,reps", [(4096, 64, 2, synth.SW128, 1), (512, 32, 4, synth.SW128, 2),
                                            (512, 64, 1, synth.SW64, 1), (256, 8, 4, synth.SW32, 1)])
def test_lowered_paired_boxes(axe, monkeypatch, pair, rev, chunk, n, t, es, sw, reps):
    """Two (the default) or four consecutive boxes whose image slots are contiguous form one ring unit (one
    TMA tensor op per box, one image-side bulk copy per unit), or one box per unit (AXE_TMA_PAIR=0),
    persistent and in-order grids (3 units per CTA: a ragged last CTA), both directions, destination
    replicas -- against the oracle."""
    monkeypatch.setenv("AXE_TMA_PAIR", pair)
    monkeypatch.setenv("AXE_CHUNK", chunk)
    cfg = synth.config2(n, t, es, sw, rev)
    if reps > 1 and not rev:
        cfg = dict(cfg, name="c2_pair_rep", dst=layout(cfg["dst"]["D"], [(reps, n * n)]),
                   dst_st=linear_storage(reps * n * n, sw))
    desc = check(axe, cfg, "lowered", "lowered")
    assert desc["pair"] in (0, 2, 4) and desc["pair"] <= int(pair), desc
    if n == 4096:   # config 2 itself: 4096 boxes of 8 KiB, consecutive tiles contiguous in the destination
        assert desc["pair"] == int(pair), desc


@pytest.mark.parametrize("kernel", ["lowered", "auto"])
def test_lowered_schedule_destination_replicas(axe, kernel):
    """Config 2 into three replicas of the tiled destination (whole tiles apart): each fused box leaves
    once per replica."""
    n = 512
    cfg = synth.config2(n)
    cfg = dict(cfg, name="c2_rep", dst=layout(cfg["dst"]["D"], [(3, n * n)]),
               dst_st=linear_storage(3 * n * n, synth.SW128))
    d = check(axe, cfg, kernel, "lowered")
    assert d["replicas"] == 3


def test_lowered_schedule_offsets_and_grid_order(axe):
    """Source base offset (a sub-matrix), destination base offset (whole atoms) and tiles stored
    column-of-tiles first: the lowering's tiler T carries the tile order."""
    R, Cn, ld, t, es = 256, 512, 640, 64, 2
    src = layout([(R // t, t * ld), (t, ld), (Cn // t, t), (t, 1)], O={"m": 3 * ld + 64})
    dst = layout([(R // t, t * t), (t, t), (Cn // t, (R // t) * t * t), (t, 1)], O={"m": 2 * t * t})
    cfg = dict(name="lowered_off", es=es, src=src, src_st=linear_storage((R + 3) * ld),
               dst=dst, dst_st=linear_storage(R * Cn + 2 * t * t, synth.SW128), seed=41)
    d = check(axe, cfg, "lowered", "lowered")
    assert d["tensor_map"]["base"] == (3 * ld + 64) * es


@pytest.mark.parametrize("kernel", ["auto", "generic", "vector", "tile", "register", "shuffle"])
@pytest.mark.parametrize("variant", ["a", "b"])
def test_config3_small(axe, variant, kernel):
    if kernel == "shuffle" and variant == "b":  # 3b moves 2-byte elements: no 4-byte granule transpose
        return
    if kernel == "register" and variant == "a":
        with pytest.raises(axe.AxeError):   # 3a moves data across warps: not a movmatrix atom
            axe.CopyPlan(synth.config3(16, "a")["src"], synth.config3(16, "a")["src_st"],
                         synth.config3(16, "a")["dst"], synth.config3(16, "a")["dst_st"], 2, "register")
        return
    d = check(axe, synth.config3(16, variant), kernel)
    if variant == "b" and kernel == "auto":   # K3-TMA: bulk boxes + movmatrix in shared memory
        assert d["kernel"] == "tma" and d["mode"] == "bulk-load/movmatrix/bulk-store", d
    if variant == "a" and kernel == "auto":   # K6: 4 x 4 transposes of 4-byte granules across lanes
        assert d["kernel"] == "shuffle", d


@pytest.mark.parametrize("variant", ["a", "b"])
def test_config3_full_exhaustive(axe, variant):
    """BASELINE config 3 at full size: 65536 tiles of 128x256 bf16 (2^31 elements, 4 GiB each side, tile
    bases above 2^31 bytes), every destination byte against the oracle's copy of the whole batch, through
    the AUTO kernel the bench times (K6 for 3a, K3-TMA for 3b).  The source storage is filled with
    synth.values cell by cell (the register-dump storage is a bijection, so this is a full input; it saves
    the oracle's scatter pass over 2^31 elements)."""
    cfg = synth.config3(65536, variant)
    es = cfg["es"]
    cells = synth.storage_cells(cfg["src_st"])
    src = synth.values(cells, es, cfg["seed"])
    d_fill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, cfg["seed"])
    exp = d_fill.copy()
    oracle.copy(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, es, NT)
    got, d = run_gpu(axe, cfg, src, d_fill)
    assert d["kernel"] == ("shuffle" if variant == "a" else "tma"), d
    if not np.array_equal(got, exp):
        bad = np.nonzero(got != exp)[0]
        raise AssertionError(f"config3{variant}: {len(bad)} bytes differ, first at {bad[:8]}")
    del got, exp, src, d_fill
    torch.cuda.empty_cache()


def nonnested_pair(p, q, g, h, pad_s, pad_d, es, rev=False, reps=1, name="nn"):
    """x in [0, p*q*g*h) read as (p*h, q*g) on the source (row pitch q*g + pad_s) and re-split as
    (q*h, p*g) on the destination (row pitch p*g + pad_d): innermost extents q*g and p*g with
    gcd(p, q) = 1 -- suffix products not nested except through their common factor g."""
    A1, A2, B1, B2 = p * h, q * g, q * h, p * g
    ls, ld = A2 + pad_s, B2 + pad_d
    src = layout([(A1, ls), (A2, 1)])
    if rev:   # the destination rows in reverse order (negative stride on the outer digit)
        dst = layout([(B1, -ld), (B2, 1)], [(reps, B1 * ld)] if reps > 1 else [], {"m": (B1 - 1) * ld})
    else:
        dst = layout([(B1, ld), (B2, 1)], [(reps, B1 * ld)] if reps > 1 else [])
    return dict(name=name, es=es, src=src, src_st=linear_storage(A1 * ls), dst=dst,
                dst_st=linear_storage(reps * B1 * ld), seed=p * 100 + q * 10 + g)


@pytest.mark.parametrize("p,q,g,h,pad_s,pad_d,es,rev,reps", [
    (3, 2, 64, 8, 8, 16, 2, False, 1), (3, 2, 16, 5, 4, 8, 4, True, 1), (5, 3, 32, 3, 4, 4, 8, False, 2),
    (7, 4, 2, 6, 1, 3, 2, False, 1), (3, 2, 8, 4, 2, 6, 16, True, 3), (2, 3, 128, 2, 64, 32, 1, False, 1),
    (3, 2, 4096, 3, 64, 128, 2, False, 1), (5, 2, 2048, 2, 32, 16, 4, True, 2)])
def test_dual_decoding_non_nested(axe, p, q, g, h, pad_s, pad_d, es, rev, reps):
    """K8 on non-nested digit systems (re-pitching reshapes between padded buffers), against the oracle
    and the generic kernel K0; AUTO picks K8 whenever the innermost extents share a factor (g >= 2; both
    pitches padded, else one side is a single run and the pair nests).  g = 4096 / 2048: inner blocks of
    >= 256 vectors, the chunked form (one outer decode per CTA chunk)."""
    cfg = nonnested_pair(p, q, g, h, pad_s, pad_d, es, rev, reps)
    d = check(axe, cfg, "auto")
    assert d["kernel"] == "dual", d
    check(axe, cfg, "generic")


@pytest.mark.parametrize("p,q,h,pad_s,pad_d,es,rev,reps", [
    (3, 2, 40, 1, 3, 2, False, 1), (7, 4, 33, 1, 2, 4, True, 1), (5, 3, 64, 3, 5, 8, False, 2),
    (4096, 2187, 3, 64, 5, 2, False, 1), (2187, 4096, 2, 5, 64, 1, True, 1), (31, 17, 50, 2, 1, 16, False, 3)])
def test_dual_decoding_gcd1_odometer(axe, p, q, h, pad_s, pad_d, es, rev, reps):
    """gcd-1 digit systems (no factor shared even by the fastest pair): K8's odometer form -- per-lane
    carries of both innermost digits, the outer digits re-decoded on wrap -- against the oracle and K0.
    Innermost extents below and above 32 lanes, a reversed destination, replicas, 1..16-byte elements."""
    cfg = nonnested_pair(p, q, 1, h, pad_s, pad_d, es, rev, reps)
    d = check(axe, cfg, "auto")
    assert d["kernel"] == "dual" and d["odometer"] == 1, d
    check(axe, cfg, "generic")


@pytest.mark.parametrize("form", ["bulk", "chunked", "per_vector"])
def test_dual_decoding_large(axe, form, monkeypatch):
    """The bench row's shape at a size that still checks quickly: (3*2^13, 2*2^7) blocks of 2^13 bf16 ->
    (2*2^7, 3*2^13) with padded pitches; K8's bulk form (16 KiB cp.async.bulk boxes), its chunked vector
    form and its per-vector form."""
    monkeypatch.setenv("AXE_K8_BULK", "1" if form == "bulk" else "0")
    monkeypatch.setenv("AXE_K8_CHUNKED", "1" if form == "chunked" else "0")
    cfg = nonnested_pair(3, 2, 8192, 128, 64, 128, 2)
    d = check(axe, cfg, "auto")
    assert d["kernel"] == "dual" and d["vec_bytes"] == 16, d
    assert d["bulk"] == (form == "bulk") and d["chunked"] == (form == "chunked"), d


@pytest.mark.parametrize("p,q,g,h,pad_s,pad_d,es,reps", [
    (3, 2, 64, 8, 8, 16, 2, 1), (5, 3, 32, 3, 4, 4, 8, 2), (3, 2, 8, 4, 2, 6, 16, 3), (2, 3, 1024, 5, 8, 24, 4, 1)])
def test_dual_decoding_bulk_small_runs(axe, p, q, g, h, pad_s, pad_d, es, reps, monkeypatch):
    """K8's bulk form down to 16-byte runs (AXE_K8_BULK_MIN_RUN=16), with destination replicas, and runs
    longer than one 16 KiB box (g = 1024 fp32: 12 / 8 KiB runs)."""
    monkeypatch.setenv("AXE_K8_BULK_MIN_RUN", "16")
    cfg = nonnested_pair(p, q, g, h, pad_s, pad_d, es, False, reps)
    d = check(axe, cfg, "auto")
    assert d["kernel"] == "dual" and d["bulk"] == 1, d


def test_identity_and_transpose_reduce_to_torch(axe):
    """Special cases that reduce to library routines: identity = clone, row->column major = .t()."""
    R, Cn = 1000, 777
    x = torch.randint(-2**15, 2**15 - 1, (R, Cn), dtype=torch.int16, device="cuda")
    y = torch.empty_like(x)
    axe.axe_copy(layout([(R, Cn), (Cn, 1)]), linear_storage(R * Cn), x, layout([(R, Cn), (Cn, 1)]),
                 linear_storage(R * Cn), y, 2)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    z = torch.empty(Cn, R, dtype=torch.int16, device="cuda")
    axe.axe_copy(layout([(R, Cn), (Cn, 1)]), linear_storage(R * Cn), x, layout([(R, 1), (Cn, R)]),
                 linear_storage(R * Cn), z, 2)
    torch.cuda.synchronize()
    assert torch.equal(z, x.t().contiguous())


def test_tiling_reduces_to_torch_permute(axe):
    n, t = 1024, 64
    x = torch.randint(-2**31, 2**31 - 1, (n, n), dtype=torch.int32, device="cuda")
    y = torch.empty_like(x)
    cfg = synth.config2(n, t, 4, (0, 0, 0))
    axe.axe_copy(cfg["src"], cfg["src_st"], x, cfg["dst"], cfg["dst_st"], y, 4)
    torch.cuda.synchronize()
    assert torch.equal(y.view(-1), x.view(n // t, t, n // t, t).permute(0, 2, 1, 3).contiguous().view(-1))


def rand_injective(rng, N_exts, allow_neg=True, reps=True):
    """A random injective layout over extents N_exts on axis m: a mixed radix in random order with gaps,
    optional negative strides (offset compensates) and replicas beyond the shard span."""
    n = len(N_exts)
    order = rng.permutation(n)
    strides = [0] * n
    cur = 1
    for i in order:
        strides[i] = cur
        cur *= N_exts[i] * int(rng.choice([1, 1, 1, 2]))
    O = 0
    D = []
    for i in range(n):
        s = strides[i]
        if allow_neg and rng.random() < 0.2:
            O += (N_exts[i] - 1) * s
            s = -s
        D.append((N_exts[i], s))
    R = []
    if reps and rng.random() < 0.4:
        e = int(rng.integers(2, 4))
        R.append((e, cur))
        cur *= e
    return layout(D, R, {"m": O} if O else {}), cur


def random_split(rng, N):
    exts = []
    while N > 1:
        for f in (2, 3, 4, 5, 8):
            if N % f == 0 and rng.random() < 0.5:
                exts.append(f)
                N //= f
                break
        else:
            exts.append(N)
            N = 1
    return exts or [1]


@pytest.mark.parametrize("seed", range(40))
def test_random_layout_pairs(axe, seed):
    """Brute force on small random pairs: every kernel the planner can pick, and the generic kernel."""
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.choice([64, 96, 120, 256, 360, 512, 1024]))
    es = int(rng.choice([1, 2, 4, 8, 16]))
    src, sc = rand_injective(rng, random_split(rng, N), reps=False)
    dst, dc = rand_injective(rng, random_split(rng, N))
    sw = (0, 0, 0)
    if rng.random() < 0.3 and (dc * es) % 1024 == 0:
        sw = synth.SW128
    cfg = dict(name=f"rand{seed}", es=es, src=src, src_st=linear_storage(sc), dst=dst,
               dst_st=linear_storage(dc, sw), seed=seed)
    check(axe, cfg, "auto")
    check(axe, cfg, "generic")
    if axe.CopyPlan(src, cfg["src_st"], dst, cfg["dst_st"], es).describe()["kernel"] not in ("generic", "dual"):
        check(axe, cfg, "vector")
    try:
        axe.CopyPlan(src, cfg["src_st"], dst, cfg["dst_st"], es, "tile")
    except axe.AxeError:
        return
    check(axe, cfg, "tile")


@pytest.mark.parametrize("R,Cn,es", [(256, 512, 2), (512, 256, 4), (128, 384, 8), (256, 256, 1), (64, 96, 16),
                                     (1024, 64, 2)])
def test_transposes_all_kernels(axe, R, Cn, es):
    """Row-major -> column-major at every element size through K2 (smem tile), K1 and the generic kernel."""
    cfg = dict(name=f"T{R}x{Cn}x{es}", es=es, src=layout([(R, Cn), (Cn, 1)]), src_st=linear_storage(R * Cn),
               dst=layout([(R, 1), (Cn, R)]), dst_st=linear_storage(R * Cn), seed=R + es)
    for k in ("auto", "vector", "generic"):
        check(axe, cfg, k)
    for k in ("tile",):
        try:
            axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, k)
        except axe.AxeError:
            continue
        check(axe, cfg, k)


@pytest.mark.parametrize("es,cw", [(2, 1), (2, 2), (4, 1), (4, 2), (4, 4), (8, 1), (8, 2), (8, 4)])
@pytest.mark.parametrize("asyn", [0, 2, 3])
def test_k7_batched_padded_transposes(axe, monkeypatch, es, cw, asyn):
    """K7 directly: 3 batched transposes of (2 TR) x (3 TC) tiles, padded source rows and destination columns,
    two destination replicas; every chunk width, the register-staged form and the cp.async rings of 2 and 3
    stages (several tiles per CTA, so every buffer is refilled)."""
    monkeypatch.setenv("AXE_K7_CW", str(cw))
    monkeypatch.setenv("AXE_K7_ASYNC", str(asyn))
    monkeypatch.setenv("AXE_K7_MAX_CTAS", "4")
    n = 16 // es
    cw = min(cw, 2 if es == 2 else 4)   # the widest chunk column the planner takes for this element size
    R, C = 2 * 32 * n, 3 * 8 * n * cw
    lds, ldd = C + n, R + 2 * n
    B = 3
    src = layout([(B, R * lds), (R, lds), (C, 1)])
    dst = layout([(B, C * ldd), (R, 1), (C, ldd)], [(2, B * C * ldd)])
    cfg = dict(name=f"k7_{es}_{cw}_{asyn}", es=es, src=src, src_st=linear_storage(B * R * lds), dst=dst,
               dst_st=linear_storage(2 * B * C * ldd), seed=es * 10 + cw)
    desc = check(axe, cfg, "transpose", "transpose")
    assert desc["async"] == asyn and desc["replicas"] == 2 and desc["tile"] == [32 * n, 8 * n * cw]
    assert desc["tiles"] == B * 2 * 3 and desc["ctas"] == 4


@pytest.mark.parametrize("chain", [0, 1, 2])
@pytest.mark.parametrize("kernel", ["auto", "vector", "generic"])
def test_storage_divisor_chains(axe, chain, kernel):
    """Destination storages that split the m axis over several digits (the oracle's pin:
    test_storage_divisor_chain_is_numpy_blocking) at a size the kernels tile: 4096 x 24 bf16."""
    M, Nn = 4096, 24
    st = [storage([("m", 16, 256), ("n", Nn), ("m", 256, 1)]),
          storage([("m", 2, 2048), ("n", Nn), ("m", 8, 256), ("m", 256, 1)]),
          storage([("m", 64, 64), ("m", 64, 1), ("n", Nn)])][chain]
    cfg = dict(name=f"chain{chain}", es=2, src=layout([(M, Nn), (Nn, 1)]), src_st=linear_storage(M * Nn),
               dst=layout([(M, 1, "m"), (Nn, 1, "n")]), dst_st=st, seed=80 + chain)
    check(axe, cfg, kernel)


def _in_order_cases():
    n8 = 16 // 8
    R, C = 2 * 32 * n8, 3 * 8 * n8 * 4
    k7 = dict(name="k7_chunk", es=8, src=layout([(3, R * (C + 2)), (R, C + 2), (C, 1)]),
              src_st=linear_storage(3 * R * (C + 2)), dst=layout([(3, C * R), (R, 1), (C, R)], [(2, 3 * C * R)]),
              dst_st=linear_storage(2 * 3 * C * R), seed=71)
    rows, cols, run = 96, 2048, 256           # 512-byte runs of a padded 2-byte matrix, column blocks first
    gat = dict(name="gather_chunk", es=2, src=layout([(cols // run, run), (rows, cols + 64), (run, 1)]),
               src_st=linear_storage(rows * (cols + 64)), dst=layout([(cols // run, rows * run), (rows, run), (run, 1)]),
               dst_st=linear_storage(rows * cols), seed=72)
    ne = 3 * 65536 + 4096                     # identity, 16-byte vectors / 16 KiB bulk boxes and a short tail box
    ident = dict(name="ident_chunk", es=4, src=layout([(ne, 1)]), src_st=linear_storage(ne), dst=layout([(ne, 1)]),
                 dst_st=linear_storage(ne), seed=73)
    k9 = dict(name="k9_chunk", es=2, src=layout([(2, 131 * 259), (131, 259), (257, 1)]),   # odd extents: K9
              src_st=linear_storage(2 * 131 * 259), dst=layout([(2, 257 * 133), (131, 1), (257, 133)]),
              dst_st=linear_storage(2 * 257 * 133), seed=74)
    lw = synth.config2(512)                   # the lowered schedule: 64 fused 8 KiB boxes
    return [("tile", gat, "tile", "tile"), ("dual_pervec", nonnested_pair(3, 2, 16, 4, 8, 4, 2, name="dual_pv"), "dual", "dual"),
            ("k9", k9, "transpose", "transpose"), ("lowered", lw, "lowered", "lowered"), ("lowered_r", synth.config2(512, reverse=True), "lowered", "lowered"),
            ("k7", k7, "transpose", "transpose"), ("vector", gat, "vector", "vector"), ("tma", gat, "tma", "tma"),
            ("bulk", ident, "tma", "tma"), ("shuffle", synth.config3(64, "a"), "shuffle", "shuffle"),
            ("k3tma", synth.config3(64, "b"), "auto", "tma"),
            ("dual", nonnested_pair(3, 2, 2048, 4, 64, 32, 2, name="dual_chunk"), "auto", "dual")]


@pytest.mark.parametrize("case", range(12))
@pytest.mark.parametrize("chunk", ["1", "2", "3", "5"])
def test_in_order_schedule_every_kernel(axe, monkeypatch, case, chunk):
    """The in-order schedule (kernels.cuh unit_range: `chunk` consecutive units per CTA over a covering grid)
    forced on every kernel that has it, with unit counts that leave the last CTA ragged: byte-exact against
    the oracle, like the persistent grid."""
    monkeypatch.setenv("AXE_CHUNK", chunk)
    monkeypatch.setenv("AXE_K7_ASYNC", "3")
    name, cfg, kernel, expect = _in_order_cases()[case]
    if name == "dual_pervec":   # K8's per-vector form (neither bulk boxes nor chunked items)
        monkeypatch.setenv("AXE_K8_BULK", "0")
        monkeypatch.setenv("AXE_K8_CHUNKED", "0")
    desc = check(axe, cfg, kernel, expect)
    if "chunk" in desc:
        assert desc["chunk"] == int(chunk), desc


def test_alias_and_alignment_errors(axe):
    x = torch.zeros(1024, dtype=torch.int32, device="cuda")
    L = layout([(512, 1)])
    st = linear_storage(512)
    with pytest.raises(axe.AxeError) as e:
        axe.axe_copy(L, st, x, L, st, x[256:], 4)
    assert e.value.name == "AXE_ERR_ALIAS"
    plan = axe.CopyPlan(L, st, L, st, 4)
    with pytest.raises(axe.AxeError) as e:
        plan.execute(x[1:], x[600:])     # 4-byte offset breaks the 16-byte vector plan
    assert e.value.name == "AXE_ERR_ALIGNMENT"
    y = torch.zeros(1100, dtype=torch.int32, device="cuda")
    axe.axe_copy(L, st, x[1:], L, st, y[3:], 4)     # the cached path re-plans for 4-byte alignment
    torch.cuda.synchronize()
    assert torch.equal(y[3:515], x[1:513])


@pytest.mark.parametrize("kernel", ["auto", "vector"])
def test_dependent_chain_with_pdl(axe, kernel):
    """Back-to-back dependent copies on one stream (RAW and WAR hazards between consecutive kernels) stay
    exact with programmatic dependent launch: forward/reverse config-2 chains return the input."""
    n = 1024
    fwd, rev = synth.config2(n), synth.config2(n, reverse=True)
    pf = axe.CopyPlan(fwd["src"], fwd["src_st"], fwd["dst"], fwd["dst_st"], 2, kernel)
    pr = axe.CopyPlan(rev["src"], rev["src_st"], rev["dst"], rev["dst_st"], 2, kernel)
    x = torch.randint(-2**31, 2**31 - 1, (n * n // 2,), dtype=torch.int32, device="cuda")
    a, b, c = x.clone(), torch.empty_like(x), torch.empty_like(x)
    for _ in range(50):
        pf.execute(a, b)      # b <- tiles(a)
        pr.execute(b, c)      # RAW on b
        pf.execute(c, a)      # RAW on c, WAR... a is rewritten after being read two kernels ago
        pr.execute(a, b)      # b <- rowmajor(a) = x
        pf.execute(b, a)      # WAR on a (read by the previous kernel) and RAW on b
        pr.execute(a, c)
        a, c = c, a
    torch.cuda.synchronize()
    assert torch.equal(a, x)
    # independent copies interleaved with dependent ones
    outs = [torch.empty_like(x) for _ in range(4)]
    for i in range(40):
        pf.execute(x, outs[i % 4])
    pr.execute(outs[1], c)
    torch.cuda.synchronize()
    assert torch.equal(c, x)


def test_prefetch_before_wait_raw_chains(axe):
    """The kernels prefetch their first boxes / tiles into L2 BEFORE griddepcontrol.wait (reading R28), i.e.
    while the previous kernel may still be writing those very bytes.  RAW chains at the bench's size:
    forward (lowered, TMA tensor loads + L2 tensor prefetch) then reverse (lowered, bulk prefetch) then K7
    transposes there and back (line prefetches), each reading what the kernel before it is writing; fresh
    data every round, compared at the end of every round."""
    n = 4096
    fwd, rev = synth.config2(n), synth.config2(n, reverse=True)
    pf = axe.CopyPlan(fwd["src"], fwd["src_st"], fwd["dst"], fwd["dst_st"], 2)
    pr = axe.CopyPlan(rev["src"], rev["src_st"], rev["dst"], rev["dst_st"], 2)
    rm, cm = layout([(n, n), (n, 1)]), layout([(n, 1), (n, n)])
    pt = axe.CopyPlan(rm, linear_storage(n * n), cm, linear_storage(n * n), 2)
    ptb = axe.CopyPlan(cm, linear_storage(n * n), rm, linear_storage(n * n), 2, "transpose")
    assert pf.describe()["kernel"] == "lowered" and pr.describe()["kernel"] == "lowered"
    assert pt.describe()["kernel"] == "transpose"
    g = torch.Generator(device="cuda").manual_seed(5)
    a, b, c, d = (torch.empty(n * n // 2, dtype=torch.int32, device="cuda") for _ in range(4))
    for _ in range(30):
        x = torch.randint(-2**31, 2**31 - 1, (n * n // 2,), dtype=torch.int32, device="cuda", generator=g)
        a.copy_(x)
        pf.execute(a, b)     # b <- tiles(a)
        pr.execute(b, c)     # c <- rowmajor(b) = x      (reads b while pf may still write it)
        pt.execute(c, d)     # d <- c^T                  (reads c while pr may still write it)
        ptb.execute(d, a)    # a <- d^T = x              (reads d while pt may still write it)
        torch.cuda.synchronize()
        assert torch.equal(c, x) and torch.equal(a, x)


def test_lowered_schedule_in_pdl_chains(axe):
    """The lowered schedule joins the PDL window like every copy kernel: dependent chains forward
    (lowered) / reverse (TMA store) return the input; independent lowered copies overlap."""
    n = 1024
    fwd, rev = synth.config2(n), synth.config2(n, reverse=True)
    pf = axe.CopyPlan(fwd["src"], fwd["src_st"], fwd["dst"], fwd["dst_st"], 2, "lowered")
    pr = axe.CopyPlan(rev["src"], rev["src_st"], rev["dst"], rev["dst_st"], 2)
    x = torch.randint(-2**31, 2**31 - 1, (n * n // 2,), dtype=torch.int32, device="cuda")
    a, b, c = x.clone(), torch.empty_like(x), torch.empty_like(x)
    for _ in range(50):
        pf.execute(a, b)
        pr.execute(b, c)
        pf.execute(c, a)
        pr.execute(a, b)
        pf.execute(b, a)
        pr.execute(a, c)
        a, c = c, a
    torch.cuda.synchronize()
    assert torch.equal(a, x)
    outs = [torch.empty_like(x) for _ in range(4)]
    for i in range(40):
        pf.execute(x, outs[i % 4])
    pr.execute(outs[1], c)
    torch.cuda.synchronize()
    assert torch.equal(c, x)


def test_launch_counter(axe):
    x = torch.zeros(4096, dtype=torch.int16, device="cuda")
    y = torch.zeros_like(x)
    n0 = axe.kernel_launch_count()
    for _ in range(3):
        axe.axe_copy(layout([(4096, 1)]), linear_storage(4096), x, layout([(4096, 1)]), linear_storage(4096), y, 2)
    assert axe.kernel_launch_count() - n0 == 3


def test_execute_host_e2e(axe):
    cfg = synth.config2(512, 64)
    src, d_fill, exp = prepare(cfg)
    plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2)
    hs = torch.from_numpy(src).pin_memory()
    hd = torch.from_numpy(d_fill.copy()).pin_memory()
    ds = torch.empty(src.nbytes, dtype=torch.uint8, device="cuda")
    dd = torch.empty(d_fill.nbytes, dtype=torch.uint8, device="cuda")
    plan.execute_host(hs, hd, ds, dd)
    torch.cuda.synchronize()
    assert np.array_equal(hd.numpy(), exp)


@pytest.mark.parametrize("seed", range(16))
def test_random_permutes_reduce_to_numpy(axe, seed):
    """Random N-d permutations (numpy.transpose semantics): src row-major (s0..sn), dst row-major over the
    permuted dims.  Every kernel that can run the pair must produce numpy's transpose exactly."""
    rng = np.random.default_rng(77 + seed)
    nd = int(rng.integers(2, 5))
    shape = [int(rng.choice([2, 4, 8, 16, 32, 64, 128])) for _ in range(nd)]
    while np.prod(shape) < 4096:
        shape[int(rng.integers(0, nd))] *= 2
    while np.prod(shape) > (1 << 20):
        i = int(np.argmax(shape))
        shape[i] //= 2
    perm = list(rng.permutation(nd))
    es = int(rng.choice([1, 2, 4, 8]))
    N = int(np.prod(shape))
    rs = [int(np.prod(shape[i + 1:])) for i in range(nd)]            # row-major strides of the source
    pshape = [shape[p] for p in perm]
    prs = [int(np.prod(pshape[i + 1:])) for i in range(nd)]          # row-major strides of the destination
    dst_stride = [0] * nd
    for i, p in enumerate(perm):
        dst_stride[p] = prs[i]
    src = layout([(shape[i], rs[i]) for i in range(nd)])
    dst = layout([(shape[i], dst_stride[i]) for i in range(nd)])
    dt = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[es]
    v = synth.values(N, es, seed)
    expect = np.ascontiguousarray(v.view(dt).reshape(shape).transpose(perm)).reshape(-1)
    for kernel in ("auto", "vector", "tile", "generic"):
        try:
            plan = axe.CopyPlan(src, linear_storage(N), dst, linear_storage(N), es, kernel)
        except axe.AxeError:
            continue
        s = torch.from_numpy(v.copy()).cuda()
        d = torch.zeros_like(s)
        plan.execute(s, d)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy().view(dt), expect), (kernel, shape, perm, es, plan.describe())


@pytest.mark.parametrize("case", ["config2", "config2r", "padded"])
def test_execute_host_pipelined(axe, case):
    """axe_copy_plan_execute_host with the slab pipeline (H2D / kernel / D2H on three streams): host-to-host
    result equals the oracle, including destination cells outside the image (padded rows keep the sentinel)."""
    if case == "padded":
        n, pitch = 2048, 2056
        cfg = dict(name="padded", es=2, src=layout([(n, n), (n, 1)]), src_st=linear_storage(n * n),
                   dst=layout([(n, pitch), (n, 1)]), dst_st=linear_storage(n * pitch), seed=4)
    else:
        cfg = synth.config2(reverse=case == "config2r")
    src, d_fill, exp = prepare(cfg)
    plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2)
    assert plan.describe().get("host_chunks", 0) >= 2, plan.describe()
    hs = torch.from_numpy(src).pin_memory()
    hd = torch.from_numpy(d_fill.copy()).pin_memory()
    ds = torch.empty(src.nbytes, dtype=torch.uint8, device="cuda")
    dd = torch.empty(d_fill.nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        plan.execute_host(hs, hd, ds, dd)
    torch.cuda.synchronize()
    assert np.array_equal(hd.numpy(), exp)


@pytest.mark.parametrize("slabs", [2, 4])
def test_execute_host_alternating_streams(axe, slabs):
    """The serving pattern bench.py's e2e uses: consecutive execute_host calls of one plan (host_slabs set
    through axe_copy_plan_create_ex) on two user streams with two host / device buffer sets, so one call's
    host->device copies overlap the previous call's device->host copies.  Every call's result is exact."""
    cfg = synth.config2()
    src, d_fill, exp = prepare(cfg)
    plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, host_slabs=slabs)
    assert plan.describe()["host_chunks"] == slabs
    srcs = [src, np.ascontiguousarray(src[::-1])]       # a second, different input
    exps = [exp]
    e2 = d_fill.copy()
    oracle.copy(cfg["src"], cfg["src_st"], srcs[1], cfg["dst"], cfg["dst_st"], e2, 2)
    exps.append(e2)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    hs = [torch.from_numpy(s).pin_memory() for s in srcs]
    hd = [torch.from_numpy(d_fill.copy()).pin_memory() for _ in range(2)]
    ds = [torch.empty(src.nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    dd = [torch.empty(d_fill.nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    for i in range(6):
        k = i % 2
        plan.execute_host(hs[k], hd[k], ds[k], dd[k], streams[k])
    torch.cuda.synchronize()
    for k in range(2):
        assert np.array_equal(hd[k].numpy(), exps[k])


def test_tma_small_boxes_regression(axe):
    """Found by tools/fuzz_gpu.py (case 1540651327): a TMA plan with 64-byte boxes placed ring slots 64 B
    apart, but TMA needs 128-byte aligned shared-memory destinations (misaligned address).  Slots are now
    rounded up to 128 B (1024 B when swizzled)."""
    src = layout([(2, 16384), (2, 1), (2, 131072), (2, 65536), (4096, 4)])
    dst = layout([(4, 1), (2, 32768), (8192, 4)])
    cfg = dict(name="tma64", es=16, src=src, src_st=linear_storage(262144), dst=dst, dst_st=linear_storage(65536),
               seed=11)
    d = axe.CopyPlan(src, cfg["src_st"], dst, cfg["dst_st"], 16, "tma").describe()  # AUTO now prefers K1 here
    assert d["kernel"] == "tma" and d["box_bytes"] == 64
    check(axe, cfg, "tma")


def test_concurrent_streams_from_threads(axe):
    """Two host threads, each on its own stream, issue one-shot axe_copy calls (shared plan cache and PDL
    bookkeeping) back to back; every result is exact."""
    import threading
    cfgs = [synth.config2(512), synth.config2(512, reverse=True)]
    data = []
    for c in cfgs:
        src, d_fill, exp = prepare(c)
        data.append((c, torch.from_numpy(src).cuda(), d_fill, exp))
    errors = []

    def work(i):
        try:
            c, s, d_fill, exp = data[i]
            st = torch.cuda.Stream()
            outs = [torch.from_numpy(d_fill).cuda() for _ in range(4)]
            with torch.cuda.stream(st):
                for rep in range(25):
                    axe.axe_copy(c["src"], c["src_st"], s, c["dst"], c["dst_st"], outs[rep % 4], c["es"], st)
            st.synchronize()
            for o in outs:
                assert np.array_equal(o.cpu().numpy(), exp)
        except Exception as e:
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_pdl_window_two_launches_back(axe):
    """Regression (tools/pdl_chain_probe.py): A writes X (a 256 MiB copy), B touches unrelated buffers, C reads
    the tail of X.  C must not skip griddepcontrol.wait just because it is disjoint from B: B itself did not
    wait, so A may still be running.  The per-stream window of in-flight ranges catches it."""
    N, n = 1 << 27, 1 << 12
    big = axe.CopyPlan(layout([(N, 1)]), linear_storage(N), layout([(N, 1)]), linear_storage(N), 2)
    small = axe.CopyPlan(layout([(n, 1)]), linear_storage(n), layout([(n, 1)]), linear_storage(n), 2)
    readc = axe.CopyPlan(layout([(n, 1)], O={"m": N - n}), linear_storage(N), layout([(n, 1)]), linear_storage(n), 2)
    S = torch.full((N,), 7, dtype=torch.int16, device="cuda")
    X = torch.zeros(N, dtype=torch.int16, device="cuda")
    a, b = torch.zeros(n, dtype=torch.int16, device="cuda"), torch.zeros(n, dtype=torch.int16, device="cuda")
    Y = torch.zeros(n, dtype=torch.int16, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(20):
        X.zero_()
        Y.fill_(-1)
        torch.cuda.synchronize()
        big.execute(S, X, st)
        small.execute(a, b, st)
        readc.execute(X, Y, st)
        torch.cuda.synchronize()
        assert bool((Y == 7).all())


def test_k3_tma_with_destination_replicas(axe):
    """K3-TMA with two destination replicas (the permuted 3b tiles written twice, 16 tiles apart on the cta
    axis): every box is stored once per replica after the in-smem movmatrix."""
    tiles = 16
    dst = synth.config3b_dst(tiles)
    dst = layout(dst["D"], [(2, tiles, "cta")], dst["O"])
    cfg = dict(name="3b_rep", es=2, src=synth.config3_src(tiles), src_st=synth._regdump_storage(tiles), dst=dst,
               dst_st=synth._regdump_storage(2 * tiles), seed=13)
    d = check(axe, cfg, "auto")
    assert d["kernel"] == "tma" and d["replicas"] == 2, d


@pytest.mark.parametrize("n", [1, 2, 3, 7, 31, 33])
@pytest.mark.parametrize("es", [1, 2, 4, 8, 16])
def test_degenerate_sizes(axe, n, es):
    """Tiny and odd sizes (the degenerate cases of every kernel): a single element, odd extents, a reversed
    order with an offset, and a replicated destination -- every forced kernel that accepts the plan."""
    src = layout([(n, 1)])
    dst = layout([(n, -1)], [(2, n)], {"m": n - 1})
    cfg = dict(name=f"tiny{n}x{es}", es=es, src=src, src_st=linear_storage(n), dst=dst,
               dst_st=linear_storage(2 * n + 3), seed=n * 16 + es)
    check(axe, cfg, "auto")
    for k in ("generic", "vector", "tile", "tma", "register", "dual"):
        try:
            axe.CopyPlan(src, cfg["src_st"], dst, cfg["dst_st"], es, k)
        except axe.AxeError:
            continue
        check(axe, cfg, k)


@pytest.mark.parametrize("K,n", [(1, 1), (2, 1), (3, 5), (5, 3), (300, 1)])
def test_degenerate_reductions(axe, K, n):
    """Reductions with one output element, odd extents, and K > 256 over a single element."""
    cfg = synth.reduce_local(K, 1, n, "i32")
    vals = synth.numbers(K * n, "i32", K + n)
    fill = synth.sentinel(n * 4, 3)
    exp = fill.copy()
    oracle.reduce(cfg["src"], cfg["src_st"], vals, cfg["dst"], cfg["dst_st"], exp, "i32")
    s_dev, d_dev = torch.from_numpy(vals.copy()).cuda(), torch.from_numpy(fill.copy()).cuda()
    axe.ReducePlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], "i32").execute(s_dev, d_dev)
    torch.cuda.synchronize()
    assert np.array_equal(d_dev.cpu().numpy(), exp)
