"""Host-side tests of libaxe (no GPU): the library loads and exports every symbol
include/axe.h declares; layout creation / evaluation / bounds / canonicalisation
agree with the independent oracle; copy planning validates and chooses kernels.
No compute call (kernel launch) happens here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage, storage

import paper_2601_19092_b200 as axe

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    with open(os.path.join(ROOT, "include", "axe.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"^\s*(?:axe_status|void|const char \*|int64_t)\s*\*?\s*(axe_\w+)\(", txt, re.M)))


def test_every_header_symbol_is_exported():
    names = header_functions()
    assert len(names) >= 25
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2601_19092_b200", "libaxe.so"))
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(axe.EXPORTED)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_2601_19092_b200", "libaxe.so")], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def sets(coords):
    return sorted(sorted((a, v) for a, v in c.items() if v != 0) for c in coords)


def rand_layout(rng, axes=("m", "lane", "warp")):
    D = [(int(rng.integers(1, 7)), int(rng.choice([-1, 1]) * rng.integers(1, 24)), str(rng.choice(axes)))
         for _ in range(rng.integers(1, 5))]
    R = [(int(rng.integers(1, 4)), int(rng.choice([-1, 1]) * rng.integers(1, 24)), str(rng.choice(axes)))
         for _ in range(rng.integers(0, 3))]
    O = {str(a): int(rng.integers(-5, 6)) for a in rng.choice(axes, size=rng.integers(0, 3))}
    return layout(D, R, O)


def test_eval_matches_oracle_random():
    rng = np.random.default_rng(1)
    for _ in range(300):
        spec = rand_layout(rng)
        L = axe.Layout(spec=spec)
        ed, er = oracle.sizes(spec)
        assert (L.E_D, L.E_R) == (ed, er)
        for x in range(0, ed, max(1, ed // 5)):
            assert sets(L.eval(x)) == sets(oracle.eval(spec, x))


def test_bounds_match_oracle_bruteforce():
    rng = np.random.default_rng(2)
    for _ in range(200):
        spec = rand_layout(rng)
        L = axe.Layout(spec=spec)
        for a in ("m", "lane", "warp"):
            b = oracle.bounds(spec, a)
            assert L.bounds(a) == (b if b is not None else (0, 0))


def test_canonicalize_preserves_map_and_is_idempotent():
    """Prop.: D0/D1 and C0-C2 preserve f_L; the fixpoint is stable."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        spec = rand_layout(rng)
        L = axe.Layout(spec=spec)
        Cn, _ = L.canonicalize()
        cs = Cn.spec()
        for x in range(L.E_D):
            assert sets(oracle.eval(cs, x)) == sets(oracle.eval(spec, x)), (spec, cs)
        C2, _ = Cn.canonicalize()
        assert C2.spec() == cs


@pytest.mark.parametrize("D,exp", [
    ([(2, 8), (8, 1)], [(16, 1, "m")]),                              # SPEC S:164 (D1)
    ([(1, 5), (4, 1)], [(4, 1, "m")]),                               # D0
    ([(2, 192), (8, 8), (3, 64), (8, 1)], [(2, 192, "m"), (8, 8, "m"), (3, 64, "m"), (8, 1, "m")]),
    ([(4, 4), (2, 2), (2, 1)], [(16, 1, "m")]),                      # App. F chain
    ([(4096, 4096), (4096, 1)], [(16777216, 1, "m")]),               # SURVEY §8(a) a2, config 2 source
])
def test_canonical_shard_examples(D, exp):
    Cn, _ = axe.Layout(D).canonicalize()
    assert Cn.iters(0) == exp


def test_canonical_replica_examples():
    """C1 flips a negative stride into O; C2 with q = e_i (reading R9): [(2,1),(3,2)] -> [(6,1)]."""
    Cn, gc = axe.Layout([(2, 1)], [(3, -2)]).canonicalize()
    assert Cn.iters(1) == [(3, 2, "m")] and Cn.offset() == {"m": -4}
    Cn, gc = axe.Layout([(2, 100)], [(2, 1), (3, 2)]).canonicalize()
    assert Cn.iters(1) == [(6, 1, "m")] and gc
    Cn, gc = axe.Layout([(2, 100)], [(3, 2), (2, 3)]).canonicalize()   # GC fails: 3 <= 3*2
    assert not gc


def test_layout_errors():
    with pytest.raises(axe.AxeError) as e:
        axe.Layout([(4, 0)])
    assert e.value.name == "AXE_ERR_INVALID_ARG"
    with pytest.raises(axe.AxeError) as e:
        axe.Layout([])
    assert e.value.name == "AXE_ERR_INVALID_ARG"
    with pytest.raises(axe.AxeError) as e:
        axe.Layout([(4, 1, "9bad")])
    assert e.value.name == "AXE_ERR_INVALID_ARG"
    with pytest.raises(axe.AxeError) as e:
        axe.Layout([(1 << 40, 1), (1 << 40, 1)])
    assert e.value.name == "AXE_ERR_OVERFLOW"
    with pytest.raises(axe.AxeError) as e:
        axe.Layout([(4, 1)]).eval(4)
    assert e.value.name == "AXE_ERR_DOMAIN"


# --------------------------------------------------------------------------- planning
def plan(cfg, kernel="auto"):
    return axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["es"], kernel)


def test_config2_plan_is_tma_box_copy():
    """Config 2 lowers to the paper's TMA recipe: AUTO runs the lowering itself (slice ->
    tile_of the SW128 atom -> tensor map; 8 atoms fused per 64-row box); the joint-digit TMA planner
    (forced "tma") finds the same 64 x 128 B boxes."""
    d = plan(synth.config2()).describe()
    assert d["kernel"] == "lowered" and d["atoms"] == 32768 and d["boxes"] == 4096 and d["box_bytes"] == 8192
    assert d["swizzle"] == 128 and d["tensor_map"]["box"] == [64, 8, 8, 1, 1]
    # joint digits (64:262144|262144),(64:4096|64),(64:64|4096),(64:1|1)
    assert d["joint"] == [[64, 262144, 262144], [64, 4096, 64], [64, 64, 4096], [64, 1, 1]]
    t = plan(synth.config2(), "tma").describe()
    assert t["kernel"] == "tma" and t["box"] == [64, 128] and t["boxes"] == 4096 and t["swizzle"] == 128
    r = plan(synth.config2(reverse=True)).describe()
    assert r["kernel"] == "lowered" and r["mode"] == "bulk-load/tensor-store"
    assert plan(synth.config2(reverse=True), "tma").describe()["mode"] == "bulk-load/tensor-store"


def test_config2_vector_plan():
    d = plan(synth.config2(), "vector").describe()
    assert d["kernel"] == "vector" and d["vec_bytes"] == 16 and d["vectors"] == 4096 * 4096 // 8


def test_config1_plan():
    d = plan(synth.config1()).describe()
    assert d["kernel"] == "vector" and d["replicas"] == 2 and d["vec_bytes"] == 16


def test_config3_plans_are_affine():
    for v in "ab":
        d = plan(synth.config3(64, v)).describe()
        # 3a: 4 x 4 transposes of 4-byte granules across lanes (K6); 3b: the movmatrix atom on bulk-copied
        # boxes in shared memory (K3-TMA); a forced "register" plan is the register kernel K3
        assert d["kernel"] == {"a": "shuffle", "b": "tma"}[v], d
    assert plan(synth.config3(64, "b"), "register").describe()["kernel"] == "register"


def test_nonnested_gcd1_decodes_both_sides_per_element():
    """(2,3):(1,2) vs (3,2):(1,3): suffix products {1,3,6} vs {1,2,6} are not nested and the innermost extents
    share no factor (SURVEY §7 hard part 3): K8 with an empty inner block, both digit lists decoded per
    element with fast divisions (the generic K0 stays for non-affine storage compositions)."""
    src, dst = layout([(2, 1), (3, 2)]), layout([(3, 1), (2, 3)])
    d = axe.CopyPlan(src, linear_storage(6), dst, linear_storage(6), 4).describe()
    assert d["kernel"] == "dual" and d["inner_block_vectors"] == 1 and d["vec_bytes"] == 4, d


def test_nonnested_with_common_factor_plans_dual():
    """(6, 8) padded -> (4, 12) padded: innermost extents 8 and 12 do not nest but share 4 -- K8 keeps the
    4-element run (8 bytes of 2-byte elements here) as its vector and decodes the outer index twice."""
    src = layout([(6, 12), (8, 1)])
    dst = layout([(4, 16), (12, 1)])
    d = axe.CopyPlan(src, linear_storage(72), dst, linear_storage(64), 2).describe()
    assert d["kernel"] == "dual" and d["vec_bytes"] == 8, d
    assert d["inner"] == [[4, 1, 1]] and d["outer_blocks"] == 12, d
    assert d["outer_src"] == [[6, 12], [2, 4]] and d["outer_dst"] == [[4, 16], [3, 4]], d


def test_ragged_transposes_plan_k9():
    """Transposes K7 cannot take (rows not whole 16-byte vectors) and K2 cannot tile (4095 = 3^2.5.7.13,
    4097 = 17.241) plan K9, the element-granular tile transpose; whole-vector extents stay on K7."""
    for R, C, es in [(4095, 4097, 2), (8191, 8193, 1), (333, 777, 4)]:
        d = axe.CopyPlan(layout([(R, C), (C, 1)]), linear_storage(R * C), layout([(R, 1), (C, R)]),
                         linear_storage(R * C), es).describe()
        assert d["kernel"] == "transpose" and d["mode"] == "ragged", (R, C, es, d)
    # extents of whole 16-byte vectors that are not whole tiles: K7 with its ragged last tile row masked
    d = axe.CopyPlan(layout([(8000, 8000), (8000, 1)]), linear_storage(8000 * 8000), layout([(8000, 1), (8000, 8000)]),
                     linear_storage(8000 * 8000), 2).describe()
    assert d["kernel"] == "transpose" and "mode" not in d and d["tile"] == [256, 64], d
    assert d["tiles"] == 32 * 125, d     # ceil(8000 / 256) tile rows x 8000 / 64 tile columns


def test_plan_errors():
    st = linear_storage(16)
    cases = [
        (layout([(16, 1)]), layout([(8, 1)]), st, "AXE_ERR_SIZE_MISMATCH"),
        (layout([(16, 1)]), layout([(4, 1), (4, 1)]), st, "AXE_ERR_NONINJECTIVE"),
        (layout([(16, 1)]), layout([(16, 1)], O={"m": 1}), st, "AXE_ERR_BOUNDS"),
        (layout([(16, 1)]), layout([(16, 1, "lane")]), st, "AXE_ERR_UNSUPPORTED_AXIS"),
        (layout([(16, 1)]), layout([(8, 1), (2, 1, "gpuid")]), st, "AXE_ERR_UNSUPPORTED_AXIS"),
    ]
    for s, d, dst_st, name in cases:
        with pytest.raises(axe.AxeError) as e:
            axe.CopyPlan(s, st, d, dst_st, 4)
        assert e.value.name == name, (d, e.value)
    with pytest.raises(axe.AxeError) as e:
        axe.CopyPlan(layout([(16, 1)]), st, layout([(16, 1)]), st, 3)
    assert e.value.name == "AXE_ERR_ALIGNMENT"
    with pytest.raises(axe.AxeError) as e:
        axe.CopyPlan(layout([(16, 1)]), st, layout([(16, 1)]), storage([("reg", 4, 3), ("reg", 4)]), 4)
    assert e.value.name == "AXE_ERR_INVALID_ARG"


def test_generic_injectivity_matches_oracle():
    """Random destination layouts: the planner accepts exactly when the oracle's copy sees no collision."""
    rng = np.random.default_rng(5)
    agree = 0
    for _ in range(300):
        n = int(rng.integers(2, 9))
        D = [(int(rng.integers(1, 5)), int(rng.integers(1, 12))) for _ in range(rng.integers(1, 4))]
        R = [(int(rng.integers(1, 3)), int(rng.integers(1, 12))) for _ in range(rng.integers(0, 2))]
        dst = layout(D, R)
        ed, er = oracle.sizes(dst)
        cells = 1 + sum((e - 1) * s for e, s, _ in dst["D"] + dst["R"])
        st = linear_storage(cells)
        src = layout([(ed, 1)])
        v = synth.values(ed, 4, 1)
        out = np.zeros(cells * 4, np.uint8)
        try:
            oracle.copy(src, linear_storage(ed), v, dst, st, out, 4)
            ok_oracle = True
        except oracle.OracleError as e:
            assert e.status == "collide"
            ok_oracle = False
        try:
            axe.CopyPlan(src, linear_storage(ed), dst, st, 4)
            ok_axe = True
        except axe.AxeError as e:
            assert e.name == "AXE_ERR_NONINJECTIVE", e
            ok_axe = False
        assert ok_axe == ok_oracle, dst
        agree += 1
    assert agree == 300


def test_copy_plan_create_ex_host_slabs():
    """axe_copy_plan_create_ex bounds the host-pipeline slab count (bench.py's e2e uses 2)."""
    cfg = synth.config2()
    for n in (2, 4, 8):
        p = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, host_slabs=n)
        assert p.describe()["host_chunks"] == n
    import ctypes as C
    h = C.c_void_p()
    s = axe.Layout(cfg["src"]["D"])
    ss, _k = axe.make_storage(cfg["src_st"])
    assert axe._lib.axe_copy_plan_create_ex(s.handle, C.byref(ss), s.handle, C.byref(ss), 2, 0, -1, C.byref(h)) == 1


def test_concurrent_planning_is_thread_safe():
    """include/axe.h promises thread-safe calls: 8 threads plan and describe copies, reductions and
    redistributions at once (shared axis interning, plan caches, error slots); results match a serial run."""
    import threading
    cfgs = [synth.config2(512), synth.config2(512, reverse=True), synth.config3(8, "a"), synth.config3(8, "b"),
            synth.config1()]
    serial = [plan(c).describe()["kernel"] for c in cfgs]
    errors, out = [], {}

    def work(tid):
        try:
            for rep in range(20):
                for i, c in enumerate(cfgs):
                    k = plan(c).describe()["kernel"]
                    out.setdefault((tid, i), set()).add(k)
                r = synth.reduce_scatter(4, 64, 64, "bf16")
                axe.RedistPlan(r["src"], r["src_st"], r["dst"], r["dst_st"], 2, 4, tid % 4, reduce_dtype="bf16")
                L = axe.Layout.parse(f"({tid + 2},8):(8,1) + [(2):(64@lane)] + {rep}@warp")
                assert L.E_D == (tid + 2) * 8
                try:
                    axe.Layout([(4, 0)])
                except axe.AxeError as e:
                    assert "stride" in str(e)
        except Exception as e:  # collected, asserted below
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(t,)) for t in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:3]
    for (tid, i), ks in out.items():
        assert ks == {serial[i]}, (tid, i, ks)


def test_tma_bulk_and_k3_tma_plans():
    """Plan structure of the TMA-family schedules: a run contiguous on both sides (identity, >= 4 KiB) is the
    bulk mode (no tensor map, 16 KiB boxes); 1 KiB rows stay on K1 in AUTO but a forced TMA plan takes them;
    config 3b is the movmatrix atom on bulk boxes (K3-TMA)."""
    ident = dict(es=2, src=layout([(1 << 24, 1)]), src_st=linear_storage(1 << 24), dst=layout([(1 << 24, 1)]),
                 dst_st=linear_storage(1 << 24))
    d = plan(ident).describe()
    assert d["kernel"] == "tma" and d["mode"] == "bulk-load/bulk-store" and d["box_bytes"] == 16384
    rows1k = dict(es=2, src=layout([(4096, 2048), (512, 1)]), src_st=linear_storage(4096 * 2048),
                  dst=layout([(4096, 512), (512, 1)]), dst_st=linear_storage(4096 * 512))
    assert plan(rows1k).describe()["kernel"] == "vector"
    assert plan(rows1k, "tma").describe()["kernel"] == "tma"
    d = plan(synth.config3(64, "b")).describe()
    assert d["mode"] == "bulk-load/movmatrix/bulk-store" and d["box_bytes"] == 8192
    # swizzled storages never take the bulk mode (bytes move verbatim)
    sw = dict(es=2, src=layout([(1 << 16, 1)]), src_st=linear_storage(1 << 16, synth.SW128),
              dst=layout([(1 << 16, 1)]), dst_st=linear_storage(1 << 16))
    assert plan(sw).describe().get("mode") != "bulk-load/bulk-store"


def test_lowered_schedule_plans():
    """AXE_KERNEL_LOWERED (the paper's TMA lowering as the copy schedule) on the host: config 2 both ways,
    fused 64-row boxes; refusals name the reason (no TMA swizzle on either side, both sides swizzled)."""
    f = plan(synth.config2(512), "lowered").describe()
    assert f["mode"] == "tensor-load/bulk-store" and f["atoms"] == 512 and f["boxes"] == 64 and f["box_bytes"] == 8192
    r = plan(synth.config2(512, reverse=True), "lowered").describe()
    assert r["mode"] == "bulk-load/tensor-store" and r["boxes"] == 64
    plain = synth.config2(512, 64, 2, (0, 0, 0))
    with pytest.raises(axe.AxeError) as e:
        plan(plain, "lowered")
    assert e.value.name == "AXE_ERR_UNSUPPORTED" and "TMA swizzle" in str(e.value)
    both = dict(synth.config2(512), src_st=linear_storage(512 * 512, synth.SW128))
    with pytest.raises(axe.AxeError) as e:
        plan(both, "lowered")
    assert "both sides swizzled" in str(e.value)
