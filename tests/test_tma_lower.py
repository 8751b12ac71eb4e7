"""The paper's TMA lowering on the layout algebra (§3.4 "TMA asynchronous copy",
P:519-536): slice -> tiler of the swizzle atom -> CuTensorMap
from L_G.  Checked against SPEC's worked plan, against the oracle's
evaluation of both layouts for every element of random regions (the plan
interpreter of S:487-491: every element lands where L_S / L_G say), and against
the tensor map the K1-TMA planner builds directly from joint digits (no GPU)."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage

import paper_2601_19092_b200 as axe


def flat(S, u):
    x = 0
    for s, v in zip(S, u):
        x = x * s + v
    return x


def m_of(spec, x):
    (c,) = oracle.eval(spec, x)
    return c.get("m", 0)


def interpret(r, LG, EG, LS, ES, es, begin):
    """Every element (u) of the region: shared offset from the tiler + row-major atom, global byte offset from
    the tensor map; both must equal the layouts' own values (oracle)."""
    rank = len(ES)
    inner = r["swizzle_bytes"] // es
    Ea = [1] * rank
    Ea[-1], Ea[-2] = inner, 8
    Eo = [e // a for e, a in zip(ES, Ea)]
    W = 8 * inner
    T = layout(r["tiler"].iters(0))
    # tensor-map dims of each logical dimension, innermost first
    per = {j: [(d, s) for d, s, lj in zip(r["dims"], r["strides"], r["logical_dim"]) if lj == j] for j in range(rank)}
    for j in range(rank):
        box = np.prod([b for b, lj in zip(r["box"], r["logical_dim"]) if lj == j] or [1])
        assert box == Ea[j]
    seen = set()
    for u in itertools.product(*[range(e) for e in ES]):
        t = [ui // a for ui, a in zip(u, Ea)]
        w = [ui % a for ui, a in zip(u, Ea)]
        sm = m_of(T, flat(Eo, t)) * W + w[-2] * inner + w[-1]
        assert sm == m_of(LS, flat(ES, u)), u
        seen.add(sm)
        g = r["base_bytes"]
        for j in range(rank):
            rem = u[j]
            for d, s in per[j]:
                g += (rem % d) * s
                rem //= d
            assert rem == 0
        gu = [b + ui for b, ui in zip(begin or [0] * rank, u)]
        assert g == m_of(LG, flat(EG, gu)) * es, u
    assert len(seen) == int(np.prod(ES))  # atoms are disjoint in shared memory


def test_spec_plan_example():
    """L_S row-major (16,64), bf16, 128 B swizzle -> 2 atoms of (8,64) at shared offsets {0, 512},
    global box origins (0,0) and (8,0)."""
    LG = layout([(16, 64), (64, 1)])
    LS = layout([(16, 64), (64, 1)])
    r = axe.tma_lower(LG, [16, 64], LS, [16, 64], 2, 128)
    assert r["atoms"] == 2 and r["tiler"].iters(0) == [(2, 1, "m")]       # (2):(1) x span 512 = {0, 512}
    assert r["box"][:2] == [64, 8] and r["strides"][:2] == [2, 128] and r["base_bytes"] == 0
    assert r["dims"][2] == 2 and r["strides"][2] == 8 * 128                  # atom t starts at row 8 t
    interpret(r, LG, [16, 64], LS, [16, 64], 2, None)


def test_spec_column_major_fails():
    """the row-major atom is not a tile of a column-major shared block."""
    with pytest.raises(axe.AxeError) as e:
        axe.tma_lower(layout([(16, 64), (64, 1)]), [16, 64], layout([(16, 1), (64, 16)]), [16, 64], 2, 128)
    assert e.value.name == "AXE_ERR_UNSUPPORTED"


def test_config2_tile_region():
    """Config 2: the (i, j) = (2, 3) 64x64 tile of a 4096^2 bf16 row-major tensor into a row-major 64x64 SW128
    shared tile: slice offset (128 * 4096 + 192) * 2 B, atoms (8, 64) stacked 8 deep along rows."""
    LG = layout([(4096, 4096), (4096, 1)])
    LS = layout([(64, 64), (64, 1)])
    r = axe.tma_lower(LG, [4096, 4096], LS, [64, 64], 2, 128, begin=[128, 192], extent=[64, 64])
    assert r["dims"] == [64, 8, 8] and r["strides"] == [2, 8192, 65536] and r["box"] == [64, 8, 1]
    assert r["base_bytes"] == (128 * 4096 + 192) * 2 and r["atoms"] == 8 and r["fused_rows"] == 64
    assert r["tiler"].iters(0) == [(8, 1, "m")]


def atom_tiled_smem(rng, ES, inner):
    """A random shared layout that is a tiling of the (8, inner) atom: the atom grid in a random order."""
    Eo = [ES[0] // 8, ES[1] // inner]
    grid = [(Eo[0], 0), (Eo[1], 1)]
    if rng.integers(0, 2):
        grid.reverse()
    stride, gs = 1, {}
    for e, d in reversed(grid):
        gs[d] = stride
        stride *= e
    W = 8 * inner
    return layout([(Eo[0], gs[0] * W), (8, inner), (Eo[1], gs[1] * W), (inner, 1)])


def test_random_regions_interpreted():
    rng = np.random.default_rng(7)
    n = 0
    for _ in range(60):
        es = int(rng.choice([1, 2, 4]))
        sw = int(rng.choice([32, 64, 128]))
        inner = sw // es
        ES = [8 * int(rng.integers(1, 5)), inner * int(rng.integers(1, 4))]
        rows, cols = ES[0] * int(rng.integers(1, 4)), ES[1] * int(rng.integers(1, 3)) + 16 // es * int(rng.integers(0, 3))
        ld = cols + 16 // es * int(rng.integers(0, 3))            # padded rows (16-byte multiples)
        LG = layout([(rows, ld), (cols, 1)])
        EG = [rows, cols]
        begin = [int(rng.integers(0, rows - ES[0] + 1)), int(rng.integers(0, (cols - ES[1]) // (16 // es) + 1)) * (16 // es)]
        LS = atom_tiled_smem(rng, ES, inner)
        try:
            r = axe.tma_lower(LG, EG, LS, ES, es, sw, begin=begin, extent=ES)
        except axe.AxeError as e:
            assert e.name in ("AXE_ERR_UNSUPPORTED", "AXE_ERR_ALIGNMENT"), e
            continue
        interpret(r, LG, EG, LS, ES, es, begin)
        n += 1
    assert n >= 30


@pytest.mark.parametrize("n,tile,es,swz", [(4096, 64, 2, synth.SW128), (1024, 64, 2, synth.SW128),
                                           (512, 128, 1, synth.SW128), (1024, 32, 2, synth.SW64),
                                           (512, 32, 4, synth.SW128), (2048, 64, 1, synth.SW64)])
def test_agrees_with_the_k1_tma_planner(n, tile, es, swz):
    """The K1-TMA planner derives its box from joint digits; for config-2 style re-tilings it must agree
    with the paper's lowering of one tile: box row bytes, rows per box (fused atoms), row stride."""
    cfg = synth.config2(n, tile, es, swz)
    d = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, "tma").describe()
    if d["kernel"] != "tma" or d["mode"] != "tensor-load/bulk-store":
        pytest.skip(f"planner chose {d['kernel']}")
    tm = d["tensor_map"]
    sw_bytes = 16 << swz[0]
    LG = layout([(n, n), (n, 1)])
    LS = layout([(tile, tile), (tile, 1)])
    r = axe.tma_lower(LG, [n, n], LS, [tile, tile], es, sw_bytes, begin=[0, 0], extent=[tile, tile])
    assert r["box"][0] * es == tm["box"][0]              # bytes of one box row
    assert r["fused_rows"] == tm["box"][1]               # rows per box
    assert r["strides"][1] == tm["strides"][1]           # global row stride (bytes)


def test_device_plan_from_the_lowering():
    """axe_tma_plan_create consumes the lowering (descriptor + T) without a GPU: atom count and image size
    of L_S; a descriptor that is not one atom per box is rejected."""
    p = axe.TmaPlan(layout([(4096, 4096), (4096, 1)]), [4096, 4096], layout([(64, 64), (64, 1)]), [64, 64], 2, 128,
                    begin=[128, 192], extent=[64, 64])
    assert p.sizes() == (8, 64 * 64 * 2)
    rng = np.random.default_rng(3)
    LS = atom_tiled_smem(rng, [32, 128], 32)              # fp32, 128-byte atoms (8 x 32), 4 x 4 grid
    q = axe.TmaPlan(layout([(64, 256), (256, 1)]), [64, 256], LS, [32, 128], 4, 128, begin=[8, 64], extent=[32, 128])
    assert q.sizes() == (16, 32 * 128 * 4)
    d = q.lowering["_desc"]
    d.box[1] = 4                                          # half an atom per box
    h = axe.C.c_void_p()
    assert axe._lib.axe_tma_plan_create(axe.C.byref(d), q.lowering["tiler"].handle, axe.C.byref(h)) == 1


def test_lowered_copy_plans_have_box_programs():
    """The lowered schedule's box table (tensor-map coordinates + image offset per fused atom box) is
    re-expressed as a mixed-radix program the kernel evaluates (tma_region.cpp fit_program, verified
    against every box): config 2 both ways, at 16384^2, with other element sizes / swizzles, and with the
    tiles stored column-of-tiles first -- none needs the global-memory table."""
    import paper_2601_19092_b200 as axe
    cfgs = [synth.config2(), synth.config2(reverse=True), synth.config2(16384), synth.config2(512, 32, 4),
            synth.config2(512, 64, 1, synth.SW64), synth.config2(256, 16, 4, synth.SW64, True)]
    R, Cn, t = 256, 512, 64
    cfgs.append(dict(src=layout([(R // t, t * Cn), (t, Cn), (Cn // t, t), (t, 1)]), src_st=linear_storage(R * Cn),
                     dst=layout([(R // t, t * t), (t, t), (Cn // t, (R // t) * t * t), (t, 1)]),
                     dst_st=linear_storage(R * Cn, synth.SW128), es=2))
    for c in cfgs:
        d = axe.CopyPlan(c["src"], c["src_st"], c["dst"], c["dst_st"], c["es"], "lowered").describe()
        assert d["kernel"] == "lowered", d
        assert d["box_program_digits"] >= 1, d
