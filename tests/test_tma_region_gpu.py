"""The paper's TMA lowering executed on the B200 (§3.4 "TMA asynchronous copy"; SURVEY
§8(f) f1): axe_tma_lower's CuTensorMap + tiler T drive one TMA tensor load and one bulk store per
swizzle atom (axe_tma_plan_*), producing an HBM image of the shared-memory tensor L_S.

Parity: the oracle's copy of the same region -- the region of the global tensor written by hand as a
layout (rows of pitch ld starting at begin), into L_S on a storage with the atom's swizzle (CUTLASS
Swizzle<B,4,3>, the hardware's 32/64/128-byte modes, S:O6) -- byte for byte, sentinel included."""
import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
SW = {32: synth.SW32, 64: synth.SW64, 128: synth.SW128}


@pytest.fixture(scope="module")
def axe():
    assert torch.cuda.is_available()
    import paper_2601_19092_b200 as m
    return m


def atom_tiled_smem(rng, ES, inner, order):
    """L_S = a tiling of the (8, inner) atom with the atom grid in row- or column-major order."""
    Eo = [ES[0] // 8, ES[1] // inner]
    grid = [(Eo[0], 0), (Eo[1], 1)]
    if order:
        grid.reverse()
    stride, gs = 1, {}
    for e, d in reversed(grid):
        gs[d] = stride
        stride *= e
    W = 8 * inner
    return layout([(Eo[0], gs[0] * W), (8, inner), (Eo[1], gs[1] * W), (inner, 1)])


def run_case(axe, rows, cols, ld, begin, ES, LS, es, sw, seed):
    LG = layout([(rows, ld), (cols, 1)])
    plan = axe.TmaPlan(LG, [rows, cols], LS, ES, es, sw, begin=begin, extent=ES)
    atoms, img = plan.sizes()
    assert atoms == ES[0] * ES[1] * es // (8 * sw) and img == ES[0] * ES[1] * es
    gbytes = rows * ld * es
    g = synth.sentinel(gbytes, seed)
    fill = synth.sentinel(img, seed + 1)
    exp = fill.copy()
    region = layout([(ES[0], ld), (ES[1], 1)], O={"m": begin[0] * ld + begin[1]})
    oracle.copy(region, linear_storage(rows * ld), g, LS, linear_storage(img // es, SW[sw]), exp, es)
    gd = torch.from_numpy(g).cuda()
    out = torch.from_numpy(fill).cuda()
    n0 = axe.kernel_launch_count()
    plan.execute(gd, out)
    plan.execute(gd, out)   # cached table + tensor map
    torch.cuda.synchronize()
    assert axe.kernel_launch_count() - n0 == 2
    got = out.cpu().numpy()
    if not np.array_equal(got, exp):
        bad = np.nonzero(got != exp)[0]
        raise AssertionError(f"{len(bad)} bytes differ, first at {bad[:8]}")
    # the reverse (TMA stores): the image back into a sentinel-filled global tensor; expected = the
    # oracle's copy of L_S (swizzled) into the hand-written region layout
    g2 = synth.sentinel(gbytes, seed + 2)
    exp2 = g2.copy()
    oracle.copy(LS, linear_storage(img // es, SW[sw]), exp, region, linear_storage(rows * ld), exp2, es)
    gd2 = torch.from_numpy(g2).cuda()
    plan.execute_store(gd2, out)
    torch.cuda.synchronize()
    assert np.array_equal(gd2.cpu().numpy(), exp2), "store direction"
    return plan


def test_config2_tile(axe):
    """The (2, 3) 64x64 tile of config 2's 4096^2 bf16 tensor into a row-major SW128 shared tile: 8 atoms."""
    p = run_case(axe, 4096, 4096, 4096, [128, 192], [64, 64], layout([(64, 64), (64, 1)]), 2, 128, 3)
    assert p.lowering["atoms"] == 8


@pytest.mark.parametrize("es,sw", [(1, 32), (1, 128), (2, 64), (2, 128), (4, 32), (4, 128), (8, 64), (8, 128)])
def test_random_regions(axe, es, sw):
    rng = np.random.default_rng(es * 1000 + sw)
    inner = sw // es
    n = 0
    for trial in range(12):
        ES = [8 * int(rng.integers(1, 6)), inner * int(rng.integers(1, 4))]
        v = 16 // es
        rows = ES[0] * int(rng.integers(1, 4)) + int(rng.integers(0, 9))
        cols = ES[1] + v * int(rng.integers(0, 5))
        ld = cols + v * int(rng.integers(0, 3))
        begin = [int(rng.integers(0, rows - ES[0] + 1)), v * int(rng.integers(0, (cols - ES[1]) // v + 1))]
        LS = atom_tiled_smem(rng, ES, inner, trial % 2)
        run_case(axe, rows, cols, ld, begin, ES, LS, es, sw, trial)
        n += 1
    assert n == 12


def test_many_atoms_per_cta(axe):
    """A large region (4096 atoms over <= 2368 CTAs, 8-slot rings wrap) -- every atom lands once."""
    ES = [512, 256]
    run_case(axe, 1024, 512, 512, [256, 128], ES, atom_tiled_smem(None, ES, 64, 1), 2, 128, 5)


@pytest.mark.parametrize("order", [0, 1])
def test_rank3_region_five_tensor_dims(axe, order):
    """A 3-D region (2 x 16 x 64 of a padded 4 x 48 x 96 bf16 tensor, 64-byte swizzle): the lowering
    needs all 5 CuTensorMap dims (column atoms split off the box); atom grid (b, row-tile, col-tile)
    in row-major or reversed order."""
    B, rows, cols, ld, es, sw = 4, 48, 96, 104, 2, 64
    inner, ES = sw // es, [2, 16, 64]
    W = 8 * inner
    strides = [4 * W, 2 * W, W] if order == 0 else [W, 2 * W, 4 * W]
    LS = layout([(2, strides[0]), (2, strides[1]), (8, inner), (2, strides[2]), (inner, 1)])
    LG = layout([(B, rows * ld), (rows, ld), (cols, 1)])
    begin = [1, 8, 16]
    plan = axe.TmaPlan(LG, [B, rows, cols], LS, ES, es, sw, begin=begin, extent=ES)
    assert plan.lowering["rank"] == 5 and plan.sizes() == (8, 2 * 16 * 64 * es)
    g = synth.sentinel(B * rows * ld * es, 21)
    fill = synth.sentinel(2 * 16 * 64 * es, 22)
    exp = fill.copy()
    region = layout([(2, rows * ld), (16, ld), (64, 1)], O={"m": begin[0] * rows * ld + begin[1] * ld + begin[2]})
    oracle.copy(region, linear_storage(B * rows * ld), g, LS, linear_storage(2 * 16 * 64, SW[sw]), exp, es)
    out = torch.from_numpy(fill).cuda()
    plan.execute(torch.from_numpy(g).cuda(), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), exp)


def test_misaligned_region_rejected(axe):
    plan = axe.TmaPlan(layout([(64, 64), (64, 1)]), [64, 64], layout([(8, 64), (64, 1)]), [8, 64], 2, 128,
                       begin=[0, 0], extent=[8, 64])
    g = torch.zeros(64 * 64 + 8, dtype=torch.int16, device="cuda")
    img = torch.zeros(8 * 64, dtype=torch.int16, device="cuda")
    with pytest.raises(axe.AxeError) as e:
        plan.execute(g[1:], img)
    assert e.value.name == "AXE_ERR_ALIGNMENT"


@pytest.mark.parametrize("es,sw", [(1, 128), (2, 64), (4, 128), (8, 32)])
def test_random_regions_table_form(axe, es, sw, monkeypatch):
    """The kernel's fallback form (box coordinates read from the atom table in global memory instead of
    the fitted mixed-radix program) on the same random regions."""
    monkeypatch.setenv("AXE_TMA_REGION_TABLE", "1")
    rng = np.random.default_rng(es * 7 + sw)
    inner = sw // es
    for trial in range(6):
        ES = [8 * int(rng.integers(1, 6)), inner * int(rng.integers(1, 4))]
        v = 16 // es
        rows = ES[0] * int(rng.integers(1, 4)) + int(rng.integers(0, 9))
        cols = ES[1] + v * int(rng.integers(0, 5))
        ld = cols + v * int(rng.integers(0, 3))
        begin = [int(rng.integers(0, rows - ES[0] + 1)), v * int(rng.integers(0, (cols - ES[1]) // v + 1))]
        run_case(axe, rows, cols, ld, begin, ES, atom_tiled_smem(rng, ES, inner, trial % 2), es, sw, 100 + trial)


def test_copy_then_tma_plan_then_copy_without_sync(axe):
    """a copy writes G, the TMA plan turns G into the image, a small copy reads the image --
    back to back on one stream with no synchronize.  The TMA plan's kernel lets its dependents launch at
    entry, so the copy after it must still wait for it (the public execute resets the PDL window)."""
    n = 512
    ES = [64, 64]
    LS = layout([(64, 64), (64, 1)])
    rm = layout([(n, n), (n, 1)])
    plan = axe.TmaPlan(rm, [n, n], LS, ES, 2, 128, begin=[64, 128], extent=ES)
    ident = axe.CopyPlan(rm, linear_storage(n * n), rm, linear_storage(n * n), 2)
    sub = layout([(64 * 64, 1)])
    read = axe.CopyPlan(sub, linear_storage(64 * 64), sub, linear_storage(64 * 64), 2)
    fwd = synth.sentinel(n * n * 2, 41)
    exp_img = synth.sentinel(64 * 64 * 2, 42)
    region = layout([(64, n), (64, 1)], O={"m": 64 * n + 128})
    oracle.copy(region, linear_storage(n * n), fwd, LS, linear_storage(64 * 64, SW[128]), exp_img, 2)
    src = torch.from_numpy(fwd).cuda()
    st = torch.cuda.current_stream()
    for _ in range(20):
        g = torch.zeros(n * n, dtype=torch.int16, device="cuda")
        img = torch.zeros(64 * 64, dtype=torch.int16, device="cuda")
        out = torch.zeros(64 * 64, dtype=torch.int16, device="cuda")
        torch.cuda.synchronize()
        ident.execute(src, g, st)
        plan.execute(g, img, st)
        read.execute(img, out, st)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint8), exp_img)
