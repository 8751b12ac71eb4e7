#!/usr/bin/env python
"""Randomised GPU parity sweep (development tool; the pytest suite holds the fixed cases).

Random layout pairs -- mixed-radix orders with gaps, negative strides, replicas,
swizzles on either side, 1..16-byte elements, sizes up to ~2^20 elements -- run
through every kernel the planner accepts (auto and each forced kernel) and
through K4 reductions, each compared byte for byte with the oracle.  Runs until
the time budget is spent; prints one JSON line per failure and a summary.

  python tools/fuzz_gpu.py [--seconds 300] [--seed 0]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import layout, linear_storage  # noqa: E402
import paper_2601_19092_b200 as axe  # noqa: E402

NT = os.cpu_count() or 4
KERNELS = ["auto", "generic", "vector", "tma", "tile", "register", "shuffle", "transpose", "lowered", "dual"]


def split(rng, N):
    exts = []
    while N > 1:
        for f in (2, 3, 4, 5, 8, 16):
            if N % f == 0 and rng.random() < 0.45:
                exts.append(f)
                N //= f
                break
        else:
            exts.append(N)
            N = 1
    return exts or [1]


def rand_layout(rng, exts, reps):
    n = len(exts)
    order = rng.permutation(n)
    strides, cur = [0] * n, 1
    for i in order:
        strides[i] = cur
        cur *= exts[i] * int(rng.choice([1, 1, 1, 2]))
    O, D = 0, []
    for i in range(n):
        s = strides[i]
        if rng.random() < 0.15:
            O += (exts[i] - 1) * s
            s = -s
        D.append((exts[i], s))
    R = []
    if reps and rng.random() < 0.3:
        e = int(rng.integers(2, 4))
        R.append((e, cur))
        cur *= e
    return layout(D, R, {"m": O} if O else {}), cur


def pad_cells(rng, cells, es):
    """Round the storage up so a swizzle can apply (whole 1 KiB blocks) sometimes."""
    if rng.random() < 0.35:
        blk = 1024 // es if es <= 1024 else 1
        return -(-cells // blk) * blk, synth.SW128 if rng.random() < 0.6 else (synth.SW64 if rng.random() < 0.5 else synth.SW32)
    return cells, (0, 0, 0)


def copy_case(rng):
    es = int(rng.choice([1, 2, 4, 8, 16]))
    N = int(rng.choice([64, 96, 256, 512, 1000, 4096, 6144, 65536, 262144, 1 << 20]))
    N = max(8, N // max(1, es // 4))
    src, sc = rand_layout(rng, split(rng, N), reps=False)
    dst, dc = rand_layout(rng, split(rng, N), reps=True)
    sc, ssw = pad_cells(rng, sc, es)
    dc, dsw = pad_cells(rng, dc, es)
    return dict(es=es, src=src, src_st=linear_storage(sc, ssw), dst=dst, dst_st=linear_storage(dc, dsw))


def tma_case(rng):
    """Re-tilings in the TMA planner's reach: a (padded) row-major matrix <-> tiles of (tr x tc) elements,
    tiles row- or column-ordered, optional SW32/64/128 on the tiled side, either direction."""
    es = int(rng.choice([1, 2, 4, 8]))
    tc = int(rng.choice([8, 16, 32, 64, 128])) // max(1, es // 2)
    tc = max(1, tc)
    tr = int(rng.choice([1, 2, 8, 16, 64]))
    R, C = tr * int(rng.integers(1, 9)), tc * int(rng.integers(1, 9))
    ld = C + (16 // es if es < 16 else 1) * int(rng.integers(0, 3))
    rm = layout([(R, ld), (C, 1)])
    bR, bC = R // tr, C // tc
    if rng.random() < 0.5:
        tl = layout([(bR, tr * C), (tr, tc), (bC, tr * tc), (tc, 1)])
    else:
        tl = layout([(bR, tr * tc), (tr, tc), (bC, bR * tr * tc), (tc, 1)])
    cells = R * C
    sw = (0, 0, 0)
    if rng.random() < 0.6:
        opts = [z for z in (synth.SW32, synth.SW64, synth.SW128) if (16 << z[0]) == tc * es and (cells * es) % 1024 == 0]
        if opts:
            sw = opts[0]
    a = dict(es=es, src=rm, src_st=linear_storage(R * ld), dst=tl, dst_st=linear_storage(cells, sw))
    if rng.random() < 0.5:
        a = dict(es=es, src=tl, src_st=linear_storage(cells, sw), dst=rm, dst_st=linear_storage(R * ld))
    return a


def run_copy(cfg, kernel, seed):
    es = cfg["es"]
    try:
        plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, kernel)
    except axe.AxeError as e:
        if kernel == "auto" and e.name not in ("AXE_ERR_NONINJECTIVE", "AXE_ERR_BOUNDS"):
            return f"plan failed: {e}"
        return "skip"
    ed, _ = oracle.sizes(cfg["src"])
    v = synth.values(ed, es, seed)
    sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, seed + 1)
    src = oracle.scatter_logical(cfg["src"], cfg["src_st"], v, es, sfill, NT)
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, seed + 2)
    exp = dfill.copy()
    oracle.copy(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, es, NT)
    s = torch.from_numpy(src).cuda()
    d = torch.from_numpy(dfill).cuda()
    plan.execute(s, d)
    torch.cuda.synchronize()
    got = d.cpu().numpy()
    if not np.array_equal(got, exp):
        bad = int(np.count_nonzero(got != exp))
        return f"mismatch ({bad} bytes) kernel={plan.describe().get('kernel')}"
    return None


def reduce_case(rng):
    dtype = str(rng.choice(["bf16", "f16", "i32", "i64"]))  # exact dtypes on synth.numbers (bit-exact check)
    es = synth.DTYPE_SIZE[dtype]
    K = int(rng.choice([1, 2, 3, 4, 8, 16]))
    Y = int(rng.choice([64, 96, 256, 1024, 4096, 65536]))
    src, sc = rand_layout(rng, split(rng, Y) + [K], reps=False)
    # the summed dimension is logically outermost: move the K iter (appended last) to the front
    src = layout([src["D"][-1]] + src["D"][:-1], src["R"], src["O"])
    dst, dc = rand_layout(rng, split(rng, Y), reps=True)
    dc, dsw = pad_cells(rng, dc, es)
    return dict(dtype=dtype, src=src, src_st=linear_storage(sc), dst=dst, dst_st=linear_storage(dc, dsw))


def run_reduce(cfg, seed):
    dtype = cfg["dtype"]
    es = synth.DTYPE_SIZE[dtype]
    try:
        plan = axe.ReducePlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], dtype)
    except axe.AxeError as e:
        if e.name in ("AXE_ERR_NONINJECTIVE", "AXE_ERR_BOUNDS"):
            return "skip"
        return f"plan failed: {e}"
    ed, _ = oracle.sizes(cfg["src"])
    v = synth.numbers(ed, dtype, seed, "narrow")  # exact partial sums: compared bit for bit
    sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, seed + 1)
    src = oracle.scatter_logical(cfg["src"], cfg["src_st"], v, es, sfill, NT)
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, seed + 2)
    exp = dfill.copy()
    oracle.reduce(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, dtype, nthreads=NT)
    s = torch.from_numpy(src).cuda()
    d = torch.from_numpy(dfill).cuda()
    plan.execute(s, d)
    torch.cuda.synchronize()
    if not np.array_equal(d.cpu().numpy(), exp):
        return f"reduce mismatch kernel={plan.describe().get('kernel')}"
    return None


def dist_side(rng, N, nranks, reps_ok):
    """A random distributed layout of N logical elements over nranks devices: one shard digit of extent P on
    gpuid at a random logical position (the rest a random mixed radix on m), and, when P < nranks, the
    remaining nranks / P devices as a gpuid replica (contiguous or strided device ids)."""
    Ps = [p for p in (1, 2, 4, 8) if nranks % p == 0 and N % p == 0 and (reps_ok or p == nranks)]
    P = int(rng.choice(Ps))
    Rn = nranks // P
    exts = split(rng, N // P)
    mem, cells = rand_layout(rng, exts, reps=False)
    pos = int(rng.integers(0, len(mem["D"]) + 1))
    contiguous = rng.random() < 0.5
    gs, rs = (Rn, 1) if contiguous else (1, P)
    D = list(mem["D"])
    D.insert(pos, (P, gs, "gpuid"))
    R = [(Rn, rs, "gpuid")] if Rn > 1 else []
    return layout(D, R, mem["O"]), cells


def redist_case(rng):
    nranks = int(rng.choice([2, 4, 8]))
    es = int(rng.choice([1, 2, 4, 8]))
    N = nranks * int(rng.choice([16, 48, 64, 256, 1024, 4096]))
    src, sc = dist_side(rng, N, nranks, True)
    dst, dc = dist_side(rng, N, nranks, True)
    return dict(es=es, nranks=nranks, src=src, src_st=linear_storage(sc), dst=dst, dst_st=linear_storage(dc))


def run_redist(cfg, seed):
    n, es = cfg["nranks"], cfg["es"]
    try:
        plans = [axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, n, r) for r in range(n)]
    except axe.AxeError as e:
        if e.name in ("AXE_ERR_NONINJECTIVE", "AXE_ERR_BOUNDS", "AXE_ERR_UNSUPPORTED"):
            return "skip"
        return f"plan failed: {e}"
    ed, _ = oracle.sizes(cfg["src"])
    v = synth.values(ed, es, seed)
    sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, seed + 1)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], v, es, n, sfill, NT)
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, seed + 2)
    exp = [dfill.copy() for _ in range(n)]
    oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, es, nthreads=NT)
    s_dev = [torch.from_numpy(x).cuda() for x in src]
    for mode in ("emulate", "peers"):
        d_dev = [torch.from_numpy(dfill).cuda() for _ in range(n)]
        if mode == "emulate":
            axe.redist_emulate(plans, s_dev, d_dev)
        else:
            for r in range(n):
                plans[r].execute_peers(s_dev[r], d_dev)
        torch.cuda.synchronize()
        for r in range(n):
            if not np.array_equal(d_dev[r].cpu().numpy(), exp[r]):
                return f"{mode} mismatch on rank {r} ({plans[0].describe().get('pattern')})"
    return None


def perm_layout(rng, exts):
    """A gap-free mixed radix over exts in random digit order (negative strides compensated by the offset):
    a bijection onto [0, prod(exts))."""
    order = rng.permutation(len(exts))
    strides, cur = [0] * len(exts), 1
    for i in order:
        strides[i] = cur
        cur *= exts[i]
    O, D = 0, []
    for i, e in enumerate(exts):
        s_ = strides[i]
        if rng.random() < 0.15:
            O += (e - 1) * s_
            s_ = -s_
        D.append((e, s_))
    return layout(D, [], {"m": O} if O else {})


def run_chain(rng, seed):
    """A random sequence of dependent and independent copies among a pool of large (2^24-element) and small
    (2^12) buffers, launched back to back on one stream without synchronisation (the PDL overlap decisions
    under test: a long copy, short unrelated copies, then a reader of the long copy's output), then compared
    with the same sequence applied by the oracle."""
    es = int(rng.choice([2, 4]))
    sizes = {"big": 1 << 24, "small": 1 << 12}
    pool = {k: [] for k in sizes}
    host, dev, cls = [], [], []
    for k, C in sizes.items():
        for _ in range(int(rng.integers(2, 4))):
            b = len(host)
            host.append(synth.values(C, es, seed + b))
            dev.append(torch.from_numpy(host[-1].copy()).cuda())
            cls.append(k)
            pool[k].append(b)
    torch.cuda.synchronize()
    steps = []
    for _ in range(int(rng.integers(4, 16))):
        k = "big" if rng.random() < 0.4 else "small"
        C = sizes[k]
        i, j = rng.choice(pool[k], 2, replace=False)
        src, dst = perm_layout(rng, split(rng, C)), perm_layout(rng, split(rng, C))
        st = linear_storage(C)
        plan = axe.CopyPlan(src, st, dst, st, es)
        steps.append((int(i), int(j), src, dst, st))
        plan.execute(dev[i], dev[j])
    torch.cuda.synchronize()
    for i, j, src, dst, st in steps:
        out = host[j].copy()
        oracle.copy(src, st, host[i], dst, st, out, es, NT)
        host[j] = out
    for b in range(len(host)):
        if not np.array_equal(dev[b].cpu().numpy(), host[b]):
            return f"chain mismatch in {cls[b]} buffer {b} after {len(steps)} copies"
    return None


def run_tma_region(crng, case_seed):
    """A random 2- or 3-D region of a padded row-major tensor lowered by axe_tma_lower and executed by
    axe_tma_plan_* into the L_S image; expected = the oracle's copy of the hand-written region layout
    into L_S with the atom's swizzle."""
    es = int(crng.choice([1, 2, 4, 8]))
    sw = int(crng.choice([32, 64, 128]))
    inner = sw // es
    if inner < 1:
        return "skip"
    v = 16 // es if es < 16 else 1
    rank = int(crng.choice([2, 3]))
    ES = ([int(crng.integers(1, 4))] if rank == 3 else []) + [8 * int(crng.integers(1, 5)),
                                                            inner * int(crng.integers(1, 4))]
    EG = [e + int(crng.integers(0, 3)) for e in ES[:-1]] + [ES[-1] + v * int(crng.integers(0, 4))]
    ld = EG[-1] + v * int(crng.integers(0, 3))
    pitch = [0] * rank
    pitch[-1], pitch[-2] = 1, ld
    if rank == 3:
        pitch[0] = ld * EG[1]
    begin = [int(crng.integers(0, EG[j] - ES[j] + 1)) for j in range(rank - 1)]
    begin.append(v * int(crng.integers(0, (EG[-1] - ES[-1]) // v + 1)))
    # L_S: the atom grid (outer iters) in a random order, atoms (8, inner) innermost
    Ea = [1] * rank
    Ea[-1], Ea[-2] = inner, 8
    Eo = [e // a for e, a in zip(ES, Ea)]
    order = list(crng.permutation(rank))
    W = 8 * inner
    gs, stride = {}, 1
    for d in reversed(order):
        gs[int(d)] = stride
        stride *= Eo[int(d)]
    D = []
    for j in range(rank):
        D.append((Eo[j], gs[j] * W))
        if Ea[j] > 1:
            D.append((Ea[j], inner if j == rank - 2 else 1))
    LS = layout(D)
    LG = layout([(EG[j], pitch[j]) for j in range(rank)])
    try:
        plan = axe.TmaPlan(LG, EG, LS, ES, es, sw, begin=begin, extent=ES)
    except axe.AxeError:
        return "skip"
    cells = int(np.prod(ES))
    gbytes = (EG[0] * pitch[0] if rank == 3 else EG[0] * ld) * es
    g = synth.sentinel(gbytes, case_seed % 1000)
    fill = synth.sentinel(cells * es, case_seed % 1000 + 1)
    exp = fill.copy()
    region = layout([(ES[j], pitch[j]) for j in range(rank)], O={"m": sum(b * p for b, p in zip(begin, pitch))})
    oracle.copy(region, linear_storage(gbytes // es), g, LS, linear_storage(cells, {32: synth.SW32, 64: synth.SW64,
                                                                                       128: synth.SW128}[sw]), exp, es)
    out = torch.from_numpy(fill).cuda()
    plan.execute(torch.from_numpy(g).cuda(), out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    if not np.array_equal(got, exp):
        return f"{int((got != exp).sum())} bytes differ (ES={ES}, EG={EG}, begin={begin}, es={es}, sw={sw})"
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--trace", action="store_true", help="print every case to stderr before it runs")
    ap.add_argument("--case", type=int, default=None, help="run only this case seed")
    ap.add_argument("--only", default="", help="chain | copy | reduce | redistribute | tma_region (default: all)")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t0 = time.time()
    n = fails = 0
    kinds = {}
    while time.time() - t0 < a.seconds:
        case_seed = int(rng.integers(1 << 31)) if a.case is None else a.case
        crng = np.random.default_rng(case_seed)
        # the in-order schedule: the planner's default, or 1..5 units per CTA forced on every kernel
        chunk = str(crng.choice(["", "", "1", "2", "3", "5"]))
        os.environ["AXE_CHUNK"] = chunk
        u = crng.random()
        if a.only:
            u = {"chain": 0.0, "redistribute": 0.1, "copy": 0.5, "reduce": 0.9, "tma_region": 0.99}[a.only]
        if u < 0.08:
            err = run_chain(crng, case_seed)
            if err == "skip":
                continue
            n += 1
            kinds["chain"] = kinds.get("chain", 0) + 1
            if err:
                fails += 1
                print(json.dumps({"case_seed": case_seed, "kind": "chain", "chunk": chunk, "error": err}), flush=True)
        elif u < 0.15:
            cfg = redist_case(crng)
            err = run_redist(cfg, case_seed)
            if err == "skip":
                continue
            n += 1
            kinds["redistribute"] = kinds.get("redistribute", 0) + 1
            if err:
                fails += 1
                print(json.dumps({"case_seed": case_seed, "kind": "redistribute", "error": err, "cfg": cfg},
                                 default=str), flush=True)
        elif u < 0.7:
            cfg = copy_case(crng) if crng.random() < 0.7 else tma_case(crng)
            for k in KERNELS:
                if a.trace:
                    print(json.dumps({"running": case_seed, "kernel": k}), file=sys.stderr, flush=True)
                err = run_copy(cfg, k, case_seed)
                if err == "skip":
                    continue
                n += 1
                kinds[k] = kinds.get(k, 0) + 1
                if err:
                    fails += 1
                    print(json.dumps({"case_seed": case_seed, "kind": "copy", "kernel": k, "chunk": chunk, "error": err,
                                      "cfg": {**cfg, "es": cfg["es"]}}, default=str), flush=True)
        elif u >= 0.96:
            err = run_tma_region(crng, case_seed)
            if err == "skip":
                continue
            n += 1
            kinds["tma_region"] = kinds.get("tma_region", 0) + 1
            if err:
                fails += 1
                print(json.dumps({"case_seed": case_seed, "kind": "tma_region", "error": err}), flush=True)
        else:
            cfg = reduce_case(crng)
            err = run_reduce(cfg, case_seed)
            if err == "skip":
                continue
            n += 1
            kinds["reduce"] = kinds.get("reduce", 0) + 1
            if err:
                fails += 1
                print(json.dumps({"case_seed": case_seed, "kind": "reduce", "chunk": chunk, "error": err, "cfg": cfg}, default=str),
                      flush=True)
        if a.case is not None:
            break
    print(json.dumps({"summary": {"runs": n, "failures": fails, "per_kernel": kinds, "seconds": time.time() - t0}}))


if __name__ == "__main__":
    main()
