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
KERNELS = ["auto", "generic", "vector", "tma", "tile", "register", "tma_tile"]


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
    v = synth.numbers(ed, dtype, seed)
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t0 = time.time()
    n = fails = 0
    kinds = {}
    while time.time() - t0 < a.seconds:
        case_seed = int(rng.integers(1 << 31))
        crng = np.random.default_rng(case_seed)
        if crng.random() < 0.7:
            cfg = copy_case(crng)
            for k in KERNELS:
                err = run_copy(cfg, k, case_seed)
                if err == "skip":
                    continue
                n += 1
                kinds[k] = kinds.get(k, 0) + 1
                if err:
                    fails += 1
                    print(json.dumps({"case_seed": case_seed, "kind": "copy", "kernel": k, "error": err,
                                      "cfg": {**cfg, "es": cfg["es"]}}, default=str), flush=True)
        else:
            cfg = reduce_case(crng)
            err = run_reduce(cfg, case_seed)
            if err == "skip":
                continue
            n += 1
            kinds["reduce"] = kinds.get("reduce", 0) + 1
            if err:
                fails += 1
                print(json.dumps({"case_seed": case_seed, "kind": "reduce", "error": err, "cfg": cfg}, default=str),
                      flush=True)
    print(json.dumps({"summary": {"runs": n, "failures": fails, "per_kernel": kinds, "seconds": time.time() - t0}}))


if __name__ == "__main__":
    main()
