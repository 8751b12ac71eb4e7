#!/usr/bin/env python
"""DRAM ceiling of a copy with one side in short segments: an R x 8192 fp32 matrix (default 256 MiB a side)
moved as column blocks of S bytes -- the source read in S-byte runs 32 KiB apart, the destination
written contiguously ("gather"), or the reverse ("scatter").  A transpose has one side in such runs
(K7's fp32 tile: 256-byte source runs, 512-byte destination runs), so these rows bound what any
transpose schedule can reach on this B200.  Graph-timed dependent steps (tools/step_floor.py's method),
AUTO kernels (and the other of vector / K1-TMA, forced); torch's copy_, a contiguous libaxe copy and the
fp32 / fp64 transposes (K7) of the same bytes are printed beside them.

  python tools/segment_probe.py [MiB per side]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import paper_2601_19092_b200 as axe  # noqa: E402
import synth  # noqa: E402
from step_floor import timed  # noqa: E402

N = 8192  # columns (a 32 KiB row pitch)
ES = 4


def main():
    mib = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    R = (mib << 20) // (N * ES)  # rows
    ne = R * N
    nb = ne * ES
    pairs = max(2, (2 << 30) // (2 * nb))  # >= 2 GiB footprint, > 16x L2
    srcs = [torch.empty(nb, dtype=torch.uint8, device="cuda").random_() for _ in range(pairs)]
    dsts = [torch.empty_like(s) for s in srcs]
    out = {}

    def put(name, us, kernel):
        out[name] = {"us": round(us, 1), "GBps": round(2 * nb / (us * 1e-6) / 1e9), "kernel": kernel}
        print(name, out[name], flush=True)

    def row(name, src, dst, es=ES, alt=True):
        st = synth.linear_storage(nb // es)
        p = axe.CopyPlan(src, st, dst, st, es)
        k = p.describe()["kernel"]
        put(name, timed(lambda i, s: p.execute(srcs[i], dsts[i], s), pairs, 16), k)
        if alt:  # the other planner of the pair, forced: does AUTO pick the faster one?
            other = {"tma": "vector", "vector": "tma"}.get(k)
            try:
                q = axe.CopyPlan(src, st, dst, st, es, other) if other else None
            except axe.AxeError:
                q = None
            if q is not None:
                put(name + "_" + other, timed(lambda i, s: q.execute(srcs[i], dsts[i], s), pairs, 16), other)

    put("torch_copy_", timed(lambda i, s: dsts[i].copy_(srcs[i]), pairs, 16), "torch")
    row("contiguous", synth.layout([(ne, 1)]), synth.layout([(ne, 1)]))
    for seg in (128, 256, 512, 1024, 2048, 4096, 16384):
        c = seg // ES
        strided = synth.layout([(N // c, c), (R, N), (c, 1)])
        packed = synth.layout([(N // c, R * c), (R, c), (c, 1)])
        row(f"gather_{seg}B", strided, packed)
        row(f"scatter_{seg}B", packed, strided)
    row("transpose_f32", synth.layout([(R, N), (N, 1)]), synth.layout([(R, 1), (N, R)]), alt=False)
    h = N // 2  # fp64 R x 4096: the same bytes
    row("transpose_f64", synth.layout([(R, h), (h, 1)]), synth.layout([(R, 1), (h, R)]), es=8, alt=False)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
