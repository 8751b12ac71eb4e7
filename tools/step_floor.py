#!/usr/bin/env python
"""What one dependent copy of a given size costs on this B200, kernel against kernel: back-to-back copies
over rotating buffers (>= 2 GiB footprint, L2 defeated), captured as one CUDA graph of N launches and
timed with CUDA events around one replay.  Rows: torch's copy_ (the driver's peak-measuring kernel), the
libaxe identity copy (K1-TMA bulk) and config 2 (the lowered TMA schedule), each at 32 MiB per side
(the bench step) and larger, so the per-launch ramp and tail show against the bytes moved.

  python tools/step_floor.py [N]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2601_19092_b200 as axe  # noqa: E402
import synth  # noqa: E402


def timed(fn, pairs, n):
    for i in range(3):
        fn(i % pairs, torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for i in range(n):
            fn(i % pairs, torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / n)
    return best * 1e3  # us


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    out = {}
    for mib in (32, 128, 512):
        nb = mib << 20
        pairs = max(2, (2 << 30) // (2 * nb))
        srcs = [torch.empty(nb, dtype=torch.uint8, device="cuda").random_() for _ in range(pairs)]
        dsts = [torch.empty_like(s) for s in srcs]
        row = {}
        row["torch_copy_"] = timed(lambda i, st: dsts[i].copy_(srcs[i]), pairs, n)
        ne = nb // 2
        ident = axe.CopyPlan(synth.layout([(ne, 1)]), synth.linear_storage(ne), synth.layout([(ne, 1)]),
                             synth.linear_storage(ne), 2)
        row["axe_identity"] = timed(lambda i, st: ident.execute(srcs[i], dsts[i], st), pairs, n)
        row["axe_identity_kernel"] = ident.describe()["kernel"]
        side = int((ne) ** 0.5)
        if side * side == ne:
            c = synth.config2(side)
            p = axe.CopyPlan(c["src"], c["src_st"], c["dst"], c["dst_st"], 2)
            row["axe_config2"] = timed(lambda i, st: p.execute(srcs[i], dsts[i], st), pairs, n)
            row["axe_config2_kernel"] = p.describe()["kernel"]
        for k in list(row):
            if isinstance(row[k], float):
                row[k + "_GBps"] = 2 * nb / (row[k] * 1e-6) / 1e9
        out[f"{mib}MiB"] = row
        del srcs, dsts
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
