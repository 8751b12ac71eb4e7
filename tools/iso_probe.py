#!/usr/bin/env python
"""Config 2's bytes (32 MiB each side) moved by different kernels, each launched a few times on its own
buffers -- run under `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,...` to compare one cold,
serialised launch of each; without ncu it prints graph-timed dependent steps (tools/step_floor.py's method).

  python tools/iso_probe.py [kernels...]   (default: lowered vector tma torch)"""
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


def main():
    names = sys.argv[1:] or ["lowered", "vector", "tma", "torch"]
    c = synth.config2()
    nb = 4096 * 4096 * 2
    pairs = 32
    srcs = [torch.empty(nb, dtype=torch.uint8, device="cuda").random_() for _ in range(pairs)]
    dsts = [torch.empty_like(s) for s in srcs]
    out = {}
    for k in names:
        if k == "torch":
            fn = lambda i, st: dsts[i].copy_(srcs[i])  # noqa: E731
        else:
            p = axe.CopyPlan(c["src"], c["src_st"], c["dst"], c["dst_st"], 2, k)
            fn = lambda i, st, p=p: p.execute(srcs[i], dsts[i], st)  # noqa: E731
        us = timed(fn, pairs, 64)
        out[k] = {"us": us, "GBps": 2 * nb / (us * 1e-6) / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
