#!/usr/bin/env python
"""Small instances of every kernel path (K0, K1 decode/tiled, K1-TMA both modes, K2, K3) for
compute-sanitizer runs: python tools/sanitize_cases.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2601_19092_b200 as axe  # noqa: E402
from synth import layout, linear_storage  # noqa: E402

cases = [
    (synth.config1(), "generic"), (synth.config1(), "auto"),
    (synth.config2(256), "tma"), (synth.config2(256, reverse=True), "tma"), (synth.config2(256), "vector"),
    (synth.config3(4, "a"), "tile"), (synth.config3(4, "a"), "vector"), (synth.config3(4, "b"), "register"),
    (dict(es=2, src=layout([(512, 256), (256, 1)]), src_st=linear_storage(512 * 256),
          dst=layout([(512, 1), (256, 512)]), dst_st=linear_storage(512 * 256)), "tile"),
]
for cfg, k in cases:
    p = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["es"], k)
    sb, db = p.sizes()
    s = torch.empty(sb, dtype=torch.uint8, device="cuda").random_()
    d = torch.zeros(db, dtype=torch.uint8, device="cuda")
    p.execute(s, d)
    p.execute(s, d)
    torch.cuda.synchronize()
    print(k, p.describe()["kernel"], "ok", flush=True)
