#!/usr/bin/env python
"""Run one config a few times (for ncu captures): python tools/profile_case.py <config> [kernel] [reps]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import paper_2601_19092_b200 as axe  # noqa: E402
from perf_configs import CONFIGS, REDUCE  # noqa: E402

name = sys.argv[1]
kernel = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = (REDUCE if name in REDUCE else CONFIGS)[name]()
if name in REDUCE:
    plan = axe.ReducePlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["dtype"])
else:
    plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["es"], kernel)
sb, db = plan.sizes()
s = torch.empty(sb, dtype=torch.uint8, device="cuda").random_()
d = torch.empty(db, dtype=torch.uint8, device="cuda")
for _ in range(reps):
    plan.execute(s, d)
torch.cuda.synchronize()
print(plan.describe())
