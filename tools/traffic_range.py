#!/usr/bin/env python
"""Steady-state DRAM traffic of one schedule: N back-to-back copies over rotating buffers (> 4x L2) inside
ONE profiler range, so ncu measures the range as a whole -- dirty lines of earlier copies are evicted
during later ones, as in the bench -- instead of one cold, cache-flushed launch.

  ncu --replay-mode app-range --cache-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      python tools/traffic_range.py [config] [N]
  (bytes per launch = range sum / N; tools/perf_configs.py names the configs)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import paper_2601_19092_b200 as axe  # noqa: E402
from perf_configs import CONFIGS  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "config2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    cfg = CONFIGS[name]()
    plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["es"])
    sb, db = plan.sizes()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    pairs = max(2, min(32, -(-4 * l2 // (sb + db))))
    srcs = [torch.empty(sb, dtype=torch.uint8, device="cuda").random_() for _ in range(pairs)]
    dsts = [torch.empty(db, dtype=torch.uint8, device="cuda") for _ in range(pairs)]
    st = torch.cuda.current_stream()
    for i in range(2 * pairs):  # steady state: L2 full of earlier copies' dirty lines
        plan.execute(srcs[i % pairs], dsts[i % pairs], st)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for i in range(n):
        plan.execute(srcs[i % pairs], dsts[i % pairs], st)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(plan.describe().get("kernel"), "alg_bytes_per_launch", sb + db if name != "config1" else None, "launches", n)


if __name__ == "__main__":
    main()
