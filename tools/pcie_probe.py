#!/usr/bin/env python
"""PCIe ceiling on the box: pinned H2D, D2H and both directions at once (torch copies, CUDA events)."""
import json

import torch


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for mib in (4, 32, 128):
    n = mib << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
    d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    bi = timed(both)
    print(json.dumps({"MiB": mib, "h2d_GBps": n / h2d / 1e6, "d2h_GBps": n / d2h / 1e6,
                      "bidir_GBps_total": 2 * n / bi / 1e6}), flush=True)
