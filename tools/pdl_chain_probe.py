"""PDL chain probe (development): K_a writes X (1 GiB), K_b touches disjoint buffers, K_c reads the tail of X.
Counts stale reads of X in K_c.  Variant 'wait': K_c also writes K_b's destination, so it must wait for K_b;
the question is whether K_b's completion implies K_a's (transitive completion)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2601_19092_b200 as axe  # noqa: E402
from synth import layout, linear_storage  # noqa: E402

torch.cuda.set_device(0)
N = 1 << 29
n = 1 << 12
big = axe.CopyPlan(layout([(N, 1)]), linear_storage(N), layout([(N, 1)]), linear_storage(N), 2)
small = axe.CopyPlan(layout([(n, 1)]), linear_storage(n), layout([(n, 1)]), linear_storage(n), 2)
readc = axe.CopyPlan(layout([(n, 1)], O={"m": N - n}), linear_storage(N), layout([(n, 1)]), linear_storage(n), 2)
S = torch.full((N,), 7, dtype=torch.int16, device="cuda")
X = torch.zeros(N, dtype=torch.int16, device="cuda")
a = torch.zeros(n, dtype=torch.int16, device="cuda")
b = torch.zeros_like(a)
Y = torch.zeros(n, dtype=torch.int16, device="cuda")
st = torch.cuda.current_stream()
for variant in ("nowait", "wait"):
    bad = 0
    for it in range(40):
        X.zero_()
        Y.fill_(-1)
        torch.cuda.synchronize()
        big.execute(S, X, st)
        small.execute(a, b, st)
        readc.execute(X, b if variant == "wait" else Y, st)
        torch.cuda.synchronize()
        out = b if variant == "wait" else Y
        if not bool((out == 7).all()):
            bad += 1
    print({"variant": variant, "iterations": 40, "stale_reads": bad}, flush=True)
