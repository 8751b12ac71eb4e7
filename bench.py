#!/usr/bin/env python
"""bench.py -- layout-copy throughput of libaxe on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): a 4096x4096 bf16
tensor, row-major -> 64x64 tiles with the 128-byte swizzle.  One step = one
axe_copy_plan_execute (plan built outside the timed region) over one tensor.
Inputs are resident in HBM; L2 is defeated by rotating over buffer pairs whose
total footprint is > 4x the L2 size.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl axe|reference]

N > 1 (under torchrun): every rank converts its own tensors (replicas only,
weak scaling; the copy has no exchange step), timing is the max over ranks.
--impl reference times the CPU oracle (oracle/) -- the only other place this
file executes oracle code besides the cpu_baseline leg.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "layout-copy GB/s (% of HBM peak) at 1 B200"
WORKLOAD = "config2: 4096x4096 bf16 row-major -> (64,64,64,64):(262144,64,4096,1) tiles + SW128"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel in the steady state, from the committed ncu range capture
    (tools/traffic_range.py: 32 back-to-back launches in one ncu app-range, read + write bytes / 32)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get("config2", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is under load."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_sample_seconds(budget_s: float, nthreads: int):
    """Time the oracle (as it stands) on 64-row bands of the config-2 conversion until the budget is spent.
    Returns (GB/s, bands, seconds)."""
    import oracle
    cfg = synth.config2()
    n, es = 4096, 2
    src = synth.values(n * n, es, cfg["seed"])
    dst = np.zeros(n * n * es, np.uint8)
    band_bytes = 64 * n * es * 2  # read + write per band
    done, t0 = 0, time.perf_counter()
    while True:
        b = done % 64
        s = {"D": [(64, n, "m"), (n, 1, "m")], "R": [], "O": {"m": b * 64 * n}}
        d = {"D": [(64, 64, "m"), (64, 4096, "m"), (64, 1, "m")], "R": [], "O": {"m": b * 64 * n}}
        oracle.copy(s, cfg["src_st"], src, d, cfg["dst_st"], dst, es, nthreads)
        done += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return done * band_bytes / el / 1e9, done, el


def run_reference(args):
    ws, rank, _ = dist_init(args)
    if rank != 0:
        return
    import oracle
    nthreads = os.cpu_count() or 1
    cfg = synth.config2()
    n, es = 4096, 2
    src = synth.values(n * n, es, cfg["seed"])
    dst = np.zeros(n * n * es, np.uint8)

    def step(i):  # one bounded sample: one 64-row band (1/64 of the workload)
        b = i % 64
        s = {"D": [(64, n, "m"), (n, 1, "m")], "R": [], "O": {"m": b * 64 * n}}
        d = {"D": [(64, 64, "m"), (64, 4096, "m"), (64, 1, "m")], "R": [], "O": {"m": b * 64 * n}}
        oracle.copy(s, cfg["src_st"], src, d, cfg["dst_st"], dst, es, nthreads)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    el = time.perf_counter() - t0
    band_bytes = 64 * n * es * 2
    v = args.steps * band_bytes / el / 1e9
    sample = "64-row band (1/64) of the 4096^2 bf16 config-2 conversion per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": sample},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": nthreads, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def measure_reshard(axe, torch, dist, ws, rank, local, stream, iters=20, warm=3):
    """axe_redistribute over NCCL on all ranks (BASELINE configs 4 and 5).  Bus GB/s = per-GPU NVLink
    ingress bytes / time (max over ranks), i.e. NCCL's busbw for all-gather / all-to-all."""
    comm = axe.Comm.from_process_group(local)
    res = {}
    try:
        ver = ".".join(str(x) for x in torch.cuda.nccl.version())
    except Exception:
        ver = None
    # the communicator the reshard rows ran on (so a scaling run records that every rank joined)
    res["nccl"] = {"version": ver, "nranks": comm.nranks, "rank0_device": torch.cuda.get_device_name(local),
                   "NCCL_DEBUG": os.environ.get("NCCL_DEBUG")}

    def timed(fn):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # config 4: 16384^2 bf16, shard(dim0) -> replicate over P = ws
    c4 = synth.config4(ws)
    p4 = axe.RedistPlan(c4["src"], c4["src_st"], c4["dst"], c4["dst_st"], 2, ws, rank)
    src = torch.randint(-2**15, 2**15 - 1, (synth.storage_cells(c4["src_st"]),), dtype=torch.int16, device="cuda")
    dst = torch.empty(synth.storage_cells(c4["dst_st"]), dtype=torch.int16, device="cuda")
    ms = timed(lambda: p4.execute(comm, src, dst, stream))
    ingress = (ws - 1) * src.numel() * 2
    ref = torch.empty_like(dst)
    ms_ref = timed(lambda: dist.all_gather_into_tensor(ref.view(torch.bfloat16), src.view(torch.bfloat16)))
    res["config4"] = {"P": ws, "pattern": p4.describe()["pattern"], "ms": ms, "ingress_bytes_per_gpu": ingress,
                      "bus_GBps": ingress / (ms * 1e-3) / 1e9, "frac_of_900": ingress / (ms * 1e-3) / 1e9 / 900,
                      "frac_of_measured_770": ingress / (ms * 1e-3) / 1e9 / 770,
                      "torch_all_gather_bus_GBps": ingress / (ms_ref * 1e-3) / 1e9}
    del src, dst, ref
    if ws == 8:
        c5 = synth.config5()
        p5 = axe.RedistPlan(c5["src"], c5["src_st"], c5["dst"], c5["dst_st"], 2, 8, rank)
        src = torch.randint(-2**15, 2**15 - 1, (synth.storage_cells(c5["src_st"]),), dtype=torch.int16, device="cuda")
        dst = torch.empty(synth.storage_cells(c5["dst_st"]), dtype=torch.int16, device="cuda")
        ms = timed(lambda: p5.execute(comm, src, dst, stream))
        ingress = max(p5.counts(q)[1] for q in range(8) if q != rank) * 2
        res["config5"] = {"mesh": "2x4", "pattern": p5.describe()["pattern"], "ms": ms,
                          "ingress_bytes_per_gpu": ingress, "bus_GBps": ingress / (ms * 1e-3) / 1e9,
                          "frac_of_900": ingress / (ms * 1e-3) / 1e9 / 900}
        del src, dst
    # §8(f) f3: reduce-scatter of (ws, 16384, 8192) bf16 partials (P:399-403 at scale); NCCL busbw
    # convention: (P-1)/P * partial bytes per GPU
    rs = synth.reduce_scatter(ws, 16384, 8192, "bf16")
    prs = axe.RedistPlan(rs["src"], rs["src_st"], rs["dst"], rs["dst_st"], 2, ws, rank, reduce_dtype="bf16")
    src = torch.empty(synth.storage_cells(rs["src_st"]), dtype=torch.bfloat16, device="cuda").normal_()
    dst = torch.empty(synth.storage_cells(rs["dst_st"]), dtype=torch.bfloat16, device="cuda")
    ms = timed(lambda: prs.execute(comm, src, dst, stream))
    ref = torch.empty_like(dst)
    ms_ref = timed(lambda: dist.reduce_scatter_tensor(ref, src))
    bus = (ws - 1) / ws * src.numel() * 2
    res["reduce_scatter"] = {"P": ws, "ms": ms, "bus_bytes_per_gpu": bus, "bus_GBps": bus / (ms * 1e-3) / 1e9,
                             "torch_reduce_scatter_bus_GBps": bus / (ms_ref * 1e-3) / 1e9}
    del src, dst, ref
    torch.cuda.synchronize()
    dist.barrier()
    del comm
    # one-sided form: copy kernels write straight into the peers' dst buffers (torch symmetric memory)
    res["one_sided"] = measure_reshard_p2p(axe, torch, dist, ws, rank, local, stream, timed)
    return res


def measure_reshard_p2p(axe, torch, dist, ws, rank, local, stream, timed):
    ok = torch.tensor([1], device="cuda")
    try:
        import torch.distributed._symmetric_memory as symm_mem  # noqa: F401
    except Exception:
        ok.zero_()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)      # every rank takes the same branch
    if not int(ok.item()):
        return {"skipped": "torch symmetric memory unavailable"}
    import torch.distributed._symmetric_memory as symm_mem
    out = {}
    cases = [("config4", synth.config4(ws))] + ([("config5", synth.config5())] if ws == 8 else [])
    for name, cfg in cases:
        plan = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, ws, rank)
        buf = symm_mem.empty(synth.storage_cells(cfg["dst_st"]), dtype=torch.bfloat16, device=f"cuda:{local}")
        hdl = symm_mem.rendezvous(buf, dist.group.WORLD)
        peers = [int(p) for p in hdl.buffer_ptrs]
        src = torch.empty(synth.storage_cells(cfg["src_st"]), dtype=torch.bfloat16, device="cuda").normal_()

        def fn():
            hdl.barrier(channel=0)
            plan.execute_peers(src, peers, stream)
            hdl.barrier(channel=0)
        ms = timed(fn)
        ingress = max(plan.counts(q)[1] for q in range(ws) if q != rank) * 2 if ws > 1 else 0
        if name == "config4":
            ingress = (ws - 1) * src.numel() * 2
        out[name] = {"ms": ms, "ingress_bytes_per_gpu": ingress, "bus_GBps": ingress / (ms * 1e-3) / 1e9,
                     "frac_of_900": ingress / (ms * 1e-3) / 1e9 / 900}
        del buf, hdl, src
    # §8(f) f2+f3: pull reduce-scatter -- one K4 kernel per rank reads every partial from its owner's
    # symmetric buffer over NVLink and writes the sum (no staging, no NCCL)
    rs = synth.reduce_scatter(ws, 16384, 8192, "bf16")
    plan = axe.RedistPlan(rs["src"], rs["src_st"], rs["dst"], rs["dst_st"], 2, ws, rank, reduce_dtype="bf16")
    sbuf = symm_mem.empty(synth.storage_cells(rs["src_st"]), dtype=torch.bfloat16, device=f"cuda:{local}")
    sbuf.normal_()
    hdl = symm_mem.rendezvous(sbuf, dist.group.WORLD)
    peers = [int(p) for p in hdl.buffer_ptrs]
    dst = torch.empty(synth.storage_cells(rs["dst_st"]), dtype=torch.bfloat16, device="cuda")

    def fn_rs():
        hdl.barrier(channel=0)
        plan.execute_peers_reduce(peers, dst, stream)
        hdl.barrier(channel=0)
    ms = timed(fn_rs)
    bus = (ws - 1) / ws * sbuf.numel() * 2
    out["reduce_scatter_pull"] = {"ms": ms, "bus_bytes_per_gpu": bus, "bus_GBps": bus / (ms * 1e-3) / 1e9,
                                  "pull_regions": plan.describe()["pull_regions"]}
    # NVLS: one multimem.ld_reduce per 16-byte vector on the multicast address; checked against
    # the pull result (the switch's summation order differs, so the check is a bf16 tolerance)
    mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
    has_mc = torch.tensor([1 if mc else 0], device="cuda")
    dist.all_reduce(has_mc, op=dist.ReduceOp.MIN)
    if int(has_mc.item()) and plan.describe().get("multicast"):
        dst2 = torch.empty_like(dst)

        def fn_mc():
            hdl.barrier(channel=0)
            plan.execute_multicast_reduce(mc, dst2, stream)
            hdl.barrier(channel=0)
        ms2 = timed(fn_mc)
        fn_rs()
        torch.cuda.synchronize()
        diff = (dst2.float() - dst.float()).abs().max().reshape(1)
        dist.all_reduce(diff, op=dist.ReduceOp.MAX)
        out["reduce_scatter_multimem"] = {"ms": ms2, "bus_GBps": bus / (ms2 * 1e-3) / 1e9,
                                          "max_abs_diff_vs_pull": float(diff.item())}
        del dst2
    else:
        out["reduce_scatter_multimem"] = {"skipped": "no multicast object (NVLS) on this group"}
    del sbuf, hdl, dst
    return out


def _time_plan(torch, plan, reps=10):
    """Graph-replayed back-to-back executes over rotating buffers (> 4x L2); returns ms per launch."""
    sb, db = plan.sizes()
    l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size
    # > 4x L2 of rotation, and >= 2 GiB (up to 32 pairs) so independent copies may overlap (PDL) as in
    # the headline loop
    pairs = max(1, min(32, max(-(-4 * l2 // (sb + db)), (2 << 30) // (sb + db))))
    srcs = [torch.empty(sb, dtype=torch.uint8, device="cuda").random_() for _ in range(pairs)]
    dsts = [torch.empty(db, dtype=torch.uint8, device="cuda") for _ in range(pairs)]
    G = pairs * max(1, 32 // pairs) if sb < (1 << 27) else pairs
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for j in range(G):
            plan.execute(srcs[j % pairs], dsts[j % pairs], torch.cuda.current_stream())
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * G)
    del srcs, dsts, g
    torch.cuda.empty_cache()
    return ms


def measure_extras(axe, torch):
    """The other single-GPU rows of SURVEY §8(a) (a6 reverse direction, a7 register permutes, K2 staging),
    each timed like the headline; GB/s = es * (1 + E_R) bytes per element / time."""
    peak, _ = peaks()
    rows = {}
    cases = {
        "config1_8x8_lane_warp_replica": synth.config1(),
        "config2_reverse_tiles_to_rowmajor": synth.config2(reverse=True),
        "config3a_mma_c_to_tcgen05_rows": synth.config3(65536, "a"),
        "config3b_mma_c_8x8_transposed": synth.config3(65536, "b"),
        "transpose_8192sq_bf16": dict(es=2, src=synth.layout([(8192, 8192), (8192, 1)]),
                                                 src_st=synth.linear_storage(8192 * 8192),
                                                 dst=synth.layout([(8192, 1), (8192, 8192)]),
                                                 dst_st=synth.linear_storage(8192 * 8192)),
        "transpose_8192sq_f32": dict(es=4, src=synth.layout([(8192, 8192), (8192, 1)]),
                                     src_st=synth.linear_storage(8192 * 8192),
                                     dst=synth.layout([(8192, 1), (8192, 8192)]),
                                     dst_st=synth.linear_storage(8192 * 8192)),
        "transpose_8192x4096_f64": dict(es=8, src=synth.layout([(8192, 4096), (4096, 1)]),
                                        src_st=synth.linear_storage(8192 * 4096),
                                        dst=synth.layout([(8192, 1), (4096, 8192)]),
                                        dst_st=synth.linear_storage(8192 * 4096)),
        # whole-vector extents that are not whole tiles: K7 with its ragged last tile row masked
        "transpose_8000sq_bf16_ragged_edges": dict(es=2, src=synth.layout([(8000, 8000), (8000, 1)]),
                                                   src_st=synth.linear_storage(8000 * 8000),
                                                   dst=synth.layout([(8000, 1), (8000, 8000)]),
                                                   dst_st=synth.linear_storage(8000 * 8000)),
        # config 2 at 16384^2 (512 MiB a side): the lowered schedule on its in-order grid
        "config2_16384sq_lowered": synth.config2(16384),
        # non-nested digit systems: (3*2^13, 2*2^13) padded -> (2*2^13, 3*2^13) padded, 768 MiB each side
        "nonnested_3x2_bf16_dual": dict(es=2, src=synth.layout([(3 << 13, (2 << 13) + 64), (2 << 13, 1)]),
                                        src_st=synth.linear_storage((3 << 13) * ((2 << 13) + 64)),
                                        dst=synth.layout([(2 << 13, (3 << 13) + 128), (3 << 13, 1)]),
                                        dst_st=synth.linear_storage((2 << 13) * ((3 << 13) + 128))),
    }
    for name, cfg in cases.items():
        plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["es"])
        ms = _time_plan(torch, plan)
        alg = plan.src.E_D * cfg["es"] * (1 + plan.dst.E_R)
        gbs = alg / (ms * 1e-3) / 1e9
        rows[name] = {"kernel": plan.describe()["kernel"], "us": ms * 1e3, "GBps": gbs, "frac_of_measured": gbs / peak,
                      "alg_bytes": alg}
    # §8(f) f3: the K4 sum over the leading dimension (K partials read once, the sum written once)
    for name, cfg in {"reduce_k8_bf16_8192x4096": synth.reduce_local(8, 8192, 4096, "bf16"),
                      "reduce_k8_bf16_into_sw128_tiles": synth.reduce_local(8, 8192, 4096, "bf16", tiled=True)}.items():
        plan = axe.ReducePlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["dtype"])
        ms = _time_plan(torch, plan)
        alg = sum(plan.sizes())
        gbs = alg / (ms * 1e-3) / 1e9
        rows[name] = {"kernel": plan.describe()["kernel"], "us": ms * 1e3, "GBps": gbs, "frac_of_measured": gbs / peak,
                      "alg_bytes": alg}
    return rows


def run_axe(args):
    import torch
    ws, rank, local = dist_init(args)
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2601_19092_b200 as axe

    cfg = synth.config2()
    es = cfg["es"]
    n = 4096
    nbytes = n * n * es
    alg_bytes = 2 * nbytes  # es * (1 + E_R) per element, E_R = 1
    plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es)
    desc = plan.describe()
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    # buffer pairs: > 4x L2 of footprint (32 pairs, 2 GiB), so no step finds its source in L2.  Every
    # kernel waits for its predecessor (griddepcontrol.wait) by default; AXE_PDL_OVERLAP=1 lets copies
    # proven disjoint from the in-flight ones skip it (opt-in, reported in roofline.pdl_overlap)
    pairs = max(int(os.environ.get("AXE_BENCH_PAIRS", "32")), -(-4 * l2 // (2 * nbytes)))
    g = torch.Generator(device="cuda").manual_seed(cfg["seed"] + rank)
    srcs = [torch.randint(-2**31, 2**31 - 1, (nbytes // 4,), dtype=torch.int32, device="cuda", generator=g)
            for _ in range(pairs)]
    dsts = [torch.empty_like(s) for s in srcs]
    stream = torch.cuda.current_stream()

    def step(i, st=None):
        plan.execute(srcs[i % pairs], dsts[i % pairs], st or stream)

    for i in range(max(3, args.warmup)):
        step(i)
    torch.cuda.synchronize()

    # The timed region is exactly args.steps launches, captured once in a CUDA graph (one kernel per
    # step, each on the next buffer pair) and replayed once: the device time of those launches, not
    # the host's ctypes / launch path.  A short sleep kernel ahead of the start event keeps the
    # stream busy while the host submits the graph, so the region starts with the first copy.
    graph = None
    in_graph_events = None
    if not args.no_graph:
        n_cap = axe.kernel_launch_count()
        graph = torch.cuda.CUDAGraph()
        cap_stream = torch.cuda.Stream()
        cap_stream.wait_stream(stream)
        try:  # timing events recorded by the graph itself (event-record nodes) around exactly the K steps
            in_graph_events = (torch.cuda.Event(enable_timing=True, external=True),
                               torch.cuda.Event(enable_timing=True, external=True))
        except TypeError:
            in_graph_events = None
        with torch.cuda.graph(graph, stream=cap_stream):
            if in_graph_events:
                in_graph_events[0].record(torch.cuda.current_stream())
            for j in range(args.steps):
                step(j, torch.cuda.current_stream())
            if in_graph_events:
                in_graph_events[1].record(torch.cuda.current_stream())
        assert axe.kernel_launch_count() - n_cap == args.steps, "one kernel per step"
        torch.cuda.synchronize()

    def run_steps():
        """args.steps steps on `stream`; returns the number of library kernels launched."""
        if graph is None:
            for i in range(args.steps):
                step(i)
        else:
            graph.replay()
        return args.steps

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        # keep the GPU loaded long enough for the clock sampler to see the timed region's clocks
        t_end = time.perf_counter() + 0.4
        while time.perf_counter() < t_end:
            for _ in range(max(1, 512 // args.steps)):
                run_steps()
            torch.cuda.synchronize()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # untimed warm-up copies on other buffer pairs right before the region (the GPU stays busy with
        # memory traffic while the host enqueues the start event and the graph: no idle gap, no cold HBM)
        # (pairs the first timed steps use are not among them, or were last touched >= 7 copies earlier)
        for j in range(max(args.steps, pairs) - 16, max(args.steps, pairs)):
            step(j)
        n0 = axe.kernel_launch_count()
        ev0.record(stream)
        launches = run_steps()
        ev1.record(stream)
        barrier()
        direct = axe.kernel_launch_count() - n0
        assert direct == (0 if graph is not None else args.steps)
        ms = ev0.elapsed_time(ev1)
        ms_outer = ms
        if in_graph_events:  # the graph's own event nodes: the K steps without the graph launch latency
            ms = in_graph_events[0].elapsed_time(in_graph_events[1])
        # the same steps launched one by one from Python (ctypes + launch path on the host each step)
        torch.cuda._sleep(2_000_000)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for i in range(args.steps):
            step(i)
        d1.record(stream)
        torch.cuda.synchronize()
        direct_ms = d0.elapsed_time(d1) / args.steps
        t0 = time.perf_counter()
        for i in range(200):
            step(i)
        host_us = (time.perf_counter() - t0) / 200 * 1e6
        torch.cuda.synchronize()
        # isolated launches bracketed by events (same stream), for reference
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
        for j, (a, b) in enumerate(evs):
            a.record(stream)
            step(j)
            b.record(stream)
        torch.cuda.synchronize()
    iso_ms = statistics.median(a.elapsed_time(b) for a, b in evs)
    k_ms = ms / args.steps  # average launch duration over the timed region (one kernel per step)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = ws * alg_bytes / (ms_step * 1e-3) / 1e9

    # end to end through the public host-buffer call: H2D of the inputs + kernel + D2H of the result.
    # Like a serving loop, consecutive steps alternate E2E_STREAMS user streams and host / device buffer
    # sets, so step k+1's host->device copies overlap step k's device->host copies on the PCIe link
    # (stream order alone would serialise the two directions across steps).
    ns = max(1, int(os.environ.get("AXE_E2E_STREAMS", "2")))
    # the same copy, planned with 2 host slabs of 16 MiB (measured best with 2 overlapping streams:
    # 91 GB/s vs 86 (4 slabs) and 81 (8 slabs); PCIe moves large transfers more efficiently)
    slabs = int(os.environ.get("AXE_E2E_SLABS", "2"))
    eplan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, host_slabs=slabs)
    hs = [torch.empty(nbytes, dtype=torch.uint8).pin_memory() for _ in range(ns)]
    for h in hs:
        h.copy_(srcs[0].view(torch.uint8).cpu())
    hd = [torch.empty(nbytes, dtype=torch.uint8).pin_memory() for _ in range(ns)]
    e_streams = [stream] + [torch.cuda.Stream() for _ in range(ns - 1)]
    e_steps = max(5, min(50, args.steps))
    for i in range(2 * ns):
        eplan.execute_host(hs[i % ns], hd[i % ns], srcs[i % pairs], dsts[i % pairs], e_streams[i % ns])
    for s_ in e_streams:
        s_.synchronize()
    barrier()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s_ in e_streams[1:]:
        s_.wait_event(e0)
    for i in range(e_steps):
        eplan.execute_host(hs[i % ns], hd[i % ns], srcs[i % pairs], dsts[i % pairs], e_streams[i % ns])
    for s_ in e_streams[1:]:
        stream.wait_stream(s_)
    e1.record(stream)
    barrier()
    e_ms = e0.elapsed_time(e1) / e_steps
    if dist:
        t = torch.tensor([e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e = ws * alg_bytes / (e_ms * 1e-3) / 1e9

    reshard = None
    if (ws > 1 or args.force_reshard) and not args.no_reshard:
        try:
            if dist is None:
                import socket
                import torch.distributed as dist
                if "RANK" not in os.environ:  # --force-reshard at N = 1 without torchrun: a 1-rank group
                    s = socket.socket()
                    s.bind(("127.0.0.1", 0))
                    os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                                      MASTER_PORT=str(s.getsockname()[1]))
                    s.close()
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            reshard = measure_reshard(axe, torch, dist, ws, rank, local, stream)
        except Exception as e:  # keep the contract line even if the reshard leg fails
            reshard = {"error": f"{type(e).__name__}: {e}"}
    extras = None
    if ws == 1 and not args.no_extras:
        try:
            extras = measure_extras(axe, torch)
        except Exception as e:
            extras = {"error": f"{type(e).__name__}: {e}"}

    peak, peak_src = peaks()
    achieved = alg_bytes / (k_ms * 1e-3) / 1e9
    out = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            nthreads = os.cpu_count() or 1
            gbs, bands, sec = oracle_sample_seconds(args.cpu_seconds, nthreads)
            gbs1, bands1, sec1 = oracle_sample_seconds(max(1.0, args.cpu_seconds / 4), 1)
            model = None
            try:
                with open("/proc/cpuinfo") as f:
                    model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
            except OSError:
                pass
            cpu = {"value": gbs, "unit": "GB/s", "cores": nthreads, "kind": "oracle",
                   "sample": f"{bands} 64-row bands of the config-2 conversion ({sec:.1f} s)",
                   "value_1_thread": gbs1, "sample_1_thread": f"{bands1} bands ({sec1:.1f} s)", "cpu_model": model}
        out = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "elem": "bf16 bit patterns (bitwise copy)",
                       "l2_defeat": f"rotating {pairs} src/dst pairs ({pairs * 2 * nbytes >> 20} MiB) > 4x L2 ({l2 >> 20} MiB)",
                       "parallelism": f"replicas x{ws}", "kernel": desc.get("kernel"),
                       "vec_bytes": desc.get("vec_bytes")},
            "pct_of_peak": 100.0 * (value / ws) / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(), "peak_source": peak_src,
                         "kernel_ms": k_ms, "event_bracketed_single_launch_ms": iso_ms,
                         "event_bracketed_note": "one launch between two event records (no PDL overlap, event and "
                                                 "launch latency included); not the kernel's duration",
                         "direct_launch_ms": direct_ms,
                         "host_us_per_call": host_us, "alg_bytes_per_launch": alg_bytes,
                         "pdl_overlap": os.environ.get("AXE_PDL_OVERLAP", "0") == "1",
                         "graph_replay_ms_incl_launch": ms_outer if graph is not None else None,
                         "timing": (f"CUDA event-record nodes inside one replayed graph of exactly {args.steps} launches"
                                    if in_graph_events else
                                    f"CUDA events around one replay of a graph of exactly {args.steps} launches")
                         if graph is not None else "CUDA events over the timed region / launches"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                    "api": "axe_copy_plan_execute_host (pinned host buffers)", "ms_per_step": e_ms,
                    "streams": ns, "host_slabs": slabs,
                    "pcie_note": "steps alternate user streams so H2D and D2H overlap"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if reshard is not None:
            out["reshard"] = reshard
        if extras is not None:
            out["other_rows"] = extras
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="axe", choices=["axe", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every step directly (no CUDA graph)")
    ap.add_argument("--no-reshard", action="store_true", help="skip the N>1 axe_redistribute measurements")
    ap.add_argument("--force-reshard", action="store_true", help="run the reshard leg even at N=1 (code-path check)")
    ap.add_argument("--no-extras", action="store_true", help="skip the other single-GPU SURVEY §8 rows")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_axe(args)


if __name__ == "__main__":
    main()
