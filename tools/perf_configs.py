#!/usr/bin/env python
"""Development timing of every single-GPU BASELINE config (not the bench contract line).

For each config: plan once, rotate over buffer pairs whose footprint exceeds
4x L2, capture G back-to-back executes in a CUDA graph, replay, report
algorithmic GB/s (es * (1 + E_R) bytes per element) and the
fraction of the measured HBM copy peak.  Kernels can be forced with
--kernel (auto|generic|vector|tma|tile).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2601_19092_b200 as axe  # noqa: E402


def transpose_cfg(R, C, es):
    return dict(name=f"transpose{R}x{C}x{es}", es=es, src=synth.layout([(R, C), (C, 1)]),
                src_st=synth.linear_storage(R * C), dst=synth.layout([(R, 1), (C, R)]),
                dst_st=synth.linear_storage(R * C), seed=7)


def nonnested_cfg(k=13, es=2):
    """(3*2^k, 2*2^k) row pitch 2*2^k + 64 -> the same x re-split as (2*2^k, 3*2^k), pitch 3*2^k + 128:
    innermost extents share only 2^k -- K8 dual decoding (K0 when forced generic)."""
    p, q, g = 3, 2, 1 << k
    A1, A2, B1, B2 = p * g, q * g, q * g, p * g
    return dict(name=f"nonnested_3x2_k{k}", es=es, src=synth.layout([(A1, A2 + 64), (A2, 1)]),
                src_st=synth.linear_storage(A1 * (A2 + 64)), dst=synth.layout([(B1, B2 + 128), (B2, 1)]),
                dst_st=synth.linear_storage(B1 * (B2 + 128)), seed=9)


def nonnested_gcd1_cfg(m=32, es=2):
    """(2187 m, 4096) row-major, pitch 4096 + 64 -> the same x re-split as (4096 m, 2187), pitch 2187 + 5:
    innermost extents 4096 and 3^7 share no factor -- element by element (K8 with an empty inner block;
    K0 when forced generic)."""
    A1, A2, B1, B2 = 2187 * m, 4096, 4096 * m, 2187
    return dict(name=f"nonnested_gcd1_m{m}", es=es, src=synth.layout([(A1, A2 + 64), (A2, 1)]),
                src_st=synth.linear_storage(A1 * (A2 + 64)), dst=synth.layout([(B1, B2 + 5), (B2, 1)]),
                dst_st=synth.linear_storage(B1 * (B2 + 5)), seed=11)


CONFIGS = {
    "nonnested_3x2": lambda: nonnested_cfg(13),
    "nonnested_gcd1": lambda: nonnested_gcd1_cfg(32),
    "config2": lambda: synth.config2(),
    "config2r": lambda: synth.config2(reverse=True),
    "config2_16k": lambda: synth.config2(16384),
    "config2_8k": lambda: synth.config2(8192),
    "config2r_16k": lambda: synth.config2(16384, reverse=True),
    "config3a": lambda: synth.config3(65536, "a"),
    "config3b": lambda: synth.config3(65536, "b"),
    "identity_4g": lambda: dict(name="identity_4g", es=2, src=synth.layout([(1 << 31, 1)]),
                                src_st=synth.linear_storage(1 << 31), dst=synth.layout([(1 << 31, 1)]),
                                dst_st=synth.linear_storage(1 << 31), seed=3),
    "identity_1g": lambda: dict(name="identity_1g", es=2, src=synth.layout([(1 << 29, 1)]),
                                src_st=synth.linear_storage(1 << 29), dst=synth.layout([(1 << 29, 1)]),
                                dst_st=synth.linear_storage(1 << 29), seed=3),
    "rows_4k": lambda: dict(name="rows_4k", es=2, src=synth.layout([(16384, 8192), (2048, 1)]),
                            src_st=synth.linear_storage(16384 * 8192), dst=synth.layout([(16384, 2048), (2048, 1)]),
                            dst_st=synth.linear_storage(16384 * 2048), seed=5),
    "rows_1k": lambda: dict(name="rows_1k", es=2, src=synth.layout([(65536, 2048), (512, 1)]),
                            src_st=synth.linear_storage(65536 * 2048), dst=synth.layout([(65536, 512), (512, 1)]),
                            dst_st=synth.linear_storage(65536 * 512), seed=5),
    "transpose_bf16": lambda: transpose_cfg(8192, 8192, 2),
    "transpose_f32": lambda: transpose_cfg(8192, 8192, 4),
    "transpose_f64": lambda: transpose_cfg(8192, 4096, 8),
    "transpose_bf16_8000": lambda: transpose_cfg(8000, 8000, 2),
    "transpose_f32_8000x8192": lambda: transpose_cfg(8000, 8192, 4),
    "transpose_bf16_4095x4097": lambda: transpose_cfg(4095, 4097, 2),
    "transpose_f32_4095x4097": lambda: transpose_cfg(4095, 4097, 4),
    "transpose_u8_8191x8193": lambda: transpose_cfg(8191, 8193, 1),
    # padded pitches (8192 + 32 elements on both sides): does the 32 KiB power-of-two stride matter?
    "transpose_f32_pad": lambda: dict(name="transpose_f32_pad", es=4,
                                      src=synth.layout([(8192, 8224), (8192, 1)]),
                                      src_st=synth.linear_storage(8192 * 8224),
                                      dst=synth.layout([(8192, 1), (8192, 8224)]),
                                      dst_st=synth.linear_storage(8192 * 8224), seed=7),
}


def time_cfg(cfg, kernel, reps=20):
    es = cfg["es"]
    plan = axe.CopyPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, kernel)
    sb, db = plan.sizes()
    ed = plan.src.E_D
    er = plan.dst.E_R
    alg = ed * es * (1 + er)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    pairs = max(1, min(32, -(-4 * l2 // (sb + db)), (16 << 30) // (sb + db)))
    pairs = max(pairs, min(32, (2 << 30) // (sb + db)))  # >= 2 GiB of rotation when it fits
    srcs = [torch.empty(sb, dtype=torch.uint8, device="cuda") for _ in range(pairs)]
    dsts = [torch.empty(db, dtype=torch.uint8, device="cuda") for _ in range(pairs)]
    for s in srcs:
        s.random_()
    G = pairs * max(1, 64 // pairs) if alg < (1 << 28) else pairs
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        for j in range(G):
            plan.execute(srcs[j % pairs], dsts[j % pairs], torch.cuda.current_stream())
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * G)
    gbs = alg / (ms * 1e-3) / 1e9
    d = plan.describe()
    del srcs, dsts, g
    torch.cuda.empty_cache()
    return {"config": cfg["name"], "kernel": d["kernel"], "mode": d.get("mode"), "us": ms * 1e3, "GB/s": gbs,
            "frac_measured": gbs / 6547.2, "alg_bytes": alg}


REDUCE = {
    "reduce_bf16_k8": lambda: synth.reduce_local(8, 8192, 4096, "bf16"),
    "reduce_bf16_k8_tiled": lambda: synth.reduce_local(8, 8192, 4096, "bf16", tiled=True),
    "reduce_f32_k8": lambda: synth.reduce_local(8, 8192, 2048, "f32"),
    "reduce_bf16_k2": lambda: synth.reduce_local(2, 16384, 8192, "bf16"),
    "reduce_bf16_k4": lambda: synth.reduce_local(4, 16384, 4096, "bf16"),
    "reduce_bf16_k3": lambda: synth.reduce_local(3, 16384, 8192, "bf16"),
    "reduce_bf16_k16": lambda: synth.reduce_local(16, 4096, 4096, "bf16"),
    # smaller outputs (2 / 8 MiB): the persistent grid or the in-order schedule (K4B / K4T were compared here)
    "reduce_bf16_k8_2m": lambda: synth.reduce_local(8, 1024, 1024, "bf16"),
    "reduce_bf16_k8_2m_tiled": lambda: synth.reduce_local(8, 1024, 1024, "bf16", tiled=True),
    "reduce_bf16_k8_8m": lambda: synth.reduce_local(8, 2048, 2048, "bf16"),
    "reduce_bf16_k8_8m_tiled": lambda: synth.reduce_local(8, 2048, 2048, "bf16", tiled=True),
    "reduce_bf16_k4_8m": lambda: synth.reduce_local(4, 2048, 2048, "bf16"),
}


def _graph_time(fn, G, reps):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for j in range(G):
            fn(j)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * G)


def time_reduce(name, reps=20):
    """K4 sum over the leading dimension; algorithmic bytes = K*Y*es read + Y*es written.  Also torch's
    own x.view(K, -1).sum(0) on the same bytes (library reference point, row-major case)."""
    cfg = REDUCE[name]()
    dt = cfg["dtype"]
    plan = axe.ReducePlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], dt)
    sb, db = plan.sizes()
    K = cfg["K"]
    alg = sb + db
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    pairs = max(1, min(4, -(-4 * l2 // (sb + db))))
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32}[dt]
    es = synth.DTYPE_SIZE[dt]
    srcs = [torch.randn(sb // es, device="cuda").to(tdt) for _ in range(pairs)]
    dsts = [torch.empty(db // es, dtype=tdt, device="cuda") for _ in range(pairs)]
    ms = _graph_time(lambda j: plan.execute(srcs[j % pairs], dsts[j % pairs], torch.cuda.current_stream()),
                     pairs * 4, reps)
    out = {"config": name, "kernel": plan.describe()["kernel"], "us": ms * 1e3, "GB/s": alg / (ms * 1e-3) / 1e9,
           "frac_measured": alg / (ms * 1e-3) / 1e9 / 6547.2, "alg_bytes": alg}
    if "tiled" not in name:
        tms = _graph_time(lambda j: torch.sum(srcs[j % pairs].view(K, -1), dim=0, out=dsts[j % pairs]), pairs * 4, reps)
        out["torch_sum_us"] = tms * 1e3
        out["torch_sum_GB/s"] = alg / (tms * 1e-3) / 1e9
    del srcs, dsts
    torch.cuda.empty_cache()
    return out


def torch_copy(nbytes, reps=20):
    """Reference point: torch's own copy_ of nbytes (read + write counted), same rotation and graph."""
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    pairs = max(1, min(8, -(-4 * l2 // (2 * nbytes))))
    srcs = [torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda") for _ in range(pairs)]
    dsts = [torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda") for _ in range(pairs)]
    G = pairs * 8
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream()):
        for j in range(G):
            dsts[j % pairs].copy_(srcs[j % pairs])
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * G)
    gbs = 2 * nbytes / (ms * 1e-3) / 1e9
    return {"config": f"torch_copy_{nbytes >> 20}MiB", "us": ms * 1e3, "GB/s": gbs, "frac_measured": gbs / 6547.2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--only", default="")
    ap.add_argument("--torch-copy", action="store_true")
    ap.add_argument("--reduce", action="store_true", help="time the K4 reduction rows instead")
    a = ap.parse_args()
    if a.reduce:
        for n in (a.only.split(",") if a.only else list(REDUCE)):
            print(json.dumps(time_reduce(n)), flush=True)
        return
    if a.torch_copy:
        for nb in (32 << 20, 1 << 30, 4 << 30):
            print(json.dumps(torch_copy(nb)), flush=True)
    names = a.only.split(",") if a.only else list(CONFIGS)
    for n in names:
        try:
            print(json.dumps(time_cfg(CONFIGS[n](), a.kernel)), flush=True)
        except Exception as e:  # report and continue
            print(json.dumps({"config": n, "error": str(e)}), flush=True)


if __name__ == "__main__":
    main()
