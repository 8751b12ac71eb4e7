"""Host logic of the reduction row (reading R24), no GPU:
K4 plan structure, the reduce-redistribute plan (partials exchanged into K
stage slabs, then summed), a CPU re-enactment of every rank's plan through the
plan maps (in one process and in a world_size-2 gloo job) compared with
oracle.reduce, and the error contract."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage

import paper_2601_19092_b200 as axe

ELEM = {"bf16": np.uint16, "f16": np.uint16, "f32": np.uint32, "f64": np.uint64, "i32": np.uint32, "i64": np.uint64}
NPF = {"f16": np.float16, "f32": np.float32, "f64": np.float64}


def test_local_plan_structure(monkeypatch):
    cfg = [synth.reduce_local(8, 64, 128, "bf16")[k] for k in ("src", "src_st", "dst", "dst_st")]
    d = axe.ReducePlan(*cfg, "bf16").describe()     # the vector form
    assert d["kernel"] == "reduce" and d["mode"] == "vector" and d["K"] == 8 and d["vec_bytes"] == 16 and d["table"]
    assert d["reduce_digits"] == [[8, 8192, 0]]          # k stride = one (64 x 128) slab, no destination stride
    assert d["streaming_stores"] == 0                     # 2-byte sums keep plain stores (measured)
    f = synth.reduce_local(8, 64, 64, "f32")
    d = axe.ReducePlan(f["src"], f["src_st"], f["dst"], f["dst_st"], "f32").describe()
    assert d["streaming_stores"] == 1                     # 4-byte sums: st.global.cs (measured 88.4 vs 94.9 us)
    big = synth.reduce_local(300, 4, 32, "f32")
    d = axe.ReducePlan(big["src"], big["src_st"], big["dst"], big["dst_st"], "f32").describe()
    assert d["K"] == 300 and not d["table"]             # decoded summand offsets beyond 256


def test_local_plan_errors():
    with pytest.raises(axe.AxeError) as e:
        axe.ReducePlan(layout([(30, 1)]), linear_storage(30), layout([(7, 1)]), linear_storage(7), "f32")
    assert e.value.name == "AXE_ERR_SIZE_MISMATCH"
    with pytest.raises(axe.AxeError) as e:                # destination collision
        axe.ReducePlan(layout([(4, 8), (8, 1)]), linear_storage(32), layout([(2, 1), (4, 1)]), linear_storage(8), "f32")
    assert e.value.name == "AXE_ERR_NONINJECTIVE"
    with pytest.raises(axe.AxeError) as e:                # gpuid belongs to the distributed form
        axe.ReducePlan(layout([(2, 1, "gpuid"), (8, 1)]), linear_storage(8), layout([(8, 1)]), linear_storage(8), "f32")
    assert e.value.name == "AXE_ERR_UNSUPPORTED_AXIS"
    ss, _k1 = axe.make_storage(linear_storage(8))
    h = C.c_void_p()
    a, b = axe.Layout([(2, 4), (4, 1)]), axe.Layout([(4, 1)])
    assert axe._lib.axe_reduce_plan_create(a.handle, C.byref(ss), b.handle, C.byref(ss), 99, C.byref(h)) == 1


@pytest.mark.parametrize("P", [2, 4, 8])
def test_reduce_scatter_plan(P):
    cfg = synth.reduce_scatter(P, 64, 64, "bf16")
    for r in range(P):
        p = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, P, r, reduce_dtype="bf16")
        d = p.describe()
        assert d["pattern"] == "reduce" and d["K"] == P
        ex = d["exchange"]
        # each rank sends its partial of every other rank's rows and receives P-1 partials of its own
        assert ex["send_elems"] == (P - 1) * 64 * 64 // P == ex["recv_elems"]
        assert ex["packs"] == 0 and ex["unpacks"] == 0  # partial rows and stage slabs are contiguous
        red = d["reduce"]
        assert red["mode"] == "vector"
        assert red["K"] == P and red["vectors"] * 16 == 64 * 64 // P * 2


@pytest.mark.parametrize("P", [2, 4, 8])
def test_all_reduce_plan_phases(P):
    """Replicated over >= 3 ranks: reduce-scatter into an even shard, then an all-gather (2(P-1)/P of a
    partial on the wire per GPU, as a ring all-reduce); over 2 ranks one exchange of the partials."""
    cfg = synth.all_reduce(P, 64, 64, "bf16")
    d = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, P, 0, reduce_dtype="bf16").describe()
    if P == 2:
        assert d["pattern"] == "reduce" and d["exchange"]["recv_elems"] == 64 * 64
    else:
        assert d["pattern"] == "reduce_scatter_allgather"
        assert d["phase_a"]["exchange"]["recv_elems"] == (P - 1) * 64 * 64 // P
        assert d["phase_b"]["pattern"] == "allgather" and d["phase_b"]["recv_elems"] == (P - 1) * 64 * 64 // P


def test_uncovered_destination_is_rejected():
    """The slab sum writes every cell of the local dst storage; a destination image that misses cells is
    refused instead of overwriting them (R24)."""
    P = 2
    src = layout([(P, 1, "gpuid"), (16, 1)])
    dst = layout([(P, 1, "gpuid"), (8, 2)])        # every other cell of a 16-cell shard
    with pytest.raises(axe.AxeError) as e:
        axe.RedistPlan(src, linear_storage(16), dst, linear_storage(16), 4, P, 0, reduce_dtype="f32")
    assert e.value.name == "AXE_ERR_UNSUPPORTED"


def enact_rank(p, rank, n, K, C_cells, dtype, src_of, wire_in):
    """Stage slabs from the plan maps (local map + the received wire), then the slab sum in fp64, rounded once."""
    et = ELEM[dtype]
    stage = np.zeros(K * C_cells, et)
    s = src_of(rank).view(et)
    for k in range(p.counts(rank)[0]):
        a, b = p.map(2, rank, k)
        stage[b] = s[a]
    for q in range(n):
        if q == rank:
            continue
        w = wire_in(q)
        assert len(w) == p.counts(q)[1]
        for k in range(len(w)):
            stage[p.map(1, q, k)[0]] = w[k]
    slabs = stage.reshape(K, C_cells)
    if dtype in ("i32", "i64"):
        return slabs.sum(axis=0, dtype=et).view(np.uint8)
    if dtype == "bf16":
        import torch
        f = torch.from_numpy(slabs.view(np.int16).copy()).view(torch.bfloat16).double().sum(0)
        return f.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint8)
    return slabs.view(NPF[dtype]).astype(np.float64).sum(axis=0).astype(NPF[dtype]).view(np.uint8)


def dist_inputs(cfg, dtype, seed=5):
    n, es = cfg["nranks"], synth.DTYPE_SIZE[dtype]
    ed, _ = oracle.sizes(cfg["src"])
    vals = synth.numbers(ed, dtype, seed, "narrow")  # exact fp64 sums: the enactment sums by numpy
    fill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, seed + 1)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], vals, es, n, fill)
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, seed + 2)
    exp = [dfill.copy() for _ in range(n)]
    oracle.reduce(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, dtype, nranks=n)
    return src, exp


@pytest.mark.parametrize("mk,dtype", [(lambda: synth.reduce_scatter(4, 16, 8, "f16"), "f16"),
                                      (lambda: synth.all_reduce(3, 8, 8, "bf16"), "bf16"),
                                      (lambda: synth.all_reduce(4, 8, 16, "f32"), "f32"),
                                      (lambda: synth.reduce_scatter(2, 8, 16, "i32"), "i32")])
def test_cpu_enactment_matches_oracle(mk, dtype):
    cfg = mk()
    n = cfg["nranks"]
    src, exp = dist_inputs(cfg, dtype)
    ed, _ = oracle.sizes(cfg["src"])
    edd, _ = oracle.sizes(cfg["dst"])
    K, Cc = ed // edd, synth.storage_cells(cfg["dst_st"])
    plans = [axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 0, n, r, reduce_dtype=dtype)
             for r in range(n)]
    et = ELEM[dtype]
    two_phase = plans[0].describe()["pattern"] == "reduce_scatter_allgather"
    red = [p.phase(0) for p in plans] if two_phase else plans
    if two_phase:
        Cc = edd // n                      # phase a reduces into (n, E_D/n):(1@gpuid, 1@m)

    def wire(sender, receiver):
        p = red[sender]
        s = src[sender].view(et)
        return np.array([s[p.map(0, receiver, k)[0]] for k in range(p.counts(receiver)[0])], et)

    got = [enact_rank(red[r], r, n, K, Cc, dtype, lambda g: src[g], lambda q: wire(q, r)) for r in range(n)]
    if two_phase:                          # phase b: a plain redistribution of the reduced shards
        gat = [p.phase(1) for p in plans]
        tmp = got
        got = [synth.sentinel(synth.storage_cells(cfg["dst_st"]) * synth.DTYPE_SIZE[dtype], 5 + 2) for _ in range(n)]
        for r in range(n):
            d = got[r].view(et)
            for k in range(gat[r].counts(r)[0]):
                a, b = gat[r].map(2, r, k)
                d[b] = tmp[r].view(et)[a]
            for q in range(n):
                if q != r:
                    for k in range(gat[r].counts(q)[1]):
                        d[gat[r].map(1, q, k)[0]] = tmp[q].view(et)[gat[q].map(0, r, k)[0]]
    for r in range(n):
        assert np.array_equal(got[r], exp[r]), r


# ------------------------------------------------------------------ world_size 2, gloo
def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for cfg, dtype in ((synth.reduce_scatter(2, 16, 32, "bf16"), "bf16"), (synth.all_reduce(2, 8, 16, "f32"), "f32")):
            src, exp = dist_inputs(cfg, dtype)     # every rank can regenerate every rank's input
            ed, _ = oracle.sizes(cfg["src"])
            edd, _ = oracle.sizes(cfg["dst"])
            K, Cc = ed // edd, synth.storage_cells(cfg["dst_st"])
            p = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 0, world, rank, reduce_dtype=dtype)
            et = ELEM[dtype]
            peer = 1 - rank
            ns, nr = p.counts(peer)
            s = src[rank].view(et)
            out = torch.from_numpy(np.array([s[p.map(0, peer, k)[0]] for k in range(ns)], et).astype(np.int64))
            inc = torch.empty(nr, dtype=torch.int64)
            reqs = [dist.isend(out, peer), dist.irecv(inc, peer)]
            for r_ in reqs:
                r_.wait()
            got = enact_rank(p, rank, world, K, Cc, dtype, lambda g: src[g], lambda q_: inc.numpy().astype(et))
            q.put((rank, cfg["name"], bool(np.array_equal(got, exp[rank]))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reduce_redistribute():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = [q.get(timeout=5) for _ in range(4)]
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, _, ok in res), res
