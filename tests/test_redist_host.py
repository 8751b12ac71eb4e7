"""Host logic of axe_redistribute (no GPU): plan patterns, owner balance, and a
CPU re-enactment of every rank's plan (pack via the send maps, exchange, unpack
via the receive maps, local maps) compared with the oracle's redistribute --
in one process and in a real world_size-2 gloo job."""
import os

import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage

import paper_2601_19092_b200 as axe


def plans_for(cfg, n):
    return [axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], cfg["es"], n, r) for r in range(n)]


def rank_inputs(cfg, n):
    es = cfg["es"]
    ed, _ = oracle.sizes(cfg["src"])
    v = synth.values(ed, es, cfg["seed"])
    fill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, cfg["seed"] + 3)
    return oracle.scatter_ranks(cfg["src"], cfg["src_st"], v, es, n, fill)


def expected(cfg, n, src):
    es = cfg["es"]
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, cfg["seed"])
    dst = [dfill.copy() for _ in range(n)]
    oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], dst, es)
    return dfill, dst


def elems(buf, es):
    return buf.view({1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[es])


def cpu_enact(plans, src, dfill, es):
    """Replay the plans with numpy: the wire carries the k-th sent element to the k-th received slot."""
    n = len(plans)
    dst = [dfill.copy() for _ in range(n)]
    for r, p in enumerate(plans):
        s, d = elems(src[r], es), elems(dst[r], es)
        for k in range(p.counts(r)[0]):
            a, b = p.map(2, r, k)
            d[b] = s[a]
    for r, p in enumerate(plans):
        for q in range(n):
            if q == r:
                continue
            cnt, _ = p.counts(q)
            wire = [elems(src[r], es)[p.map(0, q, k)[0]] for k in range(cnt)]
            assert plans[q].counts(r)[1] == cnt
            d = elems(dst[q], es)
            for k in range(cnt):
                d[plans[q].map(1, r, k)[0]] = wire[k]
    return dst


@pytest.mark.parametrize("P", [2, 4, 8])
def test_config4_is_allgather(P):
    cfg = synth.config4(P, 16384)
    for r in (0, P - 1):
        d = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, P, r).describe()
        assert d["pattern"] == "allgather" and d["packs"] == 0 and d["unpacks"] == 0
        assert d["block_elems"] == 16384 * 16384 // P


def test_config5_pairwise_balanced():
    """balanced owners make config 5 a pairwise exchange (a,b) <-> (1-a,b), 64 MiB each way."""
    cfg = synth.config5()
    for r in range(8):
        p = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, 8, r)
        d = p.describe()
        assert d["pattern"] == "exchange" and d["sends"] == 1 and d["recvs"] == 1 and d["unpacks"] == 0
        peer = r ^ 4
        for q in range(8):
            s, rc = p.counts(q)
            if q == peer:
                assert s == rc == 16384 * 2048
            elif q != r:
                assert s == rc == 0


@pytest.mark.parametrize("mk", [lambda: synth.config4(2, 32), lambda: synth.config4(4, 16),
                                lambda: synth.config5(16, 16), lambda: synth.config5(8, 8, 2, 2)])
def test_cpu_enactment_matches_oracle(mk):
    cfg = mk()
    n = cfg["nranks"]
    src = rank_inputs(cfg, n)
    dfill, exp = expected(cfg, n, src)
    got = cpu_enact(plans_for(cfg, n), src, dfill, cfg["es"])
    for r in range(n):
        assert np.array_equal(got[r], exp[r]), r


def test_shard_axis_change_1d_alltoall():
    """1-D 4-way S(0) -> S(1) (an all-to-all), packs on the sender side."""
    R, Cn, P = 16, 16, 4
    src = layout([(P, 1, "gpuid"), (R // P, Cn), (Cn, 1)])
    dst = layout([(R, Cn // P), (P, 1, "gpuid"), (Cn // P, 1)])
    cfg = dict(name="s0s1", es=4, src=src, src_st=linear_storage(R * Cn // P), dst=dst,
               dst_st=linear_storage(R * Cn // P), seed=9, nranks=P)
    src_b = rank_inputs(cfg, P)
    dfill, exp = expected(cfg, P, src_b)
    got = cpu_enact(plans_for(cfg, P), src_b, dfill, 4)
    for r in range(P):
        assert np.array_equal(got[r], exp[r])


def test_redist_errors():
    cfg = synth.config4(4, 16)
    with pytest.raises(axe.AxeError) as e:      # gpuid reaches 3 with only 2 ranks
        axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, 2, 0)
    assert e.value.name == "AXE_ERR_BOUNDS"
    bad = layout([(16, 16), (16, 1)], [(4, 1, "gpuid"), (2, 1, "gpuid")])   # two replicas on one rank cell
    with pytest.raises(axe.AxeError) as e:
        axe.RedistPlan(cfg["src"], cfg["src_st"], bad, linear_storage(256), 2, 8, 0)
    assert e.value.name == "AXE_ERR_NONINJECTIVE"


# ------------------------------------------------------------------ world_size 2, gloo
def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for cfg in (synth.config4(2, 32), synth.config5(16, 16, 2, 1)):
            es = cfg["es"]
            n = cfg["nranks"]
            assert n == world
            src = rank_inputs(cfg, n)            # every rank can regenerate every rank's input
            dfill, exp = expected(cfg, n, src)
            p = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, n, rank)
            s = elems(src[rank], es)
            d = elems(dfill.copy(), es)
            for k in range(p.counts(rank)[0]):
                a, b = p.map(2, rank, k)
                d[b] = s[a]
            peer = 1 - rank
            ns, nr = p.counts(peer)
            out = torch.from_numpy(np.array([s[p.map(0, peer, k)[0]] for k in range(ns)], dtype=s.dtype).astype(np.int64))
            inc = torch.empty(nr, dtype=torch.int64)
            reqs = [dist.isend(out, peer), dist.irecv(inc, peer)]
            for r_ in reqs:
                r_.wait()
            for k in range(nr):
                d[p.map(1, peer, k)[0]] = inc[k].item()
            ok = np.array_equal(d.view(np.uint8), exp[rank])
            q.put((rank, cfg["name"], bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_redistribute():
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


@pytest.mark.parametrize("mk", [lambda: synth.config5(64, 32), lambda: synth.config4(4, 32)])
def test_chunked_wire_order(mk, monkeypatch):
    """Wire chunks (packing chunk c+1 while chunk c is on the wire): the chunk-major wire order of the
    sender's maps matches the receiver's, and the enactment still equals the oracle."""
    monkeypatch.setenv("AXE_REDIST_CHUNK_BYTES", "128")
    cfg = mk()
    n = cfg["nranks"]
    plans = plans_for(cfg, n)
    assert plans[0].describe()["wire_chunks"] >= 2
    src = rank_inputs(cfg, n)
    dfill, exp = expected(cfg, n, src)
    got = cpu_enact(plans, src, dfill, cfg["es"])
    for r in range(n):
        assert np.array_equal(got[r], exp[r]), r
