"""GPU parity of axe_redistribute's device path on one B200: every rank's plan
(pack kernels, exchange, unpack kernels, local copies) runs through
axe_redist_emulate, with device-to-device copies standing in for NCCL, and each
rank's destination buffer is compared bit-exactly with the oracle."""
import os

import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
NT = os.cpu_count() or 4


@pytest.fixture(scope="module")
def axe():
    assert torch.cuda.is_available()
    import paper_2601_19092_b200 as m
    return m


def run(axe, cfg, only=None):
    n, es = cfg["nranks"], cfg["es"]
    ed, _ = oracle.sizes(cfg["src"])
    v = synth.values(ed, es, cfg["seed"])
    sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, cfg["seed"] + 3)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], v, es, n, sfill, NT)
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, cfg["seed"])
    ranks = range(n) if only is None else only
    plans = [axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, n, r) for r in range(n)]
    s_dev = [torch.from_numpy(s).cuda() for s in src]
    d_dev = [torch.from_numpy(dfill).cuda() for _ in range(n)]
    axe.redist_emulate(plans, s_dev, d_dev)
    torch.cuda.synchronize()
    if only is None:   # one oracle pass fills every rank's expected buffer
        exp = [dfill.copy() for _ in range(n)]
        oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, es, nthreads=NT)
        for r in range(n):
            assert np.array_equal(d_dev[r].cpu().numpy(), exp[r]), f"{cfg['name']} rank {r}"
        return plans[0].describe()
    for r in ranks:
        exp = [None] * n
        exp[r] = dfill.copy()
        oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, es, only_rank=r,
                            nthreads=NT)
        got = d_dev[r].cpu().numpy()
        assert np.array_equal(got, exp[r]), f"{cfg['name']} rank {r}"
    return plans[0].describe()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_config4_small(axe, P):
    d = run(axe, synth.config4(P, 256))
    assert d["pattern"] == "allgather"


@pytest.mark.parametrize("shape", [(64, 32), (256, 128), (32, 16, 2, 2)])
def test_config5_small(axe, shape):
    d = run(axe, synth.config5(*shape))
    assert d["pattern"] == "exchange"


def test_config5_full_every_rank(axe):
    """BASELINE config 5 at full size (32768x8192 bf16 on the 2x4 mesh): all 8 ranks' destination buffers,
    every byte, against the oracle."""
    d = run(axe, synth.config5())
    assert d["pattern"] == "exchange"


@pytest.mark.parametrize("P", [2, 4, 8])
def test_config4_full_every_rank(axe, P):
    """BASELINE config 4 at full size (16384^2 bf16 shard(0) -> replicate, P = 2 / 4 / 8): every rank's
    512 MiB replica, every byte, against the oracle."""
    d = run(axe, synth.config4(P))
    assert d["pattern"] == "allgather"
    torch.cuda.empty_cache()


def test_nccl_comm_single_rank(axe):
    """The NCCL path on the one GPU a gpurun box has: a 1-rank communicator, axe_redistribute through
    the public call (plan cache + execute), checked against the oracle."""
    comm = axe.Comm(axe.get_unique_id(), 1, 0, torch.cuda.current_device())
    R, Cn = 64, 48
    src = layout([(R, Cn), (Cn, 1)])
    dst = layout([(R, 1), (Cn, R)], [(1, 1, "gpuid")])
    v = synth.values(R * Cn, 4, 5)
    x = torch.from_numpy(v.copy()).cuda()
    y = torch.zeros_like(x)
    axe.axe_redistribute(src, linear_storage(R * Cn), x, dst, linear_storage(R * Cn), y, 4, comm)
    torch.cuda.synchronize()
    exp = np.zeros_like(v)
    oracle.redistribute(src, linear_storage(R * Cn), [v], dst, linear_storage(R * Cn), [exp], 4)
    assert np.array_equal(y.cpu().numpy(), exp)
    del comm


@pytest.mark.parametrize("seed", range(8))
def test_random_meshes(axe, seed):
    """Random 1-D/2-D meshes: the shard axis, the sharded logical dimension and replication are drawn at random."""
    rng = np.random.default_rng(seed)
    A, B = [(2, 1), (2, 2), (4, 2), (1, 4)][seed % 4]
    n = A * B
    R, Cn = 16 * A * B, 8 * A * B
    def spec(kind):
        if kind == 0:      # rows over a, columns over b
            return (layout([(A, B, "gpuid"), (R // A, Cn // B), (B, 1, "gpuid"), (Cn // B, 1)]), R // A * Cn // B)
        if kind == 1:      # rows over a, replicated over b
            return layout([(A, B, "gpuid"), (R // A, Cn), (Cn, 1)], [(B, 1, "gpuid")]), R // A * Cn
        if kind == 2:      # columns over b, replicated over a
            return layout([(R, Cn // B), (B, 1, "gpuid"), (Cn // B, 1)], [(A, B, "gpuid")]), R * Cn // B
        return layout([(R, Cn), (Cn, 1)], [(n, 1, "gpuid")]), R * Cn   # fully replicated
    ks, kd = rng.integers(0, 4, 2)
    (src, sc), (dst, dc) = spec(int(ks)), spec(int(kd))
    cfg = dict(name=f"mesh{seed}", es=int(rng.choice([2, 4])), src=src, src_st=linear_storage(sc), dst=dst,
               dst_st=linear_storage(dc), seed=seed, nranks=n)
    run(axe, cfg)


@pytest.mark.parametrize("shape", [(256, 128), (64, 32, 2, 2)])
def test_config5_chunked_emulated(axe, shape, monkeypatch):
    """Per-chunk pack kernels and wire copies (AXE_REDIST_CHUNK_BYTES forces chunking at small sizes)."""
    monkeypatch.setenv("AXE_REDIST_CHUNK_BYTES", "256")
    d = run(axe, synth.config5(*shape))
    assert d["wire_chunks"] >= 2


@pytest.mark.parametrize("mk", [lambda: synth.config4(4, 256), lambda: synth.config5(256, 128),
                                lambda: synth.config5(64, 32, 2, 2)])
def test_one_sided_peer_stores(axe, mk):
    """axe_redist_plan_execute_peers: each rank's copy kernels write straight into the receivers' dst
    buffers (on one GPU the "peer" buffers are ordinary device buffers); result equals the oracle."""
    cfg = mk()
    n, es = cfg["nranks"], cfg["es"]
    ed, _ = oracle.sizes(cfg["src"])
    v = synth.values(ed, es, cfg["seed"])
    sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, cfg["seed"] + 3)
    src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], v, es, n, sfill, NT)
    dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, cfg["seed"])
    plans = [axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, n, r) for r in range(n)]
    s_dev = [torch.from_numpy(s).cuda() for s in src]
    d_dev = [torch.from_numpy(dfill).cuda() for _ in range(n)]
    for r in range(n):
        plans[r].execute_peers(s_dev[r], d_dev)
    torch.cuda.synchronize()
    exp = [dfill.copy() for _ in range(n)]
    oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, es, nthreads=NT)
    for r in range(n):
        assert np.array_equal(d_dev[r].cpu().numpy(), exp[r]), r


def test_comm_wait_timeout_aborts(axe):
    """axe_comm_wait: a stream still busy after the timeout aborts the communicator (AXE_ERR_TIMEOUT); every
    later call on it fails with AXE_ERR_NCCL instead of hanging; a fresh communicator works."""
    comm = axe.Comm(axe.get_unique_id(), 1, 0, torch.cuda.current_device())
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        torch.cuda._sleep(2_000_000_000)   # ~1 s of GPU time
    with pytest.raises(axe.AxeError) as e:
        comm.wait(st, timeout_ms=5)
    assert e.value.name == "AXE_ERR_TIMEOUT"
    R, Cn = 32, 16
    src = layout([(R, Cn), (Cn, 1)])
    dst = layout([(R, 1), (Cn, R)], [(1, 1, "gpuid")])
    x = torch.zeros(R * Cn, dtype=torch.int32, device="cuda")
    y = torch.zeros_like(x)
    plan = axe.RedistPlan(src, linear_storage(R * Cn), dst, linear_storage(R * Cn), 4, 1, 0)
    with pytest.raises(axe.AxeError) as e:
        plan.execute(comm, x, y)
    assert e.value.name == "AXE_ERR_NCCL"
    st.synchronize()
    del comm
    comm2 = axe.Comm(axe.get_unique_id(), 1, 0, torch.cuda.current_device())
    x.copy_(torch.arange(R * Cn, dtype=torch.int32, device="cuda"))
    plan.execute(comm2, x, y)
    comm2.wait(None, timeout_ms=60000)
    assert torch.equal(y.view(Cn, R).t().reshape(-1), x)


def test_plan_executes_serialised_across_streams_and_threads(axe):
    """One redistribute plan (pack + NCCL + unpack through its own staging buffers) executed from two host
    threads on two streams at once: the plan serialises them (host lock + device event chain), every
    result is exact."""
    import threading
    comm = axe.Comm(axe.get_unique_id(), 1, 0, torch.cuda.current_device())
    R, Cn = 256, 192
    src = layout([(R, Cn), (Cn, 1)])
    dst = layout([(R, 1), (Cn, R)], [(1, 1, "gpuid")])     # transposed: pack and unpack kernels
    plan = axe.RedistPlan(src, linear_storage(R * Cn), dst, linear_storage(R * Cn), 4, 1, 0)
    ins = [torch.randint(-2**31, 2**31 - 1, (R * Cn,), dtype=torch.int32, device="cuda") for _ in range(2)]
    outs = [[torch.zeros_like(ins[0]) for _ in range(10)] for _ in range(2)]
    torch.cuda.synchronize()
    errors = []

    def work(i):
        try:
            st = torch.cuda.Stream()
            for j in range(10):
                plan.execute(comm, ins[i], outs[i][j], st)
            st.synchronize()
        except Exception as e:
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for i in range(2):
        exp = ins[i].view(R, Cn).t().reshape(-1)
        for o in outs[i]:
            assert torch.equal(o, exp)
    del comm
