"""The one-sided redistribution across PROCESSES ("distributed copy"): two ranks,
each its own process (one GPU is all a pool box has, so both map cuda:0), exchange their destination
(or source) buffers as CUDA IPC handles (axe_ipc_export / axe_ipc_import, the pointer path NVLink peer
stores take on a multi-GPU node), and every rank's copy kernels write straight into the other
process's memory.  Each rank checks its own buffer against the oracle.  The kernels of the two ranks
never wait on one another (host barriers over gloo order the phases)."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from synth import layout, linear_storage

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _cases():
    R, Cn = 256, 192
    rows_to_cols = dict(name="rows_to_cols", es=2, nranks=2,
                        src=layout([(2, 1, "gpuid"), (R // 2, Cn), (Cn, 1)]), src_st=linear_storage(R // 2 * Cn),
                        dst=layout([(R, Cn // 2), (2, 1, "gpuid"), (Cn // 2, 1)]), dst_st=linear_storage(R * Cn // 2),
                        seed=71)
    return {"config4_p2": lambda: synth.config4(2, 512), "rows_to_cols": lambda: rows_to_cols}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2601_19092_b200 as axe
        if case == "reduce_scatter_pull":
            cfg = synth.reduce_scatter(world, 128, 256, "f32")
            es, dtype = 4, "f32"
        else:
            cfg = _cases()[case]()
            es, dtype = cfg["es"], None
        n = cfg["nranks"]
        assert n == world
        ed, _ = oracle.sizes(cfg["src"])
        v = synth.numbers(ed, dtype, 72, "narrow") if dtype else synth.values(ed, es, cfg["seed"])
        sfill = synth.sentinel(synth.storage_cells(cfg["src_st"]) * es, 73)
        src = oracle.scatter_ranks(cfg["src"], cfg["src_st"], v, es, n, sfill)
        dfill = synth.sentinel(synth.storage_cells(cfg["dst_st"]) * es, 74)
        exp = [dfill.copy() for _ in range(n)]
        if dtype:
            oracle.reduce(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, dtype, nranks=n)
            plan = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, n, rank,
                                  reduce_dtype=dtype)
        else:
            oracle.redistribute(cfg["src"], cfg["src_st"], src, cfg["dst"], cfg["dst_st"], exp, es)
            plan = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], es, n, rank)
        s_dev = torch.from_numpy(src[rank]).cuda()
        d_dev = torch.from_numpy(dfill.copy()).cuda()
        shared = s_dev if dtype else d_dev          # the buffer the OTHER rank touches
        hs = [None] * world
        dist.all_gather_object(hs, axe.ipc_export(shared[64:] if rank == 1 and not dtype else shared))
        peers = []
        for r in range(world):
            if r == rank:
                peers.append(shared.data_ptr())
            else:
                p = axe.ipc_import(hs[r])
                if r == 1 and not dtype:
                    p -= 64 * shared.element_size()   # rank 1 exported an interior pointer: offset carried
                peers.append(p)
        torch.cuda.synchronize()
        dist.barrier()
        if dtype:
            plan.execute_peers_reduce(peers, d_dev)
        else:
            plan.execute_peers(s_dev, peers)
        torch.cuda.synchronize()
        dist.barrier()            # every rank's kernels into my buffer are done
        ok = np.array_equal(d_dev.cpu().numpy(), exp[rank])
        for r in range(world):
            if r != rank:
                axe.ipc_close(peers[r] + (64 * shared.element_size() if r == 1 and not dtype else 0))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, plan.describe().get("pattern")))
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, False, traceback.format_exc()[-2000:]))


@pytest.mark.parametrize("case", ["config4_p2", "rows_to_cols", "reduce_scatter_pull"])
def test_one_sided_across_processes(case):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(60)
    assert all(ok for _, ok, _ in res), res
