"""GPU: kernel (c) across ranks, run by two processes that share one GPU:
the fused path (dfx_cgp_*: rebuilt summary rows stored into every rank's
tables over peer memory through CUDA IPC, system-scope arrival counters) and
the all-gather path (dfx_cg_wave + torch.distributed all-gather of the
rebuilt rows), against the CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import _oracle

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, seed, n, path="peer"):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import torch
        from paper_2406_13881_b200.distributed import PeerSummaries, ShardedSummaries
        from paper_2406_13881_b200.gen.c5 import generate_c5
        torch.cuda.set_device(0)
        g = generate_c5(seed=seed, n_funcs=n, depth=12, n_globals=64, p_back=0.25)
        ps = PeerSummaries(g, rank, world) if path == "peer" else \
            ShardedSummaries(g, rank, world, device="cuda:0")
        res = []
        for _ in range(2):                      # two solves: flags and counters carry over
            res.append(ps.solve())
            dist.barrier()
        ps.close()
        dist.destroy_process_group()
        q.put((rank, res, None))
    except Exception as e:                      # noqa: BLE001 -- report to the parent
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("seed,n,path", [(3, 480, "peer"), (8, 1200, "peer"),
                                         (3, 480, "allgather")])
def test_summaries_two_ranks_one_gpu(seed, n, path):
    from paper_2406_13881_b200.gen.c5 import generate_c5
    from paper_2406_13881_b200.interproc import solve_call_graph
    g = generate_c5(seed=seed, n_funcs=n, depth=12, n_globals=64, p_back=0.25)
    exp = solve_call_graph(g, runner=_oracle.summaries_runner)
    one = solve_call_graph(g)                   # single-GPU engine
    assert np.array_equal(one.bits, exp.bits)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, seed, n, path)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, res, err in got:
        assert err is None, (rank, err)
        for bits, lst, ln, passes in res:
            assert np.array_equal(bits, exp.bits), rank
            assert np.array_equal(ln, exp.len)
            for f in range(ln.shape[0]):
                assert np.array_equal(lst[f, :ln[f]], exp.list[f, :ln[f]])
            assert passes == exp.passes
