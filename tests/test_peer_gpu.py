"""GPU: the fused multi-GPU kernel-(c) path (dfx_cgp_*: rebuilt summary rows
stored into every rank's tables over peer memory, system-scope arrival
counters) run by two processes that share one GPU through CUDA IPC, against
the CPU oracle and the single-GPU engine."""
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


def _worker(rank, world, port, q, seed, n):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2406_13881_b200.distributed import PeerSummaries
        from paper_2406_13881_b200.gen.c5 import generate_c5
        g = generate_c5(seed=seed, n_funcs=n, depth=12, n_globals=64, p_back=0.25)
        ps = PeerSummaries(g, rank, world)
        res = []
        for _ in range(2):                      # two solves: flags and counters carry over
            res.append(ps.solve())
            dist.barrier()
        ps.close()
        dist.destroy_process_group()
        q.put((rank, res, None))
    except Exception as e:                      # noqa: BLE001 -- report to the parent
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("seed,n", [(3, 480), (8, 1200)])
def test_peer_fused_summaries_two_ranks_one_gpu(seed, n):
    from paper_2406_13881_b200.gen.c5 import generate_c5
    from paper_2406_13881_b200.interproc import solve_call_graph
    g = generate_c5(seed=seed, n_funcs=n, depth=12, n_globals=64, p_back=0.25)
    exp = solve_call_graph(g, runner=_oracle.summaries_runner)
    one = solve_call_graph(g)                   # single-GPU engine
    assert np.array_equal(one.bits, exp.bits)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, seed, n)) for r in range(2)]
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
