"""Multi-rank host logic on CPU (gloo, world size 2): the kernel-(c) summary
exchange protocol, C3 variable sharding and C4 function sharding reproduce
the single-rank results exactly."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import _oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _summaries_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import _cg_cpu
    from paper_2406_13881_b200.distributed import ShardedSummaries
    from paper_2406_13881_b200.gen.c5 import generate_c5
    _init(rank, world, port)
    g = generate_c5(seed=3, n_funcs=480, depth=12, n_globals=64, p_back=0.25)
    st = ShardedSummaries(g, rank, world, device="cpu", wave_impl=lambda *a: 0)
    st.wave_impl = _cg_cpu.make_cpu_wave(st)
    bits, lst, ln, passes = st.solve()
    q.put((rank, bits, lst, ln, passes))
    dist.destroy_process_group()


def test_sharded_summaries_gloo_world2_equals_oracle():
    from paper_2406_13881_b200.gen.c5 import generate_c5
    from paper_2406_13881_b200.interproc import solve_call_graph
    g = generate_c5(seed=3, n_funcs=480, depth=12, n_globals=64, p_back=0.25)
    exp = solve_call_graph(g, runner=_oracle.summaries_runner)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_summaries_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, bits, lst, ln, passes in res:
        assert np.array_equal(bits, exp.bits), rank
        assert np.array_equal(ln, exp.len)
        for f in range(ln.shape[0]):
            assert np.array_equal(lst[f, :ln[f]], exp.list[f, :ln[f]])
        assert passes == exp.passes


def _c3_worker(rank, world, port, q):
    import torch
    _init(rank, world, port)
    words = 4                                    # per-rank slab
    g = _oracle.c3_generate(5, 4096, rank * words, words, 82)
    oh, od, _ = _oracle.c3_solve(g)
    t = torch.from_numpy(np.concatenate([oh, od], axis=1).astype(np.int64))
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)                      # result assembly only (no data-path collective)
    if rank == 0:
        q.put([o.numpy() for o in out])
    dist.destroy_process_group()


def test_c3_variable_sharding_gloo_world2_equals_single():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c3_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    full = _oracle.c3_generate(5, 4096, 0, 8, 82)
    oh, od, _ = _oracle.c3_solve(full)
    assert np.array_equal(np.concatenate([parts[0][:, :4], parts[1][:, :4]], axis=1), oh)
    assert np.array_equal(np.concatenate([parts[0][:, 4:], parts[1][:, 4:]], axis=1), od)


def _c4_worker(rank, world, port, q):
    from paper_2406_13881_b200.batch import C4Config, c4_cost, c4_generate, c4_shapes, lpt_shards
    from paper_2406_13881_b200.dataflow import run_replay
    _init(rank, world, port)
    cfg = C4Config(n_funcs=64, n_min=32, n_max=200)
    N, V = c4_shapes(cfg)
    mine = lpt_shards(c4_cost(N, V), world)[rank]
    b, facts = c4_generate(cfg, mine)
    raw = run_replay(b, runner=_oracle.replay_runner)
    ev = raw.events.copy()
    ev["fn"] = mine[ev["fn"]]                   # shard-local -> global function ids
    obj = [None] * world
    dist.all_gather_object(obj, (ev.tobytes(), facts))
    if rank == 0:
        q.put(obj)
    dist.destroy_process_group()


@pytest.mark.skipif(not __import__("paper_2406_13881_b200._abi", fromlist=["x"]).LIB_PATH.exists(),
                    reason="libdfx.so not built (generator)")
def test_c4_function_sharding_gloo_world2_equals_single():
    from paper_2406_13881_b200 import _abi
    from paper_2406_13881_b200.batch import C4Config, c4_generate
    from paper_2406_13881_b200.dataflow import run_replay
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c4_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    cfg = C4Config(n_funcs=64, n_min=32, n_max=200)
    b, facts = c4_generate(cfg, np.arange(64, dtype=np.int32))
    exp = run_replay(b, runner=_oracle.replay_runner).events
    got = np.concatenate([np.frombuffer(p[0], dtype=_abi.EVENT_DTYPE) for p in parts])
    key = lambda e: e[np.lexsort((e["key"], e["fn"]))]  # noqa: E731
    assert np.array_equal(key(got), key(exp))
    assert sum(p[1] for p in parts) == facts
