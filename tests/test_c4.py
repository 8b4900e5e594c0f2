"""Configuration C4: generated replay batches (generator determinism and
well-formedness on the CPU oracle; CUDA == oracle on the GPU) and LPT
sharding."""
import numpy as np
import pytest

import _golden
import _oracle
from paper_2406_13881_b200._abi import LIB_PATH
from paper_2406_13881_b200.dataflow import run_replay

pytestmark = pytest.mark.skipif(not LIB_PATH.exists(), reason="libdfx.so not built")


def _cfg(n=400, **kw):
    from paper_2406_13881_b200.batch import C4Config
    return C4Config(n_funcs=n, n_min=32, n_max=400, **kw)


def test_generator_deterministic_and_shard_invariant():
    from paper_2406_13881_b200.batch import c4_generate
    cfg = _cfg()
    a, fa = c4_generate(cfg, np.arange(100))
    b, fb = c4_generate(cfg, np.arange(100))
    assert fa == fb and all(np.array_equal(getattr(a, k), getattr(b, k))
                            for k in ("fns", "ops", "var_flags", "stmt_span", "sites", "arms"))
    # function 57 alone == function 57 inside a batch (shards generate subsets)
    c, _ = c4_generate(cfg, np.array([57]))
    d = a.fns[57]
    assert np.array_equal(c.ops, a.ops[d["op_off"]:d["op_off"] + d["n_ops"]])


def test_generated_programs_run_clean_on_oracle():
    from paper_2406_13881_b200.batch import c4_generate
    b, facts = c4_generate(_cfg(), np.arange(120))
    raw = run_replay(b, runner=_oracle.replay_runner)
    assert not (raw.events["kind"] >= 16).any(), "generated programs must not hit errors"
    assert raw.events.shape[0] > 0 and facts > 0


def test_lpt_shards_partition_and_balance():
    from paper_2406_13881_b200.batch import C4Config, c4_cost, c4_shapes, lpt_shards
    N, V = c4_shapes(C4Config(n_funcs=20000))
    cost = c4_cost(N, V)
    for world in (1, 2, 4, 8):
        sh = lpt_shards(cost, world)
        allf = np.sort(np.concatenate(sh))
        assert np.array_equal(allf, np.arange(20000))
        loads = [cost[s].sum() for s in sh]
        assert max(loads) / min(loads) < 1.001


@pytest.mark.gpu
def test_cuda_replay_matches_oracle_on_c4_batch():
    from paper_2406_13881_b200.batch import ReplayBatch, c4_generate
    b, _ = c4_generate(_cfg(), np.arange(300))
    exp = run_replay(b, runner=_oracle.replay_runner)
    got = run_replay(b)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
    rb = ReplayBatch(b)
    n, ms = rb.run()
    res = rb.fetch()
    _golden.assert_raw_equal(res.events, res.var_out, exp.events, exp.var_out)


@pytest.mark.gpu
def test_cuda_replay_matches_oracle_at_bench_shapes():
    """Functions of the benchmark's own batch (64-2048 nodes, up to 512
    variables = 16 warps per function), through the pipelined batch call and
    the device-resident one.  Large functions nest branches and loops inside
    captured if-arms; warps skip regions none of their variables is accessed
    in (replay.cu region_kernel), and a skipped region that holds a branch must
    still end in a fresh slot so the enclosing arm stays frozen (D4)."""
    from paper_2406_13881_b200.batch import C4Config, ReplayBatch, c4_generate
    b, _ = c4_generate(C4Config(), np.arange(0, 100_000, 67))
    exp = run_replay(b, runner=_oracle.replay_runner_mt)
    got = run_replay(b)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
    rb = ReplayBatch(b)
    rb.run()
    res = rb.fetch()
    _golden.assert_raw_equal(res.events, res.var_out, exp.events, exp.var_out)


@pytest.mark.gpu
def test_host_buffer_call_with_uneven_event_density():
    """dfx_replay_batch gives each pipeline range an event region sized by its
    share of the ops.  Here the first 10% of the functions carry all the
    events (the rest only write on the host), and the caller's
    capacity is the exact total, so the early ranges overflow their regions
    and are replayed again into exact-size ones: the result must not change."""
    import dataclasses
    from paper_2406_13881_b200.batch import C4Config, c4_generate
    from paper_2406_13881_b200.dataflow import ReplaySession
    b, _ = c4_generate(C4Config(), np.arange(400))
    ops = b.ops.copy()
    start = int(b.fns[40]["op_off"])    # events only in the first 10% of the functions
    code = ops[start:, 0] & 0xFF
    acc = (code >= 1) & (code <= 4)
    ops[start:, 0][acc] = (ops[start:, 0][acc] & ~0xFF) | 2        # every access -> HW
    b2 = dataclasses.replace(b, ops=ops)
    exp = run_replay(b2, runner=_oracle.replay_runner_mt)
    assert not (exp.events["fn"] >= 40).any() and exp.events.shape[0] > 10_000
    got = ReplaySession(event_cap=int(exp.events.shape[0])).run(b2)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
    small = ReplaySession(event_cap=1000)                          # NOSPC -> regrow
    got = small.run(b2)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)


@pytest.mark.gpu
def test_cuda_replay_many_chunks_and_wide_slot_masks():
    """Functions with 2,048 variables (64 warps each: the region table's
    32-bit chunk masks alias chunk c and c + 32, which may only make a warp
    skip less) and, separately, a batch whose slot budget exceeds 32, which
    selects the 64-bit slot-mask kernel; both equal to the oracle."""
    from paper_2406_13881_b200.batch import C4Config, c4_generate
    b, _ = c4_generate(C4Config(n_funcs=40, n_min=64, n_max=600, var_choices=(2048,)),
                       np.arange(40))
    exp = run_replay(b, runner=_oracle.replay_runner_mt)
    got = run_replay(b)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
    b2, _ = c4_generate(_cfg(), np.arange(120))
    b2.fns["n_slots"][::7] = 48          # a larger budget than needed: same results
    exp = run_replay(b2, runner=_oracle.replay_runner_mt)
    got = run_replay(b2)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)


@pytest.mark.gpu
def test_gate_timeout_falls_back_to_the_ungated_replay(monkeypatch):
    """if a range's region kernel cannot get an SM slot beside
    the gated launch, the call replays the batch ungated instead of failing
    (forced here with a zero wait budget)."""
    from paper_2406_13881_b200.batch import C4Config, c4_generate
    from paper_2406_13881_b200.dataflow import run_replay
    b, _ = c4_generate(C4Config(), np.arange(600))
    exp = run_replay(b, runner=_oracle.replay_runner_mt)
    monkeypatch.setenv("DFX_GATE_TIMEOUT_MS", "0")
    got = run_replay(b)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
