"""Kernel (c): interprocedural summaries (sets and dict insertion orders)
against the reference `summarize_all`."""
import pytest

import _golden
import _oracle
from paper_2406_13881_b200._host import have_dartomp
from paper_2406_13881_b200.interproc import solve_call_graph

CASES = _golden.summary_fixtures()


@pytest.mark.parametrize("idx", range(len(CASES)), ids=[c[0] for c in CASES])
def test_oracle_matches_golden(idx):
    name, g, exp = CASES[idx]
    _golden.assert_summary_equal(solve_call_graph(g, runner=_oracle.summaries_runner), exp)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(len(CASES)), ids=[c[0] for c in CASES])
def test_cuda_matches_golden(idx):
    name, g, exp = CASES[idx]
    _golden.assert_summary_equal(solve_call_graph(g), exp)


def _compare_with_reference(seed, n_funcs, runner):
    from dartomp.interproc import summarize_all as ref_sum
    from dartomp.pipeline import load
    from paper_2406_13881_b200.gen.callgraph import CallGraphConfig, generate
    from paper_2406_13881_b200.interproc import summarize_all
    a = load(path="cg.c", text=generate(seed, CallGraphConfig(n_funcs=n_funcs, depth=12)))
    ref = ref_sum(a.src, a.tu, a.cfgs, a.raw_accesses, a.table)
    mine = summarize_all(a.src, a.tu, a.cfgs, a.raw_accesses, a.table, runner=runner)
    assert list(ref) == list(mine)
    for k in ref:
        assert ref[k].snapshot() == mine[k].snapshot(), k
        assert list(ref[k].param_effects.items()) == list(mine[k].param_effects.items()), k
        assert list(ref[k].global_effects.items()) == list(mine[k].global_effects.items()), k


@pytest.mark.skipif(not have_dartomp(), reason="host front end not importable")
@pytest.mark.parametrize("seed", [100, 101])
def test_oracle_vs_reference_fresh_callgraph(seed):
    _compare_with_reference(seed, 120, _oracle.summaries_runner)


@pytest.mark.gpu
@pytest.mark.skipif(not have_dartomp(), reason="host front end not importable")
@pytest.mark.parametrize("seed", [200, 201, 202])
def test_cuda_vs_reference_fresh_callgraph(seed):
    _compare_with_reference(seed, 240, None)


@pytest.mark.gpu
def test_cuda_sharded_driver_world1_and_c5_scale():
    """The multi-GPU driver path (dfx_cg_create/dfx_cg_wave on torch-owned
    tables) at world size 1, on a 10k-function C5 graph."""
    import numpy as np
    from paper_2406_13881_b200.distributed import ShardedSummaries
    from paper_2406_13881_b200.gen.c5 import generate_c5
    g = generate_c5(seed=1)
    exp = solve_call_graph(g, runner=_oracle.summaries_runner)
    bits, lst, ln, passes = ShardedSummaries(g, 0, 1, device="cuda").solve()
    assert passes == exp.passes and np.array_equal(bits, exp.bits) and np.array_equal(ln, exp.len)
    for f in range(ln.shape[0]):
        assert np.array_equal(lst[f, :ln[f]], exp.list[f, :ln[f]])
    r = solve_call_graph(g)          # single-call path
    _golden.assert_summary_equal(r, (exp.bits, exp.list, exp.len, exp.passes))
