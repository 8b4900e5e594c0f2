"""GPU: the CUDA E1 replay engine (libdfx.so) against the parity fixtures and
against the reference analysis run in-process on fresh programs."""
import numpy as np
import pytest

import _cases
import _golden
import _oracle
from paper_2406_13881_b200._host import have_dartomp
from paper_2406_13881_b200.dataflow import pack, run_replay

pytestmark = pytest.mark.gpu


def test_cuda_replay_matches_golden_raw():
    batch, ev, vo = _golden.replay_fixture()
    raw = run_replay(batch)              # CUDA engine, no runner override
    _golden.assert_raw_equal(raw.events, raw.var_out, ev, vo)


def test_cuda_replay_tiny_event_capacity_retries():
    batch, ev, vo = _golden.replay_fixture()
    raw = run_replay(batch, event_cap=3)
    _golden.assert_raw_equal(raw.events, raw.var_out, ev, vo)


@pytest.mark.skipif(not have_dartomp(), reason="host front end (dartomp) not importable")
@pytest.mark.parametrize("seed", list(range(2000, 2060)))
def test_cuda_drop_in_vs_reference(seed):
    from dartomp.dataflow import analyze_function as ref_analyze
    from dartomp.pipeline import load
    from paper_2406_13881_b200.dataflow import analyze_functions
    a = load(path="gen%d.c" % seed, text=_cases.random_program(seed))
    names = list(a.cfgs)
    items = [(a.src, a.cfgs[n], a.accesses[n], a.table) for n in names]
    mine = analyze_functions(items)
    for n, d in zip(names, mine):
        ref = _cases.canon_result(lambda: ref_analyze(a.src, a.cfgs[n], a.accesses[n], a.table))
        got = _cases.canon_result(d.get)
        assert got == ref, n
        if ref[0] == "ok":
            assert _cases.identity_equal(d.get(), ref_analyze(a.src, a.cfgs[n], a.accesses[n], a.table))


@pytest.mark.skipif(not have_dartomp(), reason="host front end (dartomp) not importable")
def test_cuda_vs_oracle_large_batch():
    """A few hundred functions in one launch: CUDA raw == oracle raw."""
    from dartomp.pipeline import load
    from paper_2406_13881_b200.lower import lower_function
    progs = []
    for seed in range(3000, 3150):
        a = load(path="g.c", text=_cases.random_program(seed))
        for n in a.cfgs:
            progs.append(lower_function(a.src, a.cfgs[n], a.accesses[n], a.table))
    batch = pack(progs)
    got = run_replay(batch)
    exp = run_replay(batch, runner=_oracle.replay_runner)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
