"""CPU: the replay oracle against the reference's golden outputs.

The oracle (oracle/replay_oracle.c) is pinned here against (1) the committed
raw fixtures and (2) -- when the reference front end is importable -- the
reference `analyze_function` itself on fresh seeded programs.
"""
import numpy as np
import pytest

import _cases
import _golden
import _oracle
from paper_2406_13881_b200._host import have_dartomp
from paper_2406_13881_b200.dataflow import run_replay


def test_oracle_matches_golden_raw():
    batch, ev, vo = _golden.replay_fixture()
    raw = run_replay(batch, runner=_oracle.replay_runner)
    _golden.assert_raw_equal(raw.events, raw.var_out, ev, vo)


def test_golden_covers_semantics():
    """The fixture set exercises every event/position kind we claim parity on."""
    plans = _golden.reference_plans()
    seen = set()
    for case in plans.values():
        for res in case["functions"].values():
            if res[0] == "err":
                seen.add("err:" + res[1] + ":" + res[2].split(": error: ")[-1][:20])
                continue
            p = res[1]
            if p["region"]:
                seen.add("region")
            for u in p["updates"]:
                seen.add("upd:%s:%s" % (u[0], u[3]))
            for k in p["kernel_clauses"]:
                seen.add("kc:" + k[0])
            if p["suppressed"]:
                seen.add("suppressed")
    for need in ("region", "upd:update_from:before", "upd:update_from:after",
                 "upd:update_from:body_end", "upd:update_to:before",
                 "kc:firstprivate", "kc:map_to", "kc:map_from", "kc:map_tofrom",
                 "kc:map_alloc"):
        assert need in seen, need
    assert any(s.startswith("err:DeclPlacementError") for s in seen)
    assert any(s.startswith("err:PreconditionError:braces") for s in seen)
    assert any(s.startswith("err:PreconditionError:input already") for s in seen)


@pytest.mark.skipif(not have_dartomp(), reason="reference front end not importable")
@pytest.mark.parametrize("seed", list(range(1000, 1040)))
def test_oracle_vs_reference_random(seed):
    from dartomp.dataflow import analyze_function as ref_analyze
    from dartomp.pipeline import load
    from paper_2406_13881_b200.dataflow import analyze_functions
    a = load(path="gen%d.c" % seed, text=_cases.random_program(seed))
    names = list(a.cfgs)
    items = [(a.src, a.cfgs[n], a.accesses[n], a.table) for n in names]
    mine = analyze_functions(items, runner=_oracle.replay_runner)
    for n, d in zip(names, mine):
        ref = _cases.canon_result(lambda: ref_analyze(a.src, a.cfgs[n], a.accesses[n], a.table))
        got = _cases.canon_result(d.get)
        assert got == ref, n


def test_multithreaded_oracle_equals_sequential():
    """The benchmark's all-threads CPU baseline (oracle_replay_batch_mt)
    produces the sequential oracle's output exactly, event order included."""
    import numpy as np
    from paper_2406_13881_b200.batch import C4Config, c4_generate
    from paper_2406_13881_b200.dataflow import run_replay
    b, _ = c4_generate(C4Config(n_funcs=400, seed=3), np.arange(0, 400, 3, dtype=np.int32))
    seq = run_replay(b, runner=_oracle.replay_runner)
    mt = run_replay(b, runner=_oracle.replay_runner_mt)
    assert np.array_equal(seq.events, mt.events)
    assert np.array_equal(seq.var_out, mt.var_out)


def test_parallel_lowering_equals_serial():
    """Forked-worker lowering (dataflow.lower_functions) returns the serial
    lowering exactly: same arrays, and references mapped back to the
    caller's own AstNode / VariableId objects."""
    if not have_dartomp():
        pytest.skip("reference front end not importable")
    import dartomp.pipeline as rp
    from paper_2406_13881_b200.dataflow import lower_functions
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    from paper_2406_13881_b200.lower import lower_function
    a = rp.load(text=generate(11, GenConfig(n_funcs=70, n_stmts=12)))
    items = [(a.src, a.cfgs[n], a.accesses[n], a.table) for n in a.cfgs]
    par = lower_functions(items, workers=4)
    for (src, cfg, accs, table), p in zip(items, par):
        s = lower_function(src, cfg, accs, table)
        for k in ("ops", "var_flags", "stmt_span", "sites", "arms"):
            assert np.array_equal(getattr(p, k), getattr(s, k)), k
        assert (p.region_begin_start, p.n_slots, p.max_loop_depth, p.max_br_depth,
                p.max_arms) == (s.region_begin_start, s.n_slots, s.max_loop_depth,
                                s.max_br_depth, s.max_arms)
        assert p.fn is s.fn
        assert all(x is y for x, y in zip(p.stmts, s.stmts)) and len(p.stmts) == len(s.stmts)
        assert all(x is y for x, y in zip(p.vars, s.vars)) and len(p.vars) == len(s.vars)
        assert all(x is y for x, y in zip(p.kernel_stmts, s.kernel_stmts))
        assert p.premapped is s.premapped
        assert (p.region is None) == (s.region is None)
        if p.region is not None:
            assert all(x is y for x, y in zip(p.region, s.region))
