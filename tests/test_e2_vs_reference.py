"""Kernel (a)'s equations pinned to the reference itself: on
monotone-subset programs (loops, no branches, no update hoisted in front of a
loop) the fixpoint of the syntax-directed CSR equals the reference
analyzer's (H, D) at every planning visit, for every variable."""
import numpy as np
import pytest

import _oracle
from paper_2406_13881_b200._host import have_dartomp

pytestmark = pytest.mark.skipif(not have_dartomp(), reason="host front end not importable")

MONO = dict(n_funcs=0, p_if=0.0, p_switch=0.0, p_jump=0.0, p_call=0.0, p_fp_clause=0.0,
            p_late_decl=0.0, p_braceless=0.0, p_loop=0.35, max_loop_depth=3, max_depth=4)


def _cases(seeds):
    import random
    from dartomp.nodes import LOOP_KINDS
    from dartomp.pipeline import load
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    import _syntax_graph as sg
    for seed in seeds:
        r = random.Random(seed)
        cfg = GenConfig(n_stmts=r.randrange(6, 22), **MONO)
        a = load(path="m%d.c" % seed, text=generate(seed, cfg))
        args = (a.src, a.cfgs["main"], a.accesses["main"], a.table)
        try:
            graph = sg.build_graph(*args)
        except sg.Unsupported:
            continue
        ref, plan = sg.reference_states(*args, graph[-1])
        if any(u.anchor.kind in LOOP_KINDS for u in plan.updates):
            continue               # D3: an update hoisted in front of a loop
        yield seed, graph, ref


def _check(graph, ref, solver):
    import _syntax_graph as sg
    row_ptr, col, kind, R, W, S, vars_ = graph
    assert row_ptr.shape[0] - 1 == len(ref), "one node per planning visit"
    OH, OD = solver(row_ptr, col, kind, R, W, S)
    got = sg.in_states(row_ptr, col, OH, OD, len(vars_))
    for i, ((gh, gd), (rh, rd)) in enumerate(zip(got, ref)):
        assert np.array_equal(gh, rh) and np.array_equal(gd, rd), "visit %d" % i
    return len(ref) * len(vars_)


def _oracle_solver(row_ptr, col, kind, R, W, S):
    g = {"row_ptr": row_ptr, "col": col, "kind": kind, "A": R | W, "B": W, "S": S}
    OH, OD, _ = _oracle.c3_solve(g)
    return OH, OD


def test_mfp_oracle_equals_reference_on_monotone_programs():
    facts, n = 0, 0
    for seed, graph, ref in _cases(range(150)):
        facts += _check(graph, ref, _oracle_solver)
        n += 1
    assert n >= 60 and facts > 40_000, (n, facts)


@pytest.mark.gpu
def test_cuda_mfp_equals_reference_on_monotone_programs():
    from paper_2406_13881_b200.csr import CsrProblem

    def cuda_solver(row_ptr, col, kind, R, W, S):
        p = CsrProblem.from_arrays(row_ptr, col, kind, R, W, S)
        p.solve(8)
        OH, OD, _ = p.download(True, True)
        return OH, OD
    n = 0
    for seed, graph, ref in _cases(range(150, 230)):
        _check(graph, ref, cuda_solver)
        n += 1
    assert n >= 30
