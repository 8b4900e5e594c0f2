"""Transfer simulator: lowering + CPU oracle pinned to the
reference `simulate` record for record, and the CUDA simulator checked
against both (totals, aggregated stale reads, warnings, final ref counts)."""
import pathlib

import pytest

from paper_2406_13881_b200._host import have_dartomp

pytestmark = pytest.mark.skipif(not have_dartomp(), reason="host front end not importable")

GOLD = pathlib.Path(__file__).parent / "golden"


def _corpus_cases():
    from dartomp.pipeline import load, program_model, transform
    from dartomp.simulator import SimConfig
    files = sorted((GOLD / "corpus").rglob("*.c")) + sorted((GOLD / "sim").rglob("*.c"))
    for p in files:
        try:
            a = load(path=str(p))
        except Exception:      # noqa: BLE001 -- refused by the front end
            continue
        for trip in (1, 3):
            yield "%s/implicit/%d" % (p.name, trip), program_model(a), SimConfig(mode="implicit", default_trip=trip)
            yield "%s/annotated/%d" % (p.name, trip), program_model(a), SimConfig(mode="annotated", default_trip=trip)
        try:
            res, _ = transform(a)
            t = load(path=str(p) + " (transformed)", text=res.text)
        except Exception:      # noqa: BLE001 -- already annotated / analysis errors
            continue
        yield "%s/transformed" % p.name, program_model(t), SimConfig(mode="annotated")


def _generated(lo, hi, **kw):
    import _sim
    return _sim.sim_cases(range(lo, hi), **kw)


def _check_oracle(cases):
    import _sim
    from dartomp.simulator import simulate
    from paper_2406_13881_b200.simlower import lower_program
    n = 0
    for name, model, cfg in cases:
        ref = simulate(model, cfg)
        got = _sim.oracle_report(lower_program(model, cfg))
        assert _sim.exact_fields(got) == _sim.exact_fields(ref), name
        n += 1
    return n


def test_sim_oracle_matches_reference_on_corpus():
    assert _check_oracle(_corpus_cases()) >= 90


def test_sim_oracle_matches_reference_on_generated_programs():
    n = _check_oracle(_generated(0, 60))
    n += _check_oracle(_generated(1000, 1040, p_jump=0.08, p_call=0.15))
    assert n >= 100


def test_sim_lowering_records_control_warnings():
    from dartomp.pipeline import load, program_model
    from dartomp.simulator import SimConfig
    from paper_2406_13881_b200.simlower import lower_program
    text = ("double a[8];\nvoid f(double *p) { f(p); }\n"
            "int main() {\n#pragma omp target update to(zz)\n  f(a);\n  return 0;\n}\n")
    a = load(path="w.c", text=text)
    prog = lower_program(program_model(a), SimConfig(max_call_depth=2))
    texts = [prog.warnings[k] for k in prog.static_warnings]
    assert any("unknown variable 'zz'" in t for t in texts)
    assert any("call depth limit" in t for t in texts)


# ---------------------------------------------------------------------------
# CUDA
# ---------------------------------------------------------------------------
def _check_cuda(cases):
    import _sim
    from dartomp.simulator import simulate
    from paper_2406_13881_b200.simlower import lower_program
    from paper_2406_13881_b200.simulator import simulate_batch
    cases = list(cases)
    got = simulate_batch([(m, c) for _, m, c in cases])
    for (name, model, cfg), g in zip(cases, got):
        ref = simulate(model, cfg)
        orc = _sim.oracle_report(lower_program(model, cfg))
        assert _sim.aggregate_fields(g) == _sim.aggregate_fields(orc) == _sim.aggregate_fields(ref), name
    return len(cases)


@pytest.mark.gpu
def test_cuda_sim_matches_reference_on_corpus():
    assert _check_cuda(_corpus_cases()) >= 90


@pytest.mark.gpu
def test_cuda_sim_matches_reference_on_generated_programs():
    n = _check_cuda(_generated(0, 80))
    n += _check_cuda(_generated(1000, 1060, p_jump=0.08, p_call=0.15))
    n += _check_cuda(_generated(2000, 2030, n_stmts=(30, 70), max_loop_depth=3))
    assert n >= 150


@pytest.mark.gpu
def test_cuda_sim_simulation_and_comparison_lines():
    """`report.simulation_lines` (non-verbose) and `comparison_lines` of the
    CUDA `compare` equal the reference's, byte for byte, on stale-free
    transformed corpus programs."""
    from dartomp.pipeline import compare as ref_compare
    from dartomp.pipeline import load
    from dartomp.report import comparison_lines, simulation_lines
    from dartomp.simulator import SimConfig
    from paper_2406_13881_b200.simulator import compare
    n = 0
    for p in sorted((GOLD / "corpus" / "transform").glob("*.c")):
        a = load(path=str(p))
        try:
            rb, rm, rr = ref_compare(a, SimConfig())
        except Exception:      # noqa: BLE001
            continue
        gb, gm, gr = compare(load(path=str(p)), SimConfig())
        assert gr.text == rr.text
        assert comparison_lines(gb, gm) == comparison_lines(rb, rm), p.name
        head = lambda rep: simulation_lines(rep)[:5]  # noqa: E731
        assert head(gb) == head(rb) and head(gm) == head(rm), p.name
        if rm.log.stale_count == 0:
            assert simulation_lines(gm) == simulation_lines(rm), p.name
        n += 1
    assert n >= 15


@pytest.mark.gpu
def test_cuda_sim_no_settle_cap():
    """A loop whose state never repeats runs 10000 concrete rounds and the
    rest is extrapolated (simulator.py:543-548), with the warning."""
    from dartomp.pipeline import load, program_model
    from dartomp.simulator import SimConfig, simulate
    from paper_2406_13881_b200.simulator import simulate as cuda_simulate
    import _sim
    a = load(path=str(GOLD / "sim" / "nosettle.c"))
    for mode in ("annotated", "implicit"):
        cfg = SimConfig(mode=mode)
        ref = simulate(program_model(a), cfg)
        got = cuda_simulate(program_model(a), cfg)
        assert _sim.aggregate_fields(got) == _sim.aggregate_fields(ref)
    assert any("did not settle" in w for w in got.warnings) or mode == "implicit"
