"""Functions beyond the narrow replay's limits (one such function
used to fail the whole batch with DFX_E_LIMIT).  They now run in the wide
replay (replay.cu Wide: 256 slots, 32-bit provenance ids, deep stacks) in the
same call, and a function beyond even those limits fails alone with an
EngineError while the rest of the batch is analysed.  The reference handles
every input here; the drop-in must match it byte for byte."""
import numpy as np
import pytest

import _e2e
import _golden
import _oracle
from paper_2406_13881_b200 import _abi
from paper_2406_13881_b200._host import have_dartomp
from paper_2406_13881_b200._abi import LIB_PATH

pytestmark = pytest.mark.skipif(not have_dartomp(), reason="host front end absent")
CPU = {"replay_runner": _oracle.replay_runner, "summary_runner": _oracle.summaries_runner}


def elseif_chain(n: int) -> str:
    """An else-if chain of n branches, a kernel and a host write per arm:
    the lowering needs ~5 state slots per level (13 branches > 64 slots)."""
    L = ["double a[64];", "double b[64];", "double s;", "int main(int argc) {", "  int k = argc;",
         "  #pragma omp target teams distribute parallel for",
         "  for (int i = 0; i < 64; ++i) { a[i] = b[i] + 1.0; }"]
    for j in range(n):
        L.append("  %sif (k == %d) {" % ("" if j == 0 else "} else ", j))
        L.append("    #pragma omp target teams distribute parallel for")
        L.append("    for (int i = 0; i < 64; ++i) { a[i] = a[i] * %d.0; }" % j)
        L.append("    b[%d] = a[%d];" % (j % 64, j % 64))
    L += ["  } else {", "    s = a[1];", "  }", "  s = a[0] + b[0];", "  return 0;", "}"]
    return "\n".join(L) + "\n"


def nested_ifs(n: int) -> str:
    """n nested ifs, each with a kernel: branch depth n (> 48 is wide)."""
    L = ["double a[64];", "double b[64];", "int main(int argc) {", "  int k = argc;"]
    for j in range(n):
        L.append("  " * (j + 1) + "if (k > %d) {" % j)
        L.append("  " * (j + 2) + "#pragma omp target teams distribute parallel for")
        L.append("  " * (j + 2) + "for (int i = 0; i < 64; ++i) { a[i] = a[i] + %d.0; }" % j)
    for j in reversed(range(n)):
        L.append("  " * (j + 2) + "b[0] = a[%d];" % (j % 64))
        L.append("  " * (j + 1) + "}")
    L += ["  return 0;", "}"]
    return "\n".join(L) + "\n"


def _lowered(text):
    from dartomp.pipeline import load
    from paper_2406_13881_b200.lower import lower_function
    a = load(text=text)
    c = a.cfgs["main"]
    return lower_function(a.src, c, a.accesses["main"], a.table)


def test_programs_exceed_narrow_limits():
    p = _lowered(elseif_chain(13))
    assert p.n_slots > 64
    p = _lowered(nested_ifs(60))
    assert p.max_br_depth > 48 and p.n_slots > 64


@pytest.mark.parametrize("n", [13, 20, 40])
def test_elseif_chain_cpu_oracle(n):
    _e2e.compare(elseif_chain(n), "elseif%d.c" % n, **CPU)


@pytest.mark.gpu
@pytest.mark.skipif(not LIB_PATH.exists(), reason="libdfx.so not built")
@pytest.mark.parametrize("n", [12, 13, 20, 40])
def test_elseif_chain_cuda(n):
    _e2e.compare(elseif_chain(n), "elseif%d.c" % n)


@pytest.mark.gpu
@pytest.mark.skipif(not LIB_PATH.exists(), reason="libdfx.so not built")
@pytest.mark.parametrize("n", [49, 60])
def test_deep_nested_ifs_cuda(n):
    _e2e.compare(nested_ifs(n), "nested%d.c" % n)


def _mixed_batch():
    """Corpus/probe fixture functions with two wide programs spliced in."""
    from paper_2406_13881_b200.dataflow import pack
    from dartomp.pipeline import load
    from paper_2406_13881_b200.lower import lower_function
    progs = []
    for text in (elseif_chain(5), elseif_chain(20), nested_ifs(10), nested_ifs(55), elseif_chain(3)):
        a = load(text=text)
        progs.append(lower_function(a.src, a.cfgs["main"], a.accesses["main"], a.table))
    return pack(progs)


@pytest.mark.gpu
@pytest.mark.skipif(not LIB_PATH.exists(), reason="libdfx.so not built")
def test_mixed_narrow_and_wide_batch_raw_equal_oracle():
    """Both launches of one call (dfx_replay_batch and the device-resident
    dfx_replay_create/run) == the oracle, event for event."""
    from paper_2406_13881_b200.batch import ReplayBatch
    from paper_2406_13881_b200.dataflow import run_replay
    b = _mixed_batch()
    assert (b.fns["n_slots"] > 64).sum() == 2
    exp = run_replay(b, runner=_oracle.replay_runner)
    got = run_replay(b)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
    rb = ReplayBatch(b)
    rb.run()
    res = rb.fetch()
    _golden.assert_raw_equal(res.events, res.var_out, exp.events, exp.var_out)


@pytest.mark.gpu
@pytest.mark.skipif(not LIB_PATH.exists(), reason="libdfx.so not built")
def test_wide_provenance_over_65534_statements():
    """A generated function of more than 65,535 statements (32-bit
    provenance ids in the wide replay) among normal ones == the oracle."""
    from paper_2406_13881_b200.batch import C4Config, c4_generate
    from paper_2406_13881_b200.dataflow import run_replay
    b, _ = c4_generate(C4Config(n_funcs=8, n_min=70_000, n_max=90_000, var_choices=(64,)),
                       np.arange(2))
    b2, _ = c4_generate(C4Config(n_funcs=64), np.arange(30))
    assert (b.fns["n_stmts"] >= 0xFFFF).all()
    from paper_2406_13881_b200.dataflow import concat_batches
    cat = concat_batches([b2, b, b2])
    exp = run_replay(cat, runner=_oracle.replay_runner_mt)
    got = run_replay(cat)
    _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)


@pytest.mark.gpu
@pytest.mark.skipif(not LIB_PATH.exists(), reason="libdfx.so not built")
def test_beyond_wide_limits_fails_alone():
    """A function whose slot budget exceeds even the wide replay gets one
    engine-error event; every other function of the batch is unaffected."""
    from paper_2406_13881_b200.dataflow import run_replay
    b = _mixed_batch()
    exp = run_replay(b, runner=_oracle.replay_runner)
    b.fns["n_slots"][1] = 300
    got = run_replay(b)
    bad = got.events[got.events["fn"] == 1]
    assert bad.shape[0] == 1 and int(bad["kind"][0]) == _abi.EV_ERR_ENGINE
    keep_g = got.events[got.events["fn"] != 1]
    keep_e = exp.events[exp.events["fn"] != 1]
    v0, v1 = int(b.fns["var_off"][1]), int(b.fns["var_off"][1] + b.fns["n_vars"][1])
    mask = np.ones(exp.var_out.shape[0], dtype=bool)
    mask[v0:v1] = False
    _golden.assert_raw_equal(keep_g, got.var_out[mask], keep_e, exp.var_out[mask])
