"""Batched emission: the native emitter (csrc/emit.cpp) is
byte-identical to the reference's `rewriter.apply_plans` and
`report.plan_lines`, errors included.  Host code only (no GPU): plans come
from the reference's own `plan_transform`, so these run on CPU."""
import pathlib
import random

import pytest

from paper_2406_13881_b200._host import have_dartomp

pytestmark = pytest.mark.skipif(not have_dartomp(), reason="host front end not importable")

GOLD = pathlib.Path(__file__).parent / "golden"


def _outcome(fn):
    try:
        return fn()
    except Exception as e:      # noqa: BLE001 -- compared with the reference's exception
        return (type(e).__name__, str(e))


def _units():
    from dartomp.pipeline import load, plan_transform
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    sources = [(str(p), p.read_text()) for p in sorted(GOLD.rglob("*.c"))]
    for seed in range(40):
        r = random.Random(seed)
        sources.append(("g%d.c" % seed, generate(seed, GenConfig(n_funcs=r.randrange(0, 4),
                                                                 n_stmts=r.randrange(10, 40)))))
    for seed in (1, 2):   # large units: the reference rewriter's InternalError path
        sources.append(("big%d.c" % seed, generate(seed, GenConfig(n_funcs=30, n_globals=24,
                                                                   n_stmts=40, p_kernel=0.3))))
    for name, text in sources:
        try:
            a = load(path=name, text=text)
            plans = plan_transform(a)
        except Exception:      # noqa: BLE001 -- analysis errors: nothing to emit
            continue
        yield name, a.src, plans


def test_native_emitter_matches_reference():
    from dartomp.report import plan_lines
    from dartomp.rewriter import apply_plans
    from paper_2406_13881_b200 import emit
    n = errs = after = 0
    for name, src, plans in _units():
        ref = _outcome(lambda: apply_plans(src, plans))
        got = _outcome(lambda: emit.apply_plans(src, plans))
        if isinstance(ref, tuple):
            assert got == ref, name
            errs += 1
        else:
            assert got.text == ref.text and got.placed == ref.placed, name
            assert got.splice_out() == src.text
        rl = _outcome(lambda: plan_lines(src, plans))
        gl = _outcome(lambda: emit.plan_lines(src, plans))
        assert gl == rl, name
        after += isinstance(rl, tuple) and rl[0] == "KeyError"
        n += 1
    assert n >= 60 and errs >= 1 and after >= 1, (n, errs, after)


def test_native_emitter_batch_equals_per_unit_and_after_lines():
    from dartomp.dataflow import AFTER
    from paper_2406_13881_b200 import emit
    units = list(_units())
    batch = emit.emit_batch([(s, p, None) for _, s, p in units], on_after="line")
    for (name, src, plans), (res, lines) in zip(units, batch):
        one = _outcome(lambda: emit.apply_plans(src, plans))
        if isinstance(one, tuple):
            assert (type(res).__name__, str(res)) == one, name
        else:
            assert res.text == one.text, name
        ups = [u for p in plans for u in p.updates if u.position == AFTER]
        if ups:                # the reference raises KeyError here; "line" reports them
            assert any("\tafter line " in ln for ln in lines), name


def test_native_emitter_non_ascii_offsets_and_indent_unit():
    """Offsets are string indices (UTF-32 inside), not bytes."""
    from dartomp.pipeline import load, plan_transform
    from dartomp.rewriter import apply_plans
    from paper_2406_13881_b200 import emit
    text = (GOLD / "corpus" / "transform" / "listing1.c").read_text()
    text = "/* déjà vu — über */\n" + text
    a = load(path="u.c", text=text)
    plans = plan_transform(a)
    for unit in (None, "\t", "  "):
        assert emit.apply_plans(a.src, plans, unit).text == apply_plans(a.src, plans, unit).text
