"""The drop-in's parser (`frontend.ClimbingParser`, precedence climbing over
the six binary levels) builds the reference parser's tree node for node and
raises the reference's errors, on the corpus, the error corpus, generated
units of every shape the benches use, and operator soup (`pipeline.load`
parses with it; tests/test_pipeline.py runs that end to end)."""
import pathlib
import random

import pytest

from paper_2406_13881_b200._host import have_dartomp

pytestmark = pytest.mark.skipif(not have_dartomp(), reason="host front end absent")
CORPUS = pathlib.Path(__file__).parent / "golden" / "corpus"


def _flat(tu):
    """Pre-order nodes and their index, for identity-free comparison."""
    order, stack = [], [tu]
    while stack:
        n = stack.pop()
        order.append(n)
        stack.extend(reversed(n.children))
    return order, {id(n): i for i, n in enumerate(order)}


def _same_tree(a, b):
    oa, ia = _flat(a)
    ob, ib = _flat(b)
    assert len(oa) == len(ob)
    for x, y in zip(oa, ob):
        assert (x.kind, x.span, x.name, x.op, x.value, x.type_info, x.unresolved_global,
                x.postfix, x.omp, len(x.children)) == \
               (y.kind, y.span, y.name, y.op, y.value, y.type_info, y.unresolved_global,
                y.postfix, y.omp, len(y.children))
        for fa, fb in ((x.decl, y.decl), (x.parent, y.parent)):
            assert (fa is None) == (fb is None)
            if fa is not None:
                assert ia.get(id(fa), "outside") == ib.get(id(fb), "outside")
                if id(fa) not in ia:    # declarations outside the tree: same object kind/span
                    assert (fa.kind, fa.span) == (fb.kind, fb.span)


def _both(text):
    from dartomp.lexer import expand_defines
    from dartomp.parser import parse as ref_parse
    from dartomp.source import SourceFile
    from paper_2406_13881_b200.frontend import parse
    src = SourceFile.from_text(text)
    out = []
    for fn in (ref_parse, parse):
        try:
            tu, warns = fn(src, expand_defines(src))
            out.append(("ok", tu, [str(w) for w in warns]))
        except Exception as e:          # the reference's error, same type and text
            out.append(("err", type(e).__name__, str(e)))
    return out


def _check(text):
    r, e = _both(text)
    assert r[0] == e[0]
    if r[0] == "ok":
        _same_tree(r[1], e[1])
        assert r[2] == e[2]
    else:
        assert r[1:] == e[1:]


@pytest.mark.parametrize("path", sorted(str(p) for p in CORPUS.rglob("*.c")),
                         ids=lambda p: pathlib.Path(p).name)
def test_corpus(path):
    _check(pathlib.Path(path).read_text())


def test_generated_units():
    from paper_2406_13881_b200.gen.c4src import C4SourceConfig, c4_source
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    from paper_2406_13881_b200.gen.lulesh import generate_lulesh
    _check(generate_lulesh(seed=1))
    _check(generate(7, GenConfig(n_funcs=60, n_globals=24, n_stmts=40, p_kernel=0.3)))
    for i in (0, 777, 4242, 99999):
        _check(c4_source(C4SourceConfig(), i))


def test_operator_soup():
    """Random expressions over every binary level, unary, casts, calls,
    subscripts and parentheses, plus truncated ones (the errors)."""
    rng = random.Random(5)
    ops = ["||", "&&", "==", "!=", "<", ">", "<=", ">=", "+", "-", "*", "/", "%"]

    def expr(d):
        r = rng.random()
        if d > 4 or r < 0.3:
            return rng.choice(["a", "b[i]", "f(a, b[1])", "2", "3.5", "-a", "!b[0]", "(double)a",
                               "i++", "--i"])
        if r < 0.4:
            return "(" + expr(d + 1) + ")"
        return expr(d + 1) + " " + rng.choice(ops) + " " + expr(d + 1)

    body = []
    for k in range(300):
        body.append("  s = %s;" % expr(0))
    head = "double a; double b[8]; double s; int i;\ndouble f(double x, double y) { return x; }\n"
    _check(head + "int main() {\n" + "\n".join(body) + "\n  return 0;\n}\n")
    for cut in ("a +", "a + * b", "a || && b", "(a + b", "a < b >", "a ==", "b[ + ]"):
        _check(head + "int main() {\n  s = %s;\n  return 0;\n}\n" % cut)


def test_paused_gc_restores_state():
    import gc
    from paper_2406_13881_b200.frontend import paused_gc
    assert gc.isenabled()
    with paused_gc():
        assert not gc.isenabled()
    assert gc.isenabled()
    gc.disable()
    try:
        with paused_gc():
            pass
        assert not gc.isenabled()
    finally:
        gc.enable()
