"""`plan_transform`'s input check (`pipeline.py:65-82`) through the drop-in:
the first pre-annotated directive of the unit, in the reference's pre-order,
raises the same PreconditionError -- found per function by the (forked,
for >= 64 functions) lowering, and by a walk of the nodes outside function
definitions.  CPU only: the check raises before any launch."""
import pytest

import _oracle
from paper_2406_13881_b200._host import import_dartomp

import_dartomp()
import dartomp.pipeline as ref  # noqa: E402
from dartomp.diagnostics import PreconditionError  # noqa: E402

from paper_2406_13881_b200 import pipeline as eng  # noqa: E402

KERNEL = """    #pragma omp target teams distribute parallel for%s
    for (int i = 0; i < N; ++i) {
        g%d[i] = g%d[i] * 2.0;
    }
"""
REGION = """    #pragma omp target data map(tofrom: g%d)
    {
%s    }
"""


def program(n_funcs: int, premapped: dict[int, str]) -> str:
    out = ["#define N 64\n"]
    out += ["double g%d[N];\n" % i for i in range(n_funcs)]
    for f in range(n_funcs):
        body = "    for (int i = 0; i < N; ++i) {\n        g%d[i] = 1.0;\n    }\n" % f
        how = premapped.get(f)
        if how == "map_clause":
            body += KERNEL % (" map(tofrom: g%d)" % f, f, f)
        elif how == "region":
            body += REGION % (f, KERNEL % ("", f, f))
        elif how == "update":
            body += KERNEL % ("", f, f) + "    #pragma omp target update from(g%d)\n" % f
        else:
            body += KERNEL % ("", f, f)
        out.append("void f%d(void) {\n%s}\n" % (f, body))
    out.append("int main(void) {\n    f0();\n    return 0;\n}\n")
    return "".join(out)


def _err(fn):
    with pytest.raises(PreconditionError) as e:
        fn()
    return str(e.value)


@pytest.mark.parametrize("n_funcs,premapped", [
    (3, {1: "region"}),
    (3, {2: "map_clause", 1: "update"}),
    (80, {50: "map_clause", 70: "region"}),          # forked lowering
    (80, {79: "update"}),
    (70, {3: "update", 4: "region", 66: "map_clause"}),
])
def test_first_preannotated_directive_raises_like_the_reference(n_funcs, premapped):
    a = ref.load(text=program(n_funcs, premapped))
    exp = _err(lambda: ref.plan_transform(a))
    got = _err(lambda: eng.plan_transform(a, replay_runner=_oracle.replay_runner))
    assert got == exp


def test_clean_unit_passes_the_check():
    a = ref.load(text=program(70, {}))
    got = eng.plan_transform(a, replay_runner=_oracle.replay_runner)
    exp = ref.plan_transform(a)
    assert [(p.function.name, p.region.clause_text() if p.region else None) for p in got] == \
           [(p.function.name, p.region.clause_text() if p.region else None) for p in exp]
