"""C4-style functions from C source through the drop-in at the reference API:
a seeded program with many structured functions (gen/cprog.py), the
reference `plan_transform` (per-function `analyze_function`) beside this
package's `plan_transform` (lowering of every function + one E1 launch),
same parsed translation unit.  Prints one JSON line."""
import json
import pathlib
import statistics
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2406_13881_b200._host import import_dartomp  # noqa: E402
import_dartomp()
import dartomp.pipeline as ref  # noqa: E402

from paper_2406_13881_b200 import pipeline as eng  # noqa: E402
from paper_2406_13881_b200.gen.cprog import GenConfig, generate  # noqa: E402

n_funcs = int(sys.argv[1]) if len(sys.argv) > 1 else 400
cfg = GenConfig(n_funcs=n_funcs, n_globals=24, n_stmts=40, p_kernel=0.3)
text = generate(7, cfg)
a = ref.load(text=text)


def timed(fn, reps=3):
    fn()
    ts = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * statistics.median(ts), out


def plans_key(plans):
    return [(id(p.function), [(u.kind, u.names, id(u.anchor), u.position) for u in p.all_plans],
             (id(p.region.begin), p.region.clause_text()) if p.region is not None else None,
             tuple(p.suppressed)) for p in plans]


try:
    ms_ref, pr = timed(lambda: ref.plan_transform(a))
    ms_eng, pe = timed(lambda: eng.plan_transform(a))
    same = plans_key(pr) == plans_key(pe)
    err = None
except Exception as e:      # noqa: BLE001 -- a generated analysis error is reported, not fatal
    ms_ref = ms_eng = None
    same, err = None, repr(e)
print(json.dumps({"workload": "%d functions from C source (%d lines)" % (len(a.cfgs), len(text.splitlines())),
                  "reference_plan_transform_ms": ms_ref, "dropin_plan_transform_ms": ms_eng,
                  "identical_plans": same, "error": err}))
