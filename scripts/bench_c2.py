"""Configuration C2 through the drop-in at the reference's API: the
reference `dartomp.pipeline` (load + plan_transform + apply_plans) beside
this package's `pipeline` (same front end; kernel (c) summaries, one E1
launch for all functions), on the same LULESH-shaped source.  Prints one
JSON line: medians over repeats, and whether the transformed text is
byte-identical."""
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
from dartomp.rewriter import apply_plans  # noqa: E402

from paper_2406_13881_b200 import pipeline as eng  # noqa: E402
from paper_2406_13881_b200.gen.lulesh import generate_lulesh  # noqa: E402


def run(mod, text, reps=7):
    times = {"load": [], "plan": [], "total": []}
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        a = mod.load(text=text)
        t1 = time.perf_counter()
        plans = mod.plan_transform(a)
        t2 = time.perf_counter()
        out = apply_plans(a.src, plans)
        t3 = time.perf_counter()
        times["load"].append(t1 - t0)
        times["plan"].append(t2 - t1)
        times["total"].append(t3 - t0)
    return {k: 1e3 * statistics.median(v) for k, v in times.items()}, out


text = generate_lulesh(seed=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
run(eng, text, reps=2)                     # warm the engine (library, device)
r_ref, o_ref = run(ref, text)
r_eng, o_eng = run(eng, text)
print(json.dumps({"workload": "C2: LULESH-shaped program, %d lines" % len(text.splitlines()),
                  "reference_ms": r_ref, "dropin_ms": r_eng,
                  "identical_output": o_ref.text == o_eng.text if hasattr(o_ref, "text") else o_ref == o_eng}))
