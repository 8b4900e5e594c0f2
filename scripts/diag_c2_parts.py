"""Where the drop-in plan_transform spends its time on C2 (LULESH-shaped,
one translation unit): lowering, packing, the E1 call (dfx_replay_batch,
host buffers), decoding and the rest, medians over repeats."""
import pathlib
import statistics
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13881_b200._host import import_dartomp  # noqa: E402
import_dartomp()
import dartomp.pipeline as ref  # noqa: E402
from paper_2406_13881_b200 import dataflow as df, pipeline as eng  # noqa: E402
from paper_2406_13881_b200.gen.lulesh import generate_lulesh  # noqa: E402

a = eng.load(text=generate_lulesh(seed=1))
T = {}


def wrap(name, f):
    def g(*args, **kw):
        t = time.perf_counter()
        r = f(*args, **kw)
        T.setdefault(name, []).append(time.perf_counter() - t)
        return r
    return g


df.lower_functions = wrap("lower", df.lower_functions)
df.pack = wrap("pack", df.pack)
df.run_replay = wrap("replay", df.run_replay)
df._decode_cols = wrap("decode", df._decode_cols)
eng.plan_transform = wrap("total", eng.plan_transform)
for _ in range(5):
    eng.plan_transform(a)
T.clear()
for _ in range(30):
    eng.plan_transform(a)
ts = [time.perf_counter()]
for _ in range(30):
    ref.plan_transform(a)
ref_ms = 1e3 * (time.perf_counter() - ts[0]) / 30
n = len(T["total"])
per = {k: 1e3 * sum(v) / n for k, v in T.items()}
per["rest"] = per["total"] - sum(v for k, v in per.items() if k != "total")
print({k: round(v, 3) for k, v in per.items()}, "reference plan_transform %.3f ms" % ref_ms)
