"""Where the drop-in plan_transform spends its time on C4-style functions
from C source: lowering (forked workers), packing, the E1 launch, decoding,
and the rest (the input check, Python glue)."""
import sys, time, pathlib
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13881_b200._host import import_dartomp
import_dartomp()
import dartomp.pipeline as ref
from paper_2406_13881_b200 import dataflow as df, pipeline as eng
from paper_2406_13881_b200.gen.cprog import GenConfig, generate

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
a = ref.load(text=generate(7, GenConfig(n_funcs=n, n_globals=24, n_stmts=40, p_kernel=0.3)))
T = {}
def wrap(name, f):
    def g(*args, **kw):
        t = time.perf_counter(); r = f(*args, **kw); T[name] = T.get(name, 0) + time.perf_counter() - t
        return r
    return g
df.lower_functions = wrap("lower", df.lower_functions)
df.pack = wrap("pack", df.pack)
df.run_replay = wrap("replay", df.run_replay)
df._decode_cols = wrap("decode", df._decode_cols)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    T.clear()
    t = time.perf_counter(); eng.plan_transform(a); tot = time.perf_counter() - t
    print("total %.0f ms" % (tot * 1e3), {k: round(v * 1e3) for k, v in T.items()},
          "rest %.0f" % ((tot - sum(T.values())) * 1e3))
