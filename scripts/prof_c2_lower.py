"""cProfile of the lowering of C2 (LULESH-shaped unit), 200 repetitions."""
import cProfile
import pathlib
import pstats
import sys
import time
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13881_b200._host import import_dartomp  # noqa: E402
import_dartomp()
import dartomp.pipeline as ref  # noqa: E402
from paper_2406_13881_b200.gen.lulesh import generate_lulesh  # noqa: E402
from paper_2406_13881_b200.lower import lower_function  # noqa: E402
a = ref.load(text=generate_lulesh(seed=1))
items = [(a.src, a.cfgs[k], a.accesses[k], a.table) for k in a.cfgs]
for _ in range(20):
    [lower_function(*it) for it in items]
t = time.perf_counter()
for _ in range(200):
    [lower_function(*it) for it in items]
print("lowering %.3f ms" % ((time.perf_counter() - t) / 200 * 1e3))
cProfile.run("for _ in range(200): [lower_function(*it) for it in items]", "/tmp/c2l.prof")
pstats.Stats("/tmp/c2l.prof").sort_stats("tottime").print_stats(20)
