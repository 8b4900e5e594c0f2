"""Where the forked lowering of a large unit spends its time: pool start,
the workers' map (lowering + result pickling), the parent's rebuild of
FnPrograms, pool teardown (C4-style source program of N functions)."""
import multiprocessing as mp
import pathlib
import sys
import time
import gc

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13881_b200._host import import_dartomp  # noqa: E402
import_dartomp()
import dartomp.pipeline as ref  # noqa: E402
from paper_2406_13881_b200 import dataflow as df  # noqa: E402
from paper_2406_13881_b200.lower import lower_function  # noqa: E402
from paper_2406_13881_b200.gen.cprog import GenConfig, generate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
a = ref.load(text=generate(7, GenConfig(n_funcs=n, n_globals=24, n_stmts=40, p_kernel=0.3)))
items = [(a.src, a.cfgs[k], a.accesses[k], a.table) for k in a.cfgs]
gc.disable()
for rep in range(2):
    t0 = time.perf_counter()
    df.lower_functions(items)
    t1 = time.perf_counter()
    df._FORK_ITEMS = list(items)
    workers = min(16, mp.cpu_count())
    t2 = time.perf_counter()
    pool = mp.get_context("fork").Pool(workers)
    t3 = time.perf_counter()
    res = pool.map(df._lower_portable, range(len(items)), chunksize=max(1, len(items) // (8 * workers)))
    t4 = time.perf_counter()
    pool.close(); pool.join()
    t5 = time.perf_counter()
    print("lower_functions %.0f ms | pool start %.0f, map %.0f, teardown %.0f ms"
          % (1e3 * (t1 - t0), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t5 - t4)))
t = time.perf_counter()
for it in items[:100]:
    lower_function(*it)
print("serial lowering %.2f ms per function" % ((time.perf_counter() - t) * 10))
