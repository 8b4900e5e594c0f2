"""Configuration C5 measurement: 10k-function call graph through kernel (c)
(dfx_summaries), beside the C port and, on a sample, the reference Python.
Prints one JSON line."""
import json
import pathlib
import statistics
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2406_13881_b200.gen.c5 import generate_c5  # noqa: E402
from paper_2406_13881_b200.interproc import solve_call_graph  # noqa: E402
import _oracle  # noqa: E402  (CPU baseline leg)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
g = generate_c5(seed=0, n_funcs=n)
for _ in range(3):
    r = solve_call_graph(g)
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    r = solve_call_graph(g)
    ts.append(time.perf_counter() - t0)
t0 = time.perf_counter()
e = solve_call_graph(g, runner=_oracle.summaries_runner)
cpu = time.perf_counter() - t0
ok = bool((r.bits == e.bits).all() and (r.len == e.len).all() and r.passes == e.passes)
print(json.dumps({"workload": "C5: %d functions, depth-12 chains, 10%% back edges, 256 globals"
                  % g.n_funcs, "passes": r.passes, "wave_launches": r.launches,
                  "device_ms": r.kernel_ms, "call_ms_median": 1e3 * statistics.median(ts),
                  "c_port_ms_1core": 1e3 * cpu, "bit_exact_vs_port": ok}))
