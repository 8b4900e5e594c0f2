"""C4-from-source parity helpers (test infrastructure): the committed
reference fixture and a spawn-pool worker that parses a slice of the sample
with the host front end and runs it through the drop-in (CUDA, or the CPU
oracle when `oracle` is set), returning the indices whose result differs
from the reference's."""
from __future__ import annotations

import gzip
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden" / "c4_source_plans.json.gz"


def gold() -> dict:
    return json.loads(gzip.decompress(GOLD.read_bytes()))


def parse(i: int):
    from paper_2406_13881_b200._host import import_dartomp
    from paper_2406_13881_b200.gen.c4src import C4SourceConfig, c4_source
    import_dartomp()
    from dartomp.pipeline import load
    a = load(text=c4_source(C4SourceConfig(), i))
    name = "c4_%d" % i
    return a, (a.src, a.cfgs[name], a.accesses[name], a.table)


def check_slice(args) -> list:
    rows, oracle = args
    import os
    os.environ["DFX_LOWER_WORKERS"] = "1"     # a pool worker lowers serially
    for p in (str(ROOT), str(ROOT / "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import _cases
    from paper_2406_13881_b200.dataflow import analyze_functions
    runner = None
    if oracle:
        import _oracle
        runner = _oracle.replay_runner
    items = [parse(r["i"])[1] for r in rows]
    got = analyze_functions(items, runner=runner)
    return [r["i"] for r, g in zip(rows, got) if _cases.canon_result(g.get) != r["result"]]


def check_all(rows, oracle=False, procs=None) -> list:
    """Spawned workers (fresh processes: no CUDA state inherited)."""
    import multiprocessing as mp
    import os
    procs = procs or max(1, min(16, len(os.sched_getaffinity(0))))
    rows = sorted(rows, key=lambda r: -r["nodes"])
    slices = [rows[k::procs] for k in range(procs)]
    with mp.get_context("spawn").Pool(procs) as pool:
        bad = pool.map(check_slice, [(s, oracle) for s in slices if s])
    return sorted(i for b in bad for i in b)


# ---- C4 CPU baseline: the reference itself, one process per core

def ref_time_one(i: int):
    """Parse function i of the C4 source batch (untimed), then time the
    reference `analyze_function` (dartomp/dataflow.py:737-740) on it.
    Returns (facts, analyze seconds, parse seconds); facts = host CFG nodes x
    variables touched by the function's accesses."""
    import time
    from paper_2406_13881_b200._host import import_dartomp
    from paper_2406_13881_b200.gen.c4src import C4SourceConfig, c4_source
    import_dartomp()
    from dartomp.dataflow import analyze_function
    from dartomp.pipeline import load
    t0 = time.perf_counter()
    a = load(text=c4_source(C4SourceConfig(), i))
    name = "c4_%d" % i
    cfg, accs = a.cfgs[name], a.accesses[name]
    t1 = time.perf_counter()
    analyze_function(a.src, cfg, accs, a.table)
    t2 = time.perf_counter()
    return len(cfg.nodes) * len({id(x.var) for x in accs}), t2 - t1, t1 - t0


def host_info() -> dict:
    import os
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "cpu_model": model}


def reference_c4_baseline(n_funcs: int = 1000, stride: int = 100, procs: int | None = None) -> dict:
    """BASELINE.md §3 C4 CPU plan: the reference `analyze_function` in
    multiprocessing.Pool(ncores) over a fixed seeded sample of `n_funcs`
    functions of the C4 source batch (every `stride`-th), parse excluded.
    Aggregate facts/s = sum(facts) / (sum(analyze s) / procs): perfect
    scaling across the processes is assumed, which can only favour the
    reference."""
    import multiprocessing as mp
    import os
    import time
    procs = procs or len(os.sched_getaffinity(0))
    sample = [k * stride for k in range(n_funcs)]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(procs) as pool:
        rows = pool.map(ref_time_one, sample, chunksize=4)
    wall = time.perf_counter() - t0
    facts = sum(r[0] for r in rows)
    ana = sum(r[1] for r in rows)
    parse = sum(r[2] for r in rows)
    value = facts / (ana / procs)
    info = host_info()
    return {"value": value, "unit": "facts/s", "cores": procs, "kind": "reference",
            "sample": "reference dartomp analyze_function (dataflow.py:737) in "
                      "multiprocessing.Pool(%d) over %d functions of the C4 source batch "
                      "(gen/c4src.py seed 0, every %d-th of 100k; 64-2048 host CFG nodes); "
                      "parse excluded; facts = CFG nodes x vars touched" % (procs, n_funcs, stride),
            "facts": facts, "analyze_cpu_s": ana, "parse_cpu_s": parse, "wall_s": wall,
            "single_core_facts_per_s": facts / ana, **info}
