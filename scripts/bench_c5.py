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

# ---- drop-in comparison at the reference's own API (C source, parse excluded)
# `dartomp.interproc.summarize_all` (interproc.py:90) against this package's
# drop-in `summarize_all` (lowering + kernel (c) + CallSummary rebuild) on
# the same parsed translation unit.  Needs the reference package (the
# driver's baseline/_ref install); skipped when it is absent.
try:
    from paper_2406_13881_b200._host import have_dartomp, import_dartomp
    if "--reference" in sys.argv and have_dartomp():
        import_dartomp()
        from dartomp.access import VariableTable, classify_accesses
        from dartomp.astcfg import build_astcfg
        from dartomp.interproc import summarize_all as ref_summarize_all
        from dartomp.lexer import expand_defines
        from dartomp.nodes import defined_functions
        from dartomp.parser import parse
        from dartomp.source import SourceFile
        from paper_2406_13881_b200.gen.callgraph import CallGraphConfig, generate
        from paper_2406_13881_b200.interproc import summarize_all as our_summarize_all
        nref = int(sys.argv[sys.argv.index("--reference") + 1]) if len(sys.argv) > sys.argv.index("--reference") + 1 else 2400
        text = generate(0, CallGraphConfig(n_funcs=nref))
        src = SourceFile.from_text(text, path="c5.c")
        pre = expand_defines(src)
        tu, _ = parse(src, pre)
        table = VariableTable(src, tu)
        cfgs, raw = {}, {}
        for name, fn in defined_functions(tu).items():
            cfgs[name] = build_astcfg(src, fn)
            raw[name] = classify_accesses(src, cfgs[name], table)
        t0 = time.perf_counter()
        ref = ref_summarize_all(src, tu, cfgs, raw, table)
        t_ref = time.perf_counter() - t0
        ours = our_summarize_all(src, tu, cfgs, raw, table)     # warm
        t0 = time.perf_counter()
        ours = our_summarize_all(src, tu, cfgs, raw, table)
        t_ours = time.perf_counter() - t0
        same = list(ref) == list(ours) and all(
            list(ref[k].param_effects.items()) == list(ours[k].param_effects.items())
            and list(ref[k].global_effects.items()) == list(ours[k].global_effects.items())
            for k in ref)
        print(json.dumps({"workload": "C5 from C source: %d functions, depth-12 chains" % len(cfgs),
                          "reference_summarize_all_ms": 1e3 * t_ref,
                          "dropin_summarize_all_ms": 1e3 * t_ours,
                          "identical_summaries_and_dict_order": bool(same)}))
except ImportError:
    pass
