"""Where the drop-in summarize_all spends its time on the 10k-function C5
program: the call-graph lowering, the kernel (c) call, the CallSummary build."""
import pathlib
import sys
import time
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13881_b200._host import import_dartomp  # noqa: E402
import_dartomp()
from dartomp.access import VariableTable, classify_accesses  # noqa: E402
from dartomp.astcfg import build_astcfg  # noqa: E402
from dartomp.lexer import expand_defines  # noqa: E402
from dartomp.nodes import defined_functions  # noqa: E402
from dartomp.parser import parse  # noqa: E402
from dartomp.source import SourceFile  # noqa: E402
from paper_2406_13881_b200 import interproc as ip  # noqa: E402
from paper_2406_13881_b200.gen.callgraph import CallGraphConfig, generate  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
text = generate(7, CallGraphConfig(n_funcs=n))
src = SourceFile.from_text(text, path="c5.c")
pre = expand_defines(src)
tu, _ = parse(src, pre)
table = VariableTable(src, tu)
cfgs, raw = {}, {}
for name, fn in defined_functions(tu).items():
    cfgs[name] = build_astcfg(src, fn)
    raw[name] = classify_accesses(src, cfgs[name], table)
ip.summarize_all(src, tu, cfgs, raw, table)
for _ in range(3):
    t0 = time.perf_counter()
    g = ip.lower_call_graph(src, tu, cfgs, raw, table)
    t1 = time.perf_counter()
    r = ip.solve_call_graph(g)
    t2 = time.perf_counter()
    out = ip.summaries_from_result(g, r)
    t3 = time.perf_counter()
    print("lower %.1f ms, solve %.1f ms (device %.2f), summaries %.1f ms" % (
        1e3 * (t1 - t0), 1e3 * (t2 - t1), r.kernel_ms, 1e3 * (t3 - t2)))
print("functions %d, slots %d (params %d, globals %d), waves %d, passes %d, launches %d, sources %d" % (
    g.init_bits.shape[0], g.init_bits.shape[1], g.n_params, len(g.globals), g.wave_off.shape[0] - 1,
    r.passes, getattr(r, "launches", -1), g.src.shape[0]))
import numpy as np  # noqa: E402
ws = np.diff(g.wave_off)
print("wave sizes: max %d, mean %.1f, waves of size 1: %d" % (ws.max(), ws.mean(), int((ws == 1).sum())))
from paper_2406_13881_b200.gen.c5 import generate_c5  # noqa: E402
g5 = generate_c5(seed=0, n_funcs=10_000)
r5 = ip.solve_call_graph(g5)
print("gen/c5: functions %d, slots %d, waves %d, passes %d, device %.2f ms" % (
    g5.init_bits.shape[0], g5.init_bits.shape[1], g5.wave_off.shape[0] - 1, r5.passes, r5.kernel_ms))
so = np.diff(g.src_off)
print("sources per function: max %d (function %s), mean %.2f, >100: %d" % (
    so.max(), g.names[int(so.argmax())], so.mean(), int((so > 100).sum())))
print("gen/c5 sources per function: max %d" % int(np.diff(g5.src_off).max()))
