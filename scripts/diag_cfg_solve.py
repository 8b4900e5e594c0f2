"""Kernel (a) on a real-program CSR (cfgprog: C4 source units lowered over
their AST-CFGs): rounds, evaluations and time per chunk size."""
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2406_13881_b200._host import import_dartomp  # noqa: E402
import_dartomp()
from dartomp.pipeline import load  # noqa: E402
from paper_2406_13881_b200.cfgprog import lower_program  # noqa: E402
from paper_2406_13881_b200.csr import CsrProblem  # noqa: E402
from paper_2406_13881_b200.gen.c4src import C4SourceConfig, c4_source  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
items = []
for k in range(n):
    a = load(text=c4_source(C4SourceConfig(), k * (100_000 // n)))
    items += [(nm, a.src, a.cfgs[nm], a.accesses[nm], a.table) for nm in a.cfgs]
prog = lower_program(items)
print("nodes", prog.n_nodes, "words", prog.words, "nnz", prog.col.shape[0])
p = CsrProblem.from_acc(prog.row_ptr, prog.col, prog.kind, prog.acc_off, prog.acc, prog.S, prog.words)
for chunk in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,8,56,128,256,512,1024").split(",")]:
    for _ in range(2):
        st = p.solve(chunk)
    t = time.perf_counter()
    st = p.solve(chunk)
    print("chunk", chunk, {k: v for k, v in st.as_dict().items() if k in ("rounds_h", "rounds_d", "evaluated", "kernel_ms", "solve_ms")},
          "wall %.2f ms" % ((time.perf_counter() - t) * 1e3))
# the one-call path: dfx_mfp_acc alone vs solve_program (the Python mapping included)
import statistics  # noqa: E402
from paper_2406_13881_b200.cfgprog import solve_program  # noqa: E402
from paper_2406_13881_b200.csr import AccSession  # noqa: E402
sess = AccSession()
for label, fn in (("dfx_mfp_acc", lambda: sess.run(prog.row_ptr, prog.col, prog.kind, prog.acc_off,
                                                  prog.acc, prog.S, prog.words)),
                  ("solve_program", lambda: solve_program(prog, sess))):
    fn()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t) * 1e3)
    print(label, "%.2f ms" % statistics.median(ts), "solve_ms %.2f kernel_ms %.2f req_ms %.2f" % (
        sess.stats.solve_ms, sess.stats.kernel_ms, sess.stats.req_ms))
