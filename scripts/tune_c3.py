"""Sweep the fixpoint kernel's chunk size on configuration C3 (GPU)."""
import json
import sys
import pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2406_13881_b200.csr import C3Config, CsrProblem  # noqa: E402

chunks = [int(x) for x in sys.argv[1:]] or [32, 64, 128, 256, 512, 1024, 4096]
prob = CsrProblem.generate_c3(C3Config())
for c in chunks:
    for _ in range(2):
        prob.solve(c)
    ms = []
    for _ in range(5):
        st = prob.solve(c)
        ms.append((st.solve_ms, st.kernel_ms))
    best = min(ms)
    print(json.dumps({"chunk": c, "solve_ms": best[0], "kernel_ms": best[1],
                      "rounds": [st.rounds_h, st.rounds_d], "evaluated": st.evaluated,
                      "rows_read": st.rows_read, "rows_written": st.rows_written}), flush=True)
