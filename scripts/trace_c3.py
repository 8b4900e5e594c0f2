"""One traced C3 solve (per-round stats on stderr via DFX_TRACE=1)."""
import os
import sys
import pathlib
os.environ["DFX_TRACE"] = "1"
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2406_13881_b200.csr import C3Config, CsrProblem  # noqa: E402
prob = CsrProblem.generate_c3(C3Config())
for _ in range(3):
    st = prob.solve()
print("solve_ms", st.solve_ms, "kernel_ms", st.kernel_ms, file=sys.stderr)
