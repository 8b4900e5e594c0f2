"""Generate C3 and run N solves (for ncu captures)."""
import sys
import pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2406_13881_b200.csr import C3Config, CsrProblem  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = CsrProblem.generate_c3(C3Config())
for _ in range(n):
    st = prob.solve()
print("solve_ms", st.solve_ms, "kernel_ms", st.kernel_ms, "rounds", st.rounds_h, st.rounds_d)
