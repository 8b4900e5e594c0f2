"""Generate C3, run one solve and one requirement-list pass (for ncu captures)."""
import sys
import pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2406_13881_b200.csr import C3Config, CsrProblem  # noqa: E402
prob = CsrProblem.generate_c3(C3Config())
st = prob.solve()
rl = prob.requirements_list()
print("solve_ms", st.solve_ms, "kernel_ms", st.kernel_ms, "rounds", st.rounds_h, st.rounds_d,
      "requirements", rl.vars.shape[0])
