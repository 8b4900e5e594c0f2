"""C4 replay kernel time for the current $DFX_NV (variables per lane), full
100k batch device-resident, plus a parity check of 400 functions vs the CPU
oracle."""
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2406_13881_b200.batch import C4Config, ReplayBatch, c4_generate  # noqa: E402
from paper_2406_13881_b200.dataflow import PackedBatch, run_replay  # noqa: E402
import _golden  # noqa: E402
import _oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
b, facts = c4_generate(C4Config(n_funcs=n), np.arange(n, dtype=np.int32))
rb = ReplayBatch(b)
for _ in range(2):
    rb.run()
ms = []
for _ in range(5):
    ev, t = rb.run()
    ms.append(t)
print("functions", n, "events", ev, "kernel_ms", sorted(ms)[2], "facts/s %.3e" % (facts / sorted(ms)[2] * 1e3))
rb.close()
sel = np.arange(0, n, max(1, n // 400), dtype=np.int32)[:400]
sb, _ = c4_generate(C4Config(n_funcs=n), sel)
got = run_replay(sb)
exp = run_replay(sb, runner=_oracle.replay_runner_mt)
_golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
print("parity ok on", len(sel), "functions")
