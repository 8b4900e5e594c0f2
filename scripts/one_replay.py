"""Generate a C4 sub-batch and replay it (for ncu captures of replay_kernel)."""
import sys
import pathlib
import numpy as np
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2406_13881_b200.batch import C4Config, ReplayBatch, c4_generate  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
b, facts = c4_generate(C4Config(n_funcs=n), np.arange(n, dtype=np.int32))
rb = ReplayBatch(b)
for _ in range(2):
    ev, ms = rb.run()
print("functions", n, "facts", facts, "events", ev, "kernel_ms", ms, "facts/s", facts / ms * 1e3)
