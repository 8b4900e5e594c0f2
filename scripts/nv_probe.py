"""Replay n C4 functions once (ncu probe of replay_kernel under $DFX_NV)."""
import pathlib
import sys
import numpy as np
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2406_13881_b200.batch import C4Config, ReplayBatch, c4_generate  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
b, facts = c4_generate(C4Config(n_funcs=100000), np.arange(0, 100000, 100000 // n, dtype=np.int32)[:n])
rb = ReplayBatch(b)
ev, ms = rb.run()
print("functions", n, "events", ev, "kernel_ms", ms)
