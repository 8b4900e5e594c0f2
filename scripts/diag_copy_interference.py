"""Does a concurrent H2D copy slow the E1 kernel down?  Device-resident C4
replay timed alone and with an 8 GB pinned H2D copy running on another
stream."""
import sys, pathlib, threading
import numpy as np
import torch
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2406_13881_b200 import _abi
from paper_2406_13881_b200.batch import C4Config, ReplayBatch, c4_generate

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
eng = _abi.engine(0)
batch, _ = c4_generate(C4Config(n_funcs=n), np.arange(n))
rb = ReplayBatch(batch, eng=eng)
for _ in range(2):
    _, kms = rb.run()
print("alone: %.1f ms" % kms)
h = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True)
d = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for rep in range(2):
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    _, kms = rb.run()
    torch.cuda.synchronize()
    print("with concurrent H2D: %.1f ms" % kms)
