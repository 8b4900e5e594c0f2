"""Phase timeline of the C3 host-buffer call on byte-coded lists
(dfx_mfp_acc8 with DFX_TRACE=1): upload + decode, solve, requirements + D2H."""
import os
import pathlib
import sys
os.environ["DFX_TRACE"] = "1"
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2406_13881_b200.csr import Acc8Session, C3Config, CsrProblem, acc_to_b8, c3_scalar_mask  # noqa: E402


def pinned(shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    return torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy().view(dtype).reshape(shape)


cfg = C3Config()
prob = CsrProblem.generate_c3(cfg)
rp, col, kind, R, W = prob.export_inputs(alloc=pinned)
del R, W
off, acc = prob.export_acc(alloc=pinned)
bo, b = acc_to_b8(off, acc)
boff, bb = pinned(bo.shape, np.int32), pinned(b.shape, np.uint8)
boff[:] = bo
bb[:] = b
S = c3_scalar_mask(cfg)
sess = Acc8Session(alloc=pinned)
for _ in range(4):
    sess.run(rp, col, kind, boff, bb, S, cfg.words)
print("h2d MB", (rp.nbytes + col.nbytes + kind.nbytes + boff.nbytes + bb.nbytes) / 1e6)
print("req_ms (kernel b + byte counts + scans + encoding, device)", sess.stats.req_ms)
