"""Where the C4 host-buffer call spends its time: wall time of
dfx_replay_batch vs its device span (first range's replay start to the last
range's end) vs the device-resident launch over the same batch."""
import sys, time, pathlib
import numpy as np
import torch
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2406_13881_b200 import _abi
from paper_2406_13881_b200.batch import C4Config, ReplayBatch, c4_generate
from paper_2406_13881_b200.dataflow import ReplaySession

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
def pinned(shape, dtype):
    nb = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = torch.empty(max(1, nb), dtype=torch.uint8, pin_memory=True)
    return buf.numpy()[:nb].view(dtype).reshape(shape)
eng = _abi.engine(0)
t = time.perf_counter()
batch, _ = c4_generate(C4Config(n_funcs=n), np.arange(n), alloc=pinned)
print("generate %.0f ms" % ((time.perf_counter() - t) * 1e3))
rb = ReplayBatch(batch, eng=eng)
for _ in range(2):
    _, kms = rb.run()
print("device-resident replay %.1f ms" % kms)
sess = ReplaySession(eng, alloc=pinned, event_cap=rb.cap)
for i in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    raw = sess.run(batch)
    torch.cuda.synchronize()
    print("host-buffer call %.1f ms wall, device span %.1f ms, events %d" %
          ((time.perf_counter() - t) * 1e3, raw.kernel_ms, raw.events.shape[0]))
from paper_2406_13881_b200.dataflow import pack_ops  # noqa: E402
pk_np = pack_ops(batch.ops)
pk = pinned(pk_np.shape, np.uint32)
pk[:] = pk_np
for i in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    raw = sess.run(batch, pk)
    torch.cuda.synchronize()
    print("packed host-buffer call %.1f ms wall, device span %.1f ms" %
          ((time.perf_counter() - t) * 1e3, raw.kernel_ms))
import os  # noqa: E402
if os.environ.get("DFX_TRACE"):
    print("(trace above)")
