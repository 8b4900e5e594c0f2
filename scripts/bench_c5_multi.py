"""Configuration C5 across ranks (torchrun, one process per GPU): kernel (c)
with the summary exchange fused into the producing kernel over peer memory
(`PeerSummaries`, dfx_cgp_*) beside the all-gather path (`ShardedSummaries`:
wave kernel + NCCL all-gather of the rebuilt rows).  Prints one JSON line on
rank 0 with the max-over-ranks wall time per solve of each path.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        scripts/bench_c5_multi.py [n_funcs]

DFX_BENCH_SHARE_GPU=1 (testing only) runs every rank on GPU 0 with gloo."""
import json
import os
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2406_13881_b200 import _abi  # noqa: E402
from paper_2406_13881_b200.distributed import PeerSummaries, ShardedSummaries  # noqa: E402
from paper_2406_13881_b200.gen.c5 import generate_c5  # noqa: E402
from paper_2406_13881_b200.interproc import solve_call_graph  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    share = bool(os.environ.get("DFX_BENCH_SHARE_GPU"))
    local = 0 if share else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo" if share else "nccl")
    g = generate_c5(seed=0, n_funcs=n)
    ref = solve_call_graph(g)                         # single-GPU engine, the parity target

    def timed(fn, reps=5):
        fn()
        ts = []
        for _ in range(reps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            r = fn()
            ts.append(time.perf_counter() - t0)
        t = torch.tensor([min(ts)], dtype=torch.float64)
        if world > 1:
            t = t.cuda() if not share else t
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) * 1e3, r

    eng = _abi.engine(local)
    ps = PeerSummaries(g, rank, world, eng=eng)
    ms_peer, rp = timed(ps.solve)
    ss = ShardedSummaries(g, rank, world, device="cuda:%d" % local)
    ms_nccl, rn = timed(ss.solve)
    def exact(x):
        return bool(np.array_equal(x[0], ref.bits) and np.array_equal(x[2], ref.len)
                    and x[3] == ref.passes)
    ok_peer, ok_nccl = exact(rp), exact(rn)
    if world > 1:
        flags = torch.tensor([int(ok_peer), int(ok_nccl)], dtype=torch.int32)
        flags = flags.cuda() if not share else flags
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        ok_peer, ok_nccl = bool(flags[0]), bool(flags[1])
    if rank == 0:
        print(json.dumps({"workload": "C5: %d functions, depth-12 chains, %d rank(s)%s"
                                      % (g.n_funcs, world, " sharing one GPU" if share else ""),
                          "passes": rp[3], "fused_peer_ms": ms_peer,
                          "allgather_ms": ms_nccl, "single_gpu_device_ms": ref.kernel_ms,
                          "fused_peer_bit_exact": ok_peer, "allgather_bit_exact": ok_nccl}),
              flush=True)
    ps.close()
    ss.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
