"""One dfx_sim_batch launch over C4 source programs (transformed + original),
for ncu captures of sim_kernel.  Host preparation in a spawn pool."""
import multiprocessing as mp
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))

if __name__ == "__main__":
    import os
    import sim_worker
    from paper_2406_13881_b200.simulator import run_sim
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    jobs = [(k * (100_000 // n), m) for k in range(n) for m in ("annotated", "implicit")]
    with mp.get_context("spawn").Pool(len(os.sched_getaffinity(0))) as pool:
        rows = pool.map(sim_worker.one, jobs, chunksize=1)
    progs = [r[1] for r in rows]
    raw = run_sim(progs)
    raw = run_sim(progs)
    print("programs", len(progs), "ops", sum(p.ops.shape[0] for p in progs), "kernel_ms", raw.kernel_ms)
