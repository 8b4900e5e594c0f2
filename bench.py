#!/usr/bin/env python
"""Benchmark: data-flow facts/sec to fixpoint on configuration C3.

Workload (BASELINE.json configs[2], the HBM-roofline configuration): one
synthetic CFG of 2^20 nodes, average in-degree 2.5, 4096 variables per GPU,
20% kernel nodes, 1/32 access density, 2% firstprivate-eligible scalars
(DESIGN.md §C3).  A step = one solve of kernel (a) to the fixpoint from
scratch (both the host-valid and the device-valid phases, all rounds).
Facts = nodes x variables.  Multi-GPU: V-sharded weak scaling -- rank r owns
variables [4096 r, 4096 (r+1)) of the same graph; no collective touches the
data path (variables are independent); timing is the max over
ranks.

The same line carries a `c4` record: configuration C4 (100k independent
functions through the E1 replay kernel, LPT-sharded over the ranks, strong
scaling) with its own value, e2e, per-rank ms, roofline, a parity check and
the reference's own CPU baseline (dartomp analyze_function in a process
pool over a 1,000-function sample of the C4 source batch).
After the timed region the C3 outputs are checked against the CPU oracle on
every variable word (`parity`).

Contract: python bench.py --gpus N --steps K --warmup W  (torchrun for N>1)
prints ONE JSON line on rank 0.  `--impl reference` times the reference path
on the host cores instead: the reference package cannot ingest a CSR graph
(SURVEY §8c), so the reference arm is the C restatement of the same equations
(oracle/mfp_oracle.c, "port"), all host threads, on a bounded column sample.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "dataflow facts/sec to fixpoint (CFG nodes×vars) at 1/2/4/8 B200; %HBM roofline"
UNIT = "facts/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-nodes", type=int, default=1 << 20)
    ap.add_argument("--vars-per-gpu", type=int, default=4096)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0, help="nodes per warp task (0: default)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c3", choices=["c3", "c4"],
                    help="c3: 1M-node x 4096-var CSR fixpoint (default, the roofline "
                         "config); c4: 100k-function E1 batch, LPT-sharded")
    ap.add_argument("--c4-funcs", type=int, default=100_000)
    ap.add_argument("--no-c4", action="store_true",
                    help="skip the C4 sub-record of the default (c3) run")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the C5 sub-record of the default (c3) run")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the post-run parity check of the timed outputs")
    ap.add_argument("--c4-ref-funcs", type=int, default=1000,
                    help="functions in the reference C4 CPU-baseline sample")
    ap.add_argument("--no-sim", action="store_true",
                    help="skip the transfer-simulator (verifier) sub-record")
    ap.add_argument("--sim-funcs", type=int, default=256,
                    help="C4 source functions in the simulator (verifier) record")
    ap.add_argument("--no-emit", action="store_true",
                    help="skip the batched-emission sub-record")
    ap.add_argument("--no-api", action="store_true",
                    help="skip the reference-API record (C1, C2, C4 source through plan_transform)")
    ap.add_argument("--api-funcs", type=int, default=400,
                    help="functions of the C4-style source program in the reference-API record")
    ap.add_argument("--no-cfg", action="store_true",
                    help="skip the north-star CFG-program record (real programs -> CSR -> kernels a+b)")
    ap.add_argument("--cfg-units", type=int, default=80,
                    help="C4 source translation units in the CFG-program record")
    ap.add_argument("--emit-units", type=int, default=48,
                    help="C4 source translation units in the batched-emission record")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DFX_BENCH_SHARE_GPU=1 (testing only): several ranks on one GPU, gloo
    # collectives -- exercises the multi-rank code path on a 1-GPU box
    if os.environ.get("DFX_BENCH_SHARE_GPU"):
        import torch
        local = local % max(1, torch.cuda.device_count())
    return rank, world, local


def workload_config(args, world):
    return {"workload": "C3: single synthetic CFG, %d nodes x %d vars/GPU, avg in-degree 2.5"
                        % (args.n_nodes, args.vars_per_gpu),
            "n_nodes": args.n_nodes, "vars_per_gpu": args.vars_per_gpu,
            "total_vars": args.vars_per_gpu * world, "avg_in_degree": 2.5,
            "kernel_node_frac": 0.2, "access_density": 1 / 32, "scalar_frac": 0.02,
            "seed": args.seed, "parallelism": "V-sharded weak scaling, %d GPU(s)" % world,
            "l2": "no flush needed: inputs+state 2.5 GB/GPU >> 126 MB L2"}


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unparsed"]}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profiles():
    p = ROOT / "profiles" / "roofline_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("dram_bytes_per_launch"), d
    return None, None


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the C restatement on the host cores
# ---------------------------------------------------------------------------
def cpu_sample(args, steps=1):
    sys.path.insert(0, str(ROOT / "tests"))
    import _oracle  # noqa: E402  (cpu_baseline leg: the only bench use of oracle/)
    threads = _oracle.num_threads()
    words = max(4, min(args.vars_per_gpu // 32, 4 * threads))
    n_scalar = int(round(0.02 * args.vars_per_gpu))
    g = _oracle.c3_generate(args.seed, args.n_nodes, 0, words, n_scalar)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        _oracle.c3_solve(g)
        times.append(time.perf_counter() - t0)
    facts = args.n_nodes * words * 32
    t = statistics.median(times)
    return {"value": facts / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": "oracle/mfp_oracle.c Gauss-Seidel solve of the same C3 graph "
                      "(%d nodes), variable columns 0..%d (%d of %d vars; variables are "
                      "independent so the block is an exact sample), median of %d"
                      % (args.n_nodes, words * 32 - 1, words * 32, args.vars_per_gpu, steps),
            "seconds_per_sample": t}, times


def run_reference(args, rank, world):
    if rank != 0:
        return
    base, times = cpu_sample(args, steps=args.warmup + args.steps)
    timed = times[args.warmup:] or times
    t = sum(timed) / len(timed)
    words = int(base["sample"].split("columns 0..")[1].split(" ")[0]) + 1
    facts = args.n_nodes * words
    value = facts / t
    base["value"] = value
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (counter-hash generator, DESIGN.md §C3)",
            "config": workload_config(args, 1), "impl": "reference", "cpu_baseline": base,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    base.update(host_info())
    if not args.no_c4:
        # C4 (the batched-function workload): the reference package itself,
        # analyze_function in a process pool over a fixed sample
        sys.path.insert(0, str(ROOT / "tests"))
        import _c4src  # noqa: E402
        cb = _c4src.reference_c4_baseline(n_funcs=args.c4_ref_funcs)
        line["c4"] = {"metric": METRIC, "value": cb["value"], "unit": UNIT,
                      "impl": "reference", "cpu_baseline": cb,
                      "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}
    emit_line(line)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2406_13881_b200 import _abi
    from paper_2406_13881_b200.csr import (Acc8Session, AccSession, C3Config, CsrProblem, MfpSession,
                                           acc_to_b8,
                                           c3_scalar_mask)

    torch.cuda.set_device(local)
    eng = _abi.engine(local)
    # a dedicated (non-default) stream shared by torch events and the engine
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    eng.lib.dfx_set_stream(eng.h, __import__("ctypes").c_void_p(stream.cuda_stream))
    cfg = C3Config(n_nodes=args.n_nodes, n_vars=args.vars_per_gpu, seed=args.seed,
                   w0=rank * (args.vars_per_gpu // 32))
    prob = CsrProblem.generate_c3(cfg, eng)
    for _ in range(max(3, args.warmup)):
        prob.solve(args.chunk)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    kernel_ms, launches, stats_last = 0.0, 0, None
    barrier()
    # timed region: K solves enqueued back to back (V <= 4096: each solve is
    # two persistent launches that decide convergence on the device, so no
    # host round trip separates the steps), one synchronize at the end
    persistent = cfg.words <= 128
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            if persistent:
                prob.solve_async(args.chunk)
                launches += 2
            else:
                st = prob.solve(args.chunk)
                launches += st.rounds_h + st.rounds_d
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    # per-solve statistics and phase-kernel time from synchronous solves
    for _ in range(5):
        st = prob.solve(args.chunk)
        kernel_ms += st.kernel_ms
    kernel_ms *= args.steps / 5.0
    stats_last = {k: getattr(st, k) for k, _ in st._fields_}
    total_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    facts_total = args.n_nodes * args.vars_per_gpu * world
    value = facts_total / (ms_per_step / 1e3)

    # roofline of the dominant kernel (mfp_round_kernel): algorithmic bytes
    # counted by the kernel itself / its own launch time
    rowb = cfg.words * 4
    nnz = prob.eng.lib.dfx_csr_nnz(prob.h)
    rounds = stats_last["rounds_h"] + stats_last["rounds_d"]
    meta = rounds * (5 * args.n_nodes + 8 * nnz) + 12 * stats_last["evaluated"]
    bytes_per_solve = (stats_last["rows_read"] + stats_last["rows_written"]) * rowb + meta
    kernel_ms_per_solve = kernel_ms / args.steps
    achieved = bytes_per_solve / (kernel_ms_per_solve / 1e3) / 1e9
    peak, peak_src = measured_peak()
    traffic, _ = traffic_from_profiles()
    pattern = None      # practical ceiling of the access pattern (profiles/, microbenchmark)
    pc = ROOT / "profiles" / "r01b_gather_ceiling.json"
    if pc.exists():
        pattern = {r["pattern"]: r["GB_s"] for r in json.loads(pc.read_text())["results"]}
    survey_bytes = stats_last["evaluated"] * args.vars_per_gpu * (11 / 16)

    # kernel (b) once (not part of the fixpoint metric), for the record
    rows = prob.requirements()
    req_ms = prob.stats.req_ms

    # e2e: the reference-facing all-in-one C-ABI calls with pinned host
    # buffers, host<->device copies inside the timed region.  Headline:
    # dfx_mfp_acc -- per-node access lists in (the reference's per-statement
    # MemoryAccess lists), per-node requirement variable lists out.  Beside
    # it: dfx_mfp_csr on dense R/W bitplanes in, compacted mask rows out.
    e2e = None
    if args.e2e_steps > 0:
        def pinned(shape, dtype):
            n = int(np.prod(shape)) * np.dtype(dtype).itemsize
            buf = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            return buf.numpy().view(dtype).reshape(shape)

        def timed(run):
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            d2h = 0
            for _ in range(args.e2e_steps):
                d2h += run().nbytes
            e1.record(stream)
            torch.cuda.synchronize()
            et = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], dtype=torch.float64,
                              device="cuda")
            if world > 1:
                dist.all_reduce(et, op=dist.ReduceOp.MAX)
            return float(et.item()), d2h // args.e2e_steps

        rp, col, kind, R, W = prob.export_inputs(alloc=pinned)
        S = c3_scalar_mask(cfg)
        n_req_bits = int(np.bitwise_count(rows.masks).sum())
        # dense-plane path
        h2d_planes = rp.nbytes + col.nbytes + kind.nbytes + R.nbytes + W.nbytes + S.nbytes
        sess = MfpSession(eng, alloc=pinned)
        out = sess.run(rp, col, kind, R, W, S)                   # warm (allocates)
        assert out.masks.shape[0] == rows.masks.shape[0], "e2e output differs from device run"
        ms_planes, d2h_planes = timed(lambda: sess.run(rp, col, kind, R, W, S))
        del R, W, out, sess
        # uint16 list path
        acc_off, acc = prob.export_acc(alloc=pinned)
        h2d_u16 = rp.nbytes + col.nbytes + kind.nbytes + acc_off.nbytes + acc.nbytes + S.nbytes
        usess = AccSession(eng, alloc=pinned)
        out_u16 = usess.run(rp, col, kind, acc_off, acc, S, cfg.words)   # warm (allocates)
        assert out_u16.vars.shape[0] == n_req_bits, "list output differs from the mask rows"
        ms_u16, d2h_u16 = timed(lambda: usess.run(rp, col, kind, acc_off, acc, S, cfg.words))
        n_acc = int(acc.shape[0])
        # byte-coded list path (headline): the same lists in ~1.2 bytes per
        # entry (include/dfx.h B8), encoded before the timed region like the
        # uint16 lists above
        boff_np, b_np = acc_to_b8(acc_off, acc)
        del acc_off, acc, usess
        boff = pinned(boff_np.shape, np.int32)
        boff[:] = boff_np
        b8in = pinned(b_np.shape, np.uint8)
        b8in[:] = b_np
        del boff_np, b_np
        h2d = rp.nbytes + col.nbytes + kind.nbytes + boff.nbytes + b8in.nbytes + S.nbytes
        asess = Acc8Session(eng, alloc=pinned)
        out8 = asess.run(rp, col, kind, boff, b8in, S, cfg.words)       # warm (allocates)
        ms, d2h = timed(lambda: asess.run(rp, col, kind, boff, b8in, S, cfg.words))
        out = out8.to_lists()
        assert out.vars.shape[0] == n_req_bits, "byte-list output differs from the mask rows"
        # throughput of a stream of problems: two host threads, each with its
        # own handle and buffers, issue complete host-buffer calls; one
        # call's D2H overlaps the other's H2D and solve (full-duplex PCIe)
        two = None
        if args.e2e_steps > 0 and world == 1:
            import threading
            eng2 = _abi.Engine(_abi.load_lib(), local)
            s2 = torch.cuda.Stream()
            eng2.lib.dfx_set_stream(eng2.h, __import__("ctypes").c_void_p(s2.cuda_stream))
            sess2 = Acc8Session(eng2, alloc=pinned)
            sess2.run(rp, col, kind, boff, b8in, S, cfg.words)       # warm
            n_each = max(2, args.e2e_steps)

            def worker(sess_):
                for _ in range(n_each):
                    sess_.run(rp, col, kind, boff, b8in, S, cfg.words)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ths = [threading.Thread(target=worker, args=(x,)) for x in (asess, sess2)]
            for th in ths:
                th.start()
            for th in ths:
                th.join()
            torch.cuda.synchronize()
            ms2 = (time.perf_counter() - t0) * 1e3 / (2 * n_each)
            two = {"value": facts_total / (ms2 / 1e3), "ms_per_problem": ms2,
                   "how": "2 host threads x %d dfx_mfp_acc8 calls, own handles, wall clock" % n_each}
            del sess2
            eng2.close()
        e2e = {"value": facts_total / (ms / 1e3), "unit": UNIT,
               "ms_per_step": ms, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "two_calls_in_flight": two,
               "path": "dfx_mfp_acc8 (pinned host buffers): H2D CSR + per-node access lists "
                       "(byte-coded, include/dfx.h B8), decode to bitplanes, kernels (a)+(b), "
                       "D2H per-node requirement lists (byte-coded) + int32 row offsets",
               "accesses": n_acc, "requirements": int(out.vars.shape[0]),
               "bytes_per_access": float(b8in.nbytes) / max(1, n_acc),
               "bytes_per_requirement": float(out8.bytes.nbytes) / max(1, out.vars.shape[0]),
               "lists_u16_path": {
                   "value": facts_total / (ms_u16 / 1e3), "ms_per_step": ms_u16,
                   "h2d_bytes_per_step": int(h2d_u16), "d2h_bytes_per_step": int(d2h_u16),
                   "path": "dfx_mfp_acc: uint16 access lists in, uint16 requirement lists out"},
               "dense_planes_path": {
                   "value": facts_total / (ms_planes / 1e3), "ms_per_step": ms_planes,
                   "h2d_bytes_per_step": int(h2d_planes), "d2h_bytes_per_step": int(d2h_planes),
                   "path": "dfx_mfp_csr: H2D dense R/W bitplanes, D2H compacted mask rows"}}

    # parity of what was timed (outside the timed region; checker only): the
    # solve's OUT_H / OUT_D planes, kernel (b)'s requirement planes and the
    # e2e call's per-node requirement lists == the CPU oracle on ALL variable
    # words of this rank's slab, block by block
    parity = None
    if not args.no_parity:
        sys.path.insert(0, str(ROOT / "tests"))
        import _oracle  # noqa: E402  (checker)
        t0 = time.perf_counter()
        OH, OD, _ = prob.download(True, True)
        rq, rf = rows.to_planes()
        bad = _oracle.c3_verify(cfg.seed, cfg.n_nodes, cfg.w0, cfg.words, cfg.n_scalar,
                                OH, OD, rq, rf)
        if e2e is not None:
            lq, lf = out.to_planes()
            bad["e2e_lists"] = int(np.count_nonzero(lq != rq) + np.count_nonzero(lf != rf))
            lq, lf = out_u16.to_planes()
            bad["e2e_lists_u16"] = int(np.count_nonzero(lq != rq) + np.count_nonzero(lf != rf))
            del lq, lf
        ok = all(v == 0 for v in bad.values())
        parity = {"status": "ok" if ok else "MISMATCH", "differing_words": bad,
                  "checked": "all %d variable words x %d nodes of this rank's slab vs "
                             "oracle/mfp_oracle.c (block-wise), plus the e2e lists"
                             % (cfg.words, cfg.n_nodes),
                  "check_s": time.perf_counter() - t0}
        del OH, OD, rq, rf
        pt = torch.tensor([0.0 if ok else 1.0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(pt, op=dist.ReduceOp.MAX)
        if float(pt.item()) != 0.0:
            parity["status"] = "MISMATCH"
    req_rec = {"kernel": "requirements_kernel + compact_kernel",
               "ms": req_ms, "nonzero_masks": int(rows.masks.shape[0]),
               "output_bytes": int(rows.nbytes)}
    del rows
    if e2e is not None:
        del out, out8, out_u16, asess
    prob.close()
    c4 = None
    if not args.no_c4:
        c4 = run_c4(args, rank, world, local, sub=True)
    c5 = None
    if not args.no_c5:
        c5 = run_c5(args, rank, world, local)
    sim = None
    if not args.no_sim and world == 1:
        sim = run_sim_record(args)
    emit_rec = None
    if not args.no_emit and world == 1:
        emit_rec = run_emit_record(args)
    api_rec = None
    if not args.no_api and world == 1:
        api_rec = run_api_record(args)
    cfg_rec = None
    if not args.no_cfg and world == 1:
        cfg_rec = run_cfg_record(args)
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (counter-hash generator, DESIGN.md §C3)",
            "parity": parity,
            "config": workload_config(args, world),
            "clocks": clk.summary(),
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "mfp_phase_kernel (kernel a, persistent, all rounds of a phase)",
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_solve": bytes_per_solve,
                         "launches_per_solve": 2 if cfg.words <= 128 else rounds,
                         "rounds_per_solve": rounds,
                         "kernel_ms_per_solve": kernel_ms_per_solve,
                         "survey_formula_frac": survey_bytes / (kernel_ms_per_solve / 1e3) / 1e9 / peak,
                         "access_pattern_ceiling_gbs": pattern},
            "solve": {"rounds_h": stats_last["rounds_h"], "rounds_d": stats_last["rounds_d"],
                      "evaluated_rows": stats_last["evaluated"],
                      "rows_read": stats_last["rows_read"],
                      "rows_written": stats_last["rows_written"],
                      "device_ms_incl_round_checks": ms_per_step},
            "requirements": req_rec}
    if world == 1 and not args.no_cpu_baseline:
        base, _ = cpu_sample(args, steps=1)
        base.update(host_info())
        line["cpu_baseline"] = base
    if c4 is not None:
        line["c4"] = c4
    if c5 is not None:
        line["c5"] = c5
    if sim is not None:
        line["sim"] = sim
    if emit_rec is not None:
        line["emit"] = emit_rec
    if api_rec is not None:
        line["api"] = api_rec
    if cfg_rec is not None:
        line["cfg"] = cfg_rec
    emit_line(line)


def run_cfg_record(args):
    """The north-star path on real programs (cfgprog.py): --cfg-units C4
    source translation units, parsed by the reference's front end (untimed),
    lowered into ONE block-diagonal CSR over their AST-CFGs with per-node
    access lists (host Python, timed and reported), solved by kernels (a)+(b)
    in one `dfx_mfp_acc` call with host buffers (timed: H2D, expansion,
    fixpoint, requirements, D2H).  Parity: fixpoint planes and requirement
    lists == oracle/mfp_oracle.c on the same problem."""
    from paper_2406_13881_b200._host import have_dartomp
    if not have_dartomp():
        return {"unavailable": "host front end (dartomp) not importable"}
    import numpy as np
    from dartomp.pipeline import load
    from paper_2406_13881_b200.cfgprog import fixpoint_planes, lower_program, solve_program
    from paper_2406_13881_b200.csr import AccSession
    from paper_2406_13881_b200.gen.c4src import C4SourceConfig, c4_source
    sys.path.insert(0, str(ROOT / "tests"))
    import _oracle  # noqa: E402  (the checker)
    n = args.cfg_units
    items = []
    for k in range(n):
        a = load(text=c4_source(C4SourceConfig(), k * (100_000 // max(1, n))))
        items += [(nm, a.src, a.cfgs[nm], a.accesses[nm], a.table) for nm in a.cfgs]
    t0 = time.perf_counter()
    prog = lower_program(items)
    lower_s = time.perf_counter() - t0
    sess = AccSession()
    solve_program(prog, sess)                              # warm
    ts, ks = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        reqs, st = solve_program(prog, sess)
        ts.append(time.perf_counter() - t0)
        ks.append(float(st.kernel_ms))
    call_s = statistics.median(ts)
    # parity: planes of the C restatement on the same problem
    acc = prog.acc.astype(np.int64)
    node = np.repeat(np.arange(prog.n_nodes), np.diff(prog.acc_off))

    def plane(mask):
        bits = np.zeros((prog.n_nodes, prog.words * 32), dtype=np.uint8)
        sel = (acc >> 14) & mask != 0
        bits[node[sel], (acc & 0x3FFF)[sel]] = 1
        return np.packbits(bits, axis=1, bitorder="little").view(np.uint32).reshape(
            prog.n_nodes, prog.words).copy()
    R, W = plane(1), plane(2)
    g = {"row_ptr": prog.row_ptr, "col": prog.col, "kind": prog.kind, "A": R | W, "B": W,
         "USE": R, "S": prog.S}
    OH, OD, _ = _oracle.c3_solve(g)
    REQ, FP = _oracle.c3_requirements(g, OH, OD)
    gh, gd = fixpoint_planes(prog)
    rl = sess.run(prog.row_ptr, prog.col, prog.kind, prog.acc_off, prog.acc, prog.S, prog.words)
    rq, fp = rl.to_planes()
    ok = (np.array_equal(gh, OH) and np.array_equal(gd, OD) and np.array_equal(rq, REQ)
          and np.array_equal(fp, FP))
    supported = sum(f.status == "ok" for f in prog.fns)
    facts = prog.facts
    return {"workload": "%d C4 source translation units (gen/c4src.py, every %d-th of 100k), "
                        "%d functions lowered into one CSR over their AST-CFGs"
                        % (n, 100_000 // max(1, n), len(prog.fns)),
            "unit": "facts/s (CFG nodes x variables, to fixpoint, + requirements)",
            "functions": len(prog.fns), "supported": supported,
            "nodes": prog.n_nodes, "edges": int(prog.col.shape[0]),
            "words": prog.words, "accesses": int(prog.acc.shape[0]), "facts": facts,
            "value": facts / call_s,
            "call_ms": 1e3 * call_s, "kernel_ms": statistics.median(ks),
            "h2d_bytes": int(prog.row_ptr.nbytes + prog.col.nbytes + prog.kind.nbytes
                             + prog.acc_off.nbytes + prog.acc.nbytes + prog.S.nbytes),
            "host_lowering_s": lower_s,
            "requirements": int(rl.vars.shape[0]),
            "parity": {"status": "ok" if ok else "MISMATCH",
                       "checked": "fixpoint planes (H, D) and requirement / firstprivate "
                                  "planes == oracle/mfp_oracle.c on the same problem"},
            "path": "cfgprog.lower_program -> solve_program -> dfx_mfp_acc (one call)"}


def run_api_record(args):
    """The drop-in at the reference's own API (`dartomp.pipeline`), beside
    the reference on the same source, same process, one core each:
      c1  Listing 1 (SPEC motivating example): transform text + report lines
          identical to the reference's (parity only, BASELINE configs[0]);
      c2  LULESH-shaped program (BASELINE configs[1]): load, plan_transform
          and apply_plans timed (medians), output byte-identical;
      c4_source  a C4-style program of --api-funcs structured functions:
          plan_transform timed on the same parsed unit, plans identical
          (anchor identity included).
    The front end (lexer, parser, AST-CFG, access classification) is the
    reference's on both sides; the drop-in swaps the analysis (E1, kernel c)
    and the emitter."""
    from paper_2406_13881_b200._host import have_dartomp
    if not have_dartomp():
        return {"unavailable": "host front end (dartomp) not importable"}
    import dartomp.pipeline as ref
    from dartomp.report import plan_lines as ref_lines
    from dartomp.rewriter import apply_plans as ref_apply
    from paper_2406_13881_b200 import pipeline as eng
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    from paper_2406_13881_b200.gen.lulesh import generate_lulesh

    def med(fn, reps):
        ts, out = [], None
        for _ in range(reps):
            t0 = time.perf_counter()
            out = fn()
            ts.append(1e3 * (time.perf_counter() - t0))
        return statistics.median(ts), out

    def pipeline_run(mod, apply, text, reps):
        parts = {"load": [], "plan": [], "total": []}
        out = None
        for _ in range(reps):
            t0 = time.perf_counter()
            a = mod.load(text=text)
            t1 = time.perf_counter()
            plans = mod.plan_transform(a)
            t2 = time.perf_counter()
            out = apply(a.src, plans)
            t3 = time.perf_counter()
            parts["load"].append(1e3 * (t1 - t0))
            parts["plan"].append(1e3 * (t2 - t1))
            parts["total"].append(1e3 * (t3 - t0))
        return {k: statistics.median(v) for k, v in parts.items()}, out

    rec = {"what": "the drop-in (paper_2406_13881_b200.pipeline) vs the reference "
                   "(dartomp.pipeline) on the same source, same process, one core each"}
    # C1: Listing 1
    c1 = ROOT / "tests" / "golden" / "corpus" / "transform" / "listing1.c"
    text = c1.read_text()
    ar, ae = ref.load(text=text, path=str(c1)), eng.load(text=text, path=str(c1))
    pr, pe = ref.plan_transform(ar), eng.plan_transform(ae)
    rr, re_ = ref_apply(ar.src, pr), eng.apply_plans(ae.src, pe)
    rec["c1"] = {"workload": "C1: SPEC Listing 1 (tests/golden/corpus/transform/listing1.c)",
                 "identical_output": rr.text == re_.text,
                 "identical_report": ref_lines(ar.src, pr) == eng.plan_lines(ae.src, pe),
                 "report": eng.plan_lines(ae.src, pe)}
    # C2: LULESH-shaped
    text = generate_lulesh(seed=1)
    pipeline_run(eng, eng.apply_plans, text, 2)                # warm the engine
    pipeline_run(ref, ref_apply, text, 1)
    # interleaved, so drift in the host's speed lands on both sides
    runs_ref, runs_eng = [], []
    for _ in range(15):
        runs_ref.append(pipeline_run(ref, ref_apply, text, 1))
        runs_eng.append(pipeline_run(eng, eng.apply_plans, text, 1))
    o_ref, o_eng = runs_ref[-1][1], runs_eng[-1][1]
    r_ref = {k: statistics.median(r[0][k] for r in runs_ref) for k in runs_ref[0][0]}
    r_eng = {k: statistics.median(r[0][k] for r in runs_eng) for k in runs_eng[0][0]}
    rec["c2"] = {"workload": "C2: LULESH-shaped program (gen/lulesh.py seed 1), %d lines"
                             % len(text.splitlines()),
                 "reference_ms": r_ref, "dropin_ms": r_eng,
                 "speedup_plan": r_ref["plan"] / r_eng["plan"],
                 "speedup_total": r_ref["total"] / r_eng["total"],
                 "identical_output": o_ref.text == o_eng.text}
    # C4-style functions from C source at the reference API
    n = args.api_funcs
    text = generate(7, GenConfig(n_funcs=n, n_globals=24, n_stmts=40, p_kernel=0.3))
    # the front end at scale: the reference `load` against the
    # drop-in's (its parser and the paused collector), one run each
    t0 = time.perf_counter()
    a = ref.load(text=text)
    t_load_ref = 1e3 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    a_eng = eng.load(text=text)
    t_load_eng = 1e3 * (time.perf_counter() - t0)
    same_units = (list(a_eng.cfgs) == list(a.cfgs)
                  and sum(len(v) for v in a_eng.accesses.values())
                  == sum(len(v) for v in a.accesses.values()))
    del a_eng
    eng.plan_transform(a)                                      # warm
    t_ref, p_ref = med(lambda: ref.plan_transform(a), 2)
    t_eng, p_eng = med(lambda: eng.plan_transform(a), 3)

    def key(plans):
        return [(id(p.function), [(u.kind, u.names, id(u.anchor), u.position) for u in p.all_plans],
                 (id(p.region.begin), p.region.clause_text()) if p.region is not None else None,
                 tuple(p.suppressed)) for p in plans]
    rec["c4_source"] = {"workload": "%d structured functions from C source (gen/cprog.py seed 7), "
                                    "%d lines" % (len(a.cfgs), len(text.splitlines())),
                        "reference_plan_transform_ms": t_ref, "dropin_plan_transform_ms": t_eng,
                        "speedup": t_ref / t_eng, "identical_plans": key(p_ref) == key(p_eng),
                        "load": {"reference_ms": t_load_ref, "dropin_ms": t_load_eng,
                                 "speedup": t_load_ref / t_load_eng,
                                 "same_functions_and_accesses": same_units},
                        "lowering_workers": int(os.environ.get("DFX_LOWER_WORKERS", "0"))
                        or min(16, os.cpu_count() or 1)}
    rec.update(host_info())
    return rec


def run_emit_record(args):
    """Batched emission: C4 source translation units, planned
    by the drop-in (E1), then rewritten text + report lines by the native
    emitter in one call (`dfx_emit_batch`) beside the reference's
    `rewriter.apply_plans` + `report.plan_lines` on the same plans; outputs
    compared byte for byte."""
    from paper_2406_13881_b200._host import have_dartomp
    if not have_dartomp():
        return {"unavailable": "host front end (dartomp) not importable"}
    from dartomp.report import plan_lines as ref_lines
    from dartomp.rewriter import apply_plans as ref_apply
    from paper_2406_13881_b200 import emit, pipeline
    from paper_2406_13881_b200.gen.c4src import C4SourceConfig, c4_source
    n = args.emit_units
    units = []
    for k in range(n):
        a = pipeline.load(text=c4_source(C4SourceConfig(), k * (100_000 // max(1, n))))
        units.append((a.src, pipeline.plan_transform(a)))

    def ref_all():
        out = []
        for src, plans in units:
            r = ref_apply(src, plans)
            try:
                ln = ref_lines(src, plans)
            except KeyError as e:
                ln = e
            out.append((r.text, ln))
        return out

    def nat_all():
        return [(r.text, ln) for r, ln in emit.emit_batch([(s, p, None) for s, p in units])]

    def timed(fn, reps=5):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            out = fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts), out
    tr, ro = timed(ref_all, 3)
    tn, no = timed(nat_all)
    same = all(a[0] == b[0] and (a[1] == b[1] or (isinstance(a[1], KeyError) and isinstance(b[1], KeyError)))
               for a, b in zip(ro, no))
    plans = sum(len(p.all_plans) for _, ps in units for p in ps)
    chars = sum(len(s.text) for s, _ in units)
    return {"workload": "%d C4 source translation units (gen/c4src.py, every %d-th of 100k): "
                        "%d plans, %d source characters" % (n, 100_000 // max(1, n), plans, chars),
            "unit": "translation units emitted/s (rewritten text + report lines)",
            "value": n / tn, "ms": 1e3 * tn,
            "reference": {"value": n / tr, "ms": 1e3 * tr, "cores": 1,
                          "what": "dartomp rewriter.apply_plans + report.plan_lines, same plans"},
            "identical": same,
            "path": "emit.emit_batch -> dfx_emit_batch (csrc/emit.cpp), one native call"}


def run_sim_record(args):
    """Transfer simulator as a batched verifier: C4 source
    functions, transformed (annotated mode) and original (implicit mode),
    simulated in ONE `dfx_sim_batch` launch; beside it the reference
    `simulate` (simulator.py:708) on the same programs in a process pool.
    Host preparation (parse, transform) is untimed; the host lowering is
    timed and reported.  Parity: every program's totals, aggregated stale
    reads, warnings and final reference counts equal the reference's."""
    import multiprocessing as mp
    from paper_2406_13881_b200._host import have_dartomp
    if not have_dartomp():
        return {"unavailable": "host front end (dartomp) not importable"}
    sys.path.insert(0, str(ROOT / "scripts"))
    sys.path.insert(0, str(ROOT / "tests"))
    import sim_worker  # noqa: E402
    import _sim  # noqa: E402  (aggregate view of a SimReport, for the parity check)
    from paper_2406_13881_b200.simulator import _report, run_sim
    procs = len(os.sched_getaffinity(0))
    n = args.sim_funcs
    jobs = [(k * (100_000 // max(1, n)), mode) for k in range(n) for mode in ("annotated", "implicit")]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(procs) as pool:
        rows = pool.map(sim_worker.one, jobs, chunksize=2)
    prep_wall = time.perf_counter() - t0
    progs = [r[1] for r in rows]
    lower_cpu = sum(r[3] for r in rows)
    ref_cpu = sum(r[4] for r in rows)
    for _ in range(3):
        raw = run_sim(progs)
    ks, es = [], []
    for _ in range(max(3, min(args.steps, 10))):
        t1 = time.perf_counter()
        raw = run_sim(progs)
        es.append(time.perf_counter() - t1)
        ks.append(raw.kernel_ms)
    # parity, program by program
    import numpy as np
    order = np.argsort(raw.recs["prog"], kind="stable")
    recs = raw.recs[order]
    bounds = np.searchsorted(recs["prog"], np.arange(len(progs) + 1))
    bad, stale_ann, var_off = 0, 0, 0
    for i, (p, row) in enumerate(zip(progs, rows)):
        rep = _report(p, raw.vars[var_off:var_off + p.n_vars], recs[bounds[i]:bounds[i + 1]])
        var_off += p.n_vars
        bad += _sim.aggregate_fields(rep) != row[2]
        if p.mode == "annotated":
            stale_ann += rep.log.stale_count
    nprog = len(progs)
    kms, ems = statistics.median(ks), 1e3 * statistics.median(es)
    # the 512-program launch is bound by its longest program's warps (a
    # critical path, ~9.9 ms); a batch of the same programs 16 times over
    # shows the kernel's throughput at batch scale
    rep = 16
    big = progs * rep
    run_sim(big)
    kb = statistics.median([run_sim(big).kernel_ms for _ in range(3)])
    ops = int(sum(p.ops.shape[0] for p in progs))
    return {"workload": "C4 source functions (gen/c4src.py, every %d-th of 100k): %d transformed "
                        "(annotated) + %d original (implicit) programs" % (100_000 // max(1, n), n, n),
            "unit": "programs simulated/s", "programs": nprog, "ops": ops,
            "vars": int(sum(p.n_vars for p in progs)),
            "value": nprog / (kms / 1e3), "kernel_ms": kms,
            "batch_scale": {"programs": nprog * rep, "kernel_ms": kb,
                            "value": nprog * rep / (kb / 1e3),
                            "what": "the same programs %d times over in one launch" % rep},
            "e2e": {"value": nprog / (ems / 1e3), "ms": ems,
                    "path": "dfx_sim_batch with host buffers (H2D programs, kernel, D2H per-variable "
                            "totals + records)"},
            "host_lowering": {"cpu_s": lower_cpu, "programs_per_s_per_core": nprog / lower_cpu},
            "parity": {"status": "ok" if bad == 0 else "MISMATCH", "mismatched_programs": bad,
                       "checked": "every program: totals, stale reads per (line, var, space), "
                                  "warnings, final ref counts == reference simulate"},
            "stale_reads_in_transformed_programs": int(stale_ann),
            "cpu_baseline": {"value": nprog / (ref_cpu / procs), "unit": "programs simulated/s",
                             "cores": procs, "kind": "reference",
                             "sample": "reference dartomp simulate (simulator.py:708) on the same "
                                       "%d programs, multiprocessing.Pool(%d), parse excluded; "
                                       "aggregate = programs / (CPU seconds / cores)" % (nprog, procs),
                             "cpu_s": ref_cpu, **host_info()},
            "prep_wall_s": prep_wall}


def host_info() -> dict:
    sys.path.insert(0, str(ROOT / "tests"))
    import _c4src  # noqa: E402
    return _c4src.host_info()


def c4_issue_profile():
    """Warp instructions per replay launch of the C4 batch, from the ncu
    capture committed under profiles/ (sm__inst_executed.sum)."""
    p = ROOT / "profiles" / "c4_issue.json"
    if p.exists():
        return json.loads(p.read_text())
    return None


def run_c4(args, rank, world, local, sub=False):
    """Configuration C4: 100k independent functions through the E1 replay
    kernel, LPT-sharded over the ranks (strong scaling: total work fixed).
    sub=True: returns the record (the `c4` object of the default run's line)
    instead of printing a line."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2406_13881_b200 import _abi
    from paper_2406_13881_b200.batch import (C4Config, ReplayBatch, c4_cost, c4_generate,
                                             c4_shapes, lpt_shards, program_visits)
    from paper_2406_13881_b200.dataflow import ReplaySession, pack_ops, run_replay

    torch.cuda.set_device(local)
    eng = _abi.engine(local)
    # a dedicated (non-default) stream shared by torch events and the engine
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    eng.lib.dfx_set_stream(eng.h, __import__("ctypes").c_void_p(stream.cuda_stream))
    cfg = C4Config(n_funcs=args.c4_funcs, seed=args.seed)
    N, V = c4_shapes(cfg)
    shards = lpt_shards(c4_cost(N, V), world)
    mine = shards[rank]

    def pinned(shape, dtype):
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        buf = torch.empty(max(1, n), dtype=torch.uint8, pin_memory=True)
        return buf.numpy()[:n].view(dtype).reshape(shape)

    batch, facts_mine = c4_generate(cfg, mine, alloc=pinned)
    facts_total = int((N.astype(np.int64) * V).sum())
    # fact-visits (SURVEY §8 d, E1): dynamic node visits x V_f, node visits
    # scaled from the program's dynamic/static op ratio (loops run twice)
    visits = program_visits(batch)
    n_ops = batch.fns["n_ops"].astype(np.float64)
    fact_visits_mine = float((visits / np.maximum(n_ops, 1) * N[mine] * V[mine]).sum())
    rb = ReplayBatch(batch, eng=eng)
    for _ in range(max(3, args.warmup)):
        rb.run()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def all_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world == 1:
            return [x]
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [float(o.item()) for o in out]

    barrier()
    kernel_ms = 0.0
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            n_ev, kms = rb.run()
            kernel_ms += kms
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    my_ms = ev0.elapsed_time(ev1) / args.steps
    per_rank_ms = all_ranks(my_ms)
    ms_per_step = max(per_rank_ms)
    value = facts_total / (ms_per_step / 1e3)
    kernel_ms_step = kernel_ms / args.steps
    fv_total = sum(all_ranks(fact_visits_mine))
    rb.close()
    # e2e: the host-buffer C-ABI call (dfx_replay_batch: H2D, kernel, D2H)
    e2e = None
    if args.e2e_steps > 0:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        sess = ReplaySession(eng, alloc=pinned, event_cap=rb.cap)

        def e2e_run(packed_ops=None):
            sess.run(batch, packed_ops)                   # warm (allocates)
            barrier()
            d2h = 0
            e0.record(stream)
            for _ in range(args.e2e_steps):
                raw = sess.run(batch, packed_ops)
                d2h += raw.events.nbytes + raw.var_out.nbytes
            e1.record(stream)
            torch.cuda.synchronize()
            return max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps), d2h // args.e2e_steps
        et16, d2h16 = e2e_run()
        h2d_rest = sum(a.nbytes for a in (batch.fns, batch.var_flags, batch.stmt_span,
                                          batch.sites, batch.arms))
        # headline: the ops in the 8-byte form (dfx_replay_batch_packed), packed
        # before the timed region like the rest of the program arrays
        pk_np = pack_ops(batch.ops)
        packed = pk_np is not None
        if packed:
            pk = pinned(pk_np.shape, np.uint32)
            pk[:] = pk_np
            del pk_np
            et, d2h = e2e_run(pk)
            h2d = h2d_rest + pk.nbytes
        else:
            et, d2h, h2d = et16, d2h16, h2d_rest + batch.ops.nbytes
        e2e = {"value": facts_total / (et / 1e3), "unit": UNIT,
               "ms_per_step": et, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "path": "dfx_replay_batch%s (pinned host buffers): H2D programs in 32 function "
                       "ranges (copy stream), %sregion tables per range (2 streams), one "
                       "persistent E1 launch whose items wait for their range, D2H events per "
                       "range as it completes (D2H stream)"
                       % (("_packed", "ops in 8 bytes unpacked on the device and ")
                          if packed else ("", "")),
               "ops_16_byte_path": {"value": facts_total / (et16 / 1e3), "ms_per_step": et16,
                                    "h2d_bytes_per_step": int(h2d_rest + batch.ops.nbytes),
                                    "path": "dfx_replay_batch: ops in the 16-byte form"}}
        del sess
    # parity of the engine on this batch: a fixed sample of the same
    # functions through the host-buffer call == the CPU oracle (checker)
    parity = None
    if not args.no_parity and rank == 0:
        sys.path.insert(0, str(ROOT / "tests"))
        import _golden  # noqa: E402
        import _oracle  # noqa: E402  (checker)
        samp = mine[:: max(1, len(mine) // 1000)][:1000]
        sb, _ = c4_generate(cfg, samp)
        exp = run_replay(sb, runner=_oracle.replay_runner_mt)
        got = run_replay(sb)
        try:
            _golden.assert_raw_equal(got.events, got.var_out, exp.events, exp.var_out)
            st = "ok"
        except AssertionError as e:
            st = "MISMATCH: %s" % str(e)[:200]
        parity = {"status": st, "checked": "%d functions of this batch (every %d-th of rank 0's "
                                           "shard): events + per-variable bits == "
                                           "oracle/replay_oracle.c" % (len(samp), max(1, len(mine) // 1000))}
    peak, peak_src = measured_peak()
    alg_bytes = 1.125 * fv_total
    prof = c4_issue_profile()
    issue = None
    if prof is not None and world == 1 and prof.get("n_funcs") == cfg.n_funcs:
        clock = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
        peak_issue = 148 * 4 * clock               # warp instructions / s (4 schedulers / SM)
        inst = float(prof["inst_per_launch"])
        issue = {"achieved_warp_inst_per_s": inst / (kernel_ms_step / 1e3),
                 "peak_warp_inst_per_s": peak_issue,
                 "frac": inst / (kernel_ms_step / 1e3) / peak_issue,
                 "inst_per_launch": inst, "source": prof.get("source")}
    rec = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "ms_per_step": ms_per_step, "per_rank_ms": per_rank_ms,
           "higher_is_better": True, "scaling": "strong",
           "config": {"workload": "C4: batch of %d independent functions, 64-2048 nodes, "
                                  "32-512 vars, LPT-sharded" % cfg.n_funcs,
                      "functions": cfg.n_funcs, "facts_total": facts_total,
                      "parallelism": "function-sharded (LPT), %d GPU(s)" % world,
                      "l2": "programs %.1f GB > 126 MB L2" % (batch.ops.nbytes / 1e9)},
           "data": "synthetic (dfx_gen_c4 structured-program generator; C source form: "
                   "gen/c4src.py, pinned to the reference by tests/test_c4_source.py)",
           "clocks": clk.summary(), "e2e": e2e, "gpu_launches": 2 * args.steps,
           "parity": parity,
           "roofline": {"bound": "issue", "kernel": "replay_kernel (E1)",
                        "hbm_equivalent": {"achieved": alg_bytes / (kernel_ms_step / 1e3) / 1e9,
                                           "peak": peak, "unit": "GB/s",
                                           "frac": alg_bytes / (kernel_ms_step / 1e3) / 1e9 / peak,
                                           "algorithmic_bytes_per_step": alg_bytes,
                                           "fact_visits_per_step": fv_total,
                                           "bytes_per_fact_visit": 1.125,
                                           "peak_source": peak_src},
                        "issue": issue},
           "replay": {"kernel": "replay_kernel", "launches_per_step": ["region_kernel",
                                                                      "replay_kernel"],
                      "kernel_ms_per_step": kernel_ms_step,
                      "events": n_ev, "functions_rank0": int(len(mine)),
                      "ops_rank0": int(batch.ops.shape[0]),
                      "dynamic_over_static_ops": float(visits.sum() / max(1.0, n_ops.sum()))}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, str(ROOT / "tests"))
        import _c4src  # noqa: E402  (cpu_baseline leg: the reference itself)
        rec["cpu_baseline"] = _c4src.reference_c4_baseline(n_funcs=args.c4_ref_funcs)
        rec["cpu_baseline"]["extrapolated_full_batch_s"] = facts_total / rec["cpu_baseline"]["value"]
    if sub:
        return rec if rank == 0 else None
    if rank != 0:
        return None
    rec.update({"warmup": args.warmup, "vs_baseline": None, "dtype": "u32"})
    emit_line(rec)
    return None


def run_c5(args, rank, world, local):
    """Configuration C5 record: the 10k-function call graph (gen/c5.py)
    through kernel (c) -- the single-launch solve (`dfx_summaries`) and the
    component-sharded solve over the ranks' NCCL communicator
    (`dfx_summaries_sharded`: one all-reduce per pass + one all-gather) --
    and, at one rank, the reference's own summarize_all on the same-shaped C
    program (gen/callgraph.py, 10k functions; front end untimed) beside the
    drop-in summarize_all on the same parse, with an identity check."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2406_13881_b200.distributed import ComponentSummaries
    from paper_2406_13881_b200.gen.c5 import generate_c5
    from paper_2406_13881_b200.interproc import solve_call_graph

    torch.cuda.set_device(local)
    g = generate_c5(seed=0, n_funcs=10_000)
    for _ in range(3):
        r = solve_call_graph(g)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        r = solve_call_graph(g)
        ts.append(time.perf_counter() - t0)
    nf, ns = g.init_bits.shape
    if world > 1 and os.environ.get("DFX_BENCH_SHARE_GPU"):
        # ranks sharing one GPU (the 2-rank rehearsal on a 1-GPU box): NCCL
        # refuses two ranks on one device, so the sharded solve is not run
        sharded = {"skipped": "ranks share one GPU (DFX_BENCH_SHARE_GPU); NCCL needs one GPU per rank"}
        cs = None
    else:
        cs = ComponentSummaries(g, rank, world)
        cs.solve()
        tc = []
        for _ in range(5):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            bits, lst, ln, passes = cs.solve()
            tc.append(time.perf_counter() - t0)
        same = bool(np.array_equal(bits, r.bits) and np.array_equal(ln, r.len) and passes == r.passes)
        t = torch.tensor([statistics.median(tc)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sharded = {"value": nf * ns / float(t.item()), "ranks": world,
                   "call_ms_max_over_ranks": 1e3 * float(t.item()),
                   "collectives_per_solve": cs.collectives, "passes": passes,
                   "equal_to_single_launch": same,
                   "path": "dfx_summaries_sharded over the handle's NCCL "
                           "communicator (dfx_comm_init)"}
    rec = {"workload": "C5: %d functions, depth-12 chains, 10%% back edges, %d globals"
                       % (nf, ns - g.n_params),
           "unit": "summary facts/s (functions x slots per solve)",
           "single_launch": {"value": nf * ns / statistics.median(ts), "passes": r.passes,
                             "device_ms": r.kernel_ms, "call_ms": 1e3 * statistics.median(ts),
                             "path": "dfx_summaries: all passes and waves in one cooperative launch"},
           "component_sharded": sharded}
    if cs is not None:
        cs.close()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from paper_2406_13881_b200._host import have_dartomp
        if have_dartomp():
            rec["reference"] = c5_reference_compare()
    return rec if rank == 0 else None


def c5_reference_compare(n_funcs=10_000):
    """The reference's summarize_all (interproc.py:90-144) and the drop-in
    on one parse of the same C program (front end untimed)."""
    from paper_2406_13881_b200._host import import_dartomp
    import_dartomp()
    from dartomp.access import VariableTable, classify_accesses
    from dartomp.astcfg import build_astcfg
    from dartomp.interproc import summarize_all as ref_summarize_all
    from dartomp.lexer import expand_defines
    from dartomp.nodes import defined_functions
    from dartomp.parser import parse
    from dartomp.source import SourceFile
    from paper_2406_13881_b200.gen.callgraph import CallGraphConfig, generate
    from paper_2406_13881_b200.interproc import summarize_all as our_summarize_all
    text = generate(7, CallGraphConfig(n_funcs=n_funcs))
    src = SourceFile.from_text(text, path="c5.c")
    pre = expand_defines(src)
    tu, _ = parse(src, pre)
    table = VariableTable(src, tu)
    cfgs, raw = {}, {}
    for name, fn in defined_functions(tu).items():
        cfgs[name] = build_astcfg(src, fn)
        raw[name] = classify_accesses(src, cfgs[name], table)
    t0 = time.perf_counter()
    ref = ref_summarize_all(src, tu, cfgs, raw, table)
    t_ref = time.perf_counter() - t0
    our_summarize_all(src, tu, cfgs, raw, table)                 # warm
    t0 = time.perf_counter()
    ours = our_summarize_all(src, tu, cfgs, raw, table)
    t_ours = time.perf_counter() - t0
    same = list(ref) == list(ours) and all(
        list(ref[k].param_effects.items()) == list(ours[k].param_effects.items())
        and list(ref[k].global_effects.items()) == list(ours[k].global_effects.items())
        for k in ref)
    return {"workload": "C5 from C source: %d defined functions (gen/callgraph.py seed 7)" % len(cfgs),
            "reference_summarize_all_ms": 1e3 * t_ref, "dropin_summarize_all_ms": 1e3 * t_ours,
            "speedup": t_ref / t_ours, "identical_summaries_and_dict_order": bool(same),
            "cpu_baseline": {"kind": "reference", "cores": 1,
                             "sample": "the full program, one process (its passes are sequential)"},
            **host_info()}


_JSON_OUT = None


def host_cpu() -> dict:
    """The host the CPU baselines ran on: os.cpu_count(),
    the affinity set the process may use, the /proc/cpuinfo model name."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"os_cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "cpu_model": model}


def _tag_cpu_baselines(rec, host) -> None:
    if isinstance(rec, dict):
        for k, v in rec.items():
            if k == "cpu_baseline" and isinstance(v, dict) and "unavailable" not in v:
                for hk, hv in host.items():
                    v.setdefault(hk, hv)
            else:
                _tag_cpu_baselines(v, host)
    elif isinstance(rec, list):
        for v in rec:
            _tag_cpu_baselines(v, host)


def emit_line(rec) -> None:
    """The run's one JSON line, on the process's real stdout (see main).
    Every cpu_baseline record carries the host description."""
    _tag_cpu_baselines(rec, host_cpu())
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(rec) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # stdout carries exactly one JSON line: native libraries (NCCL prints its
    # version at communicator init) write to fd 1 directly, so fd 1 is pointed
    # at stderr for the run and the line goes to a private copy of stdout
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse_args()
    rank, world, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("gloo" if os.environ.get("DFX_BENCH_SHARE_GPU") else "nccl")
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        elif args.workload == "c4":
            run_c4(args, rank, world, local)
        else:
            run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
