"""Transfer-simulator checking helpers (TEST INFRASTRUCTURE).

`oracle_report(prog)` runs oracle/sim_oracle.c (the reference's global
schedule restated over a lowered program) and rebuilds the reference's exact
`SimReport` (event log, stale-read log, warnings in order, final reference
counts).  `reference_fields` / `aggregate_fields` reduce reports to what the
CUDA simulator reproduces (paper_2406_13881_b200/simulator.py docstring).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

import _oracle
from paper_2406_13881_b200._host import import_dartomp

import_dartomp()
from dartomp.access import Space  # noqa: E402
from dartomp.simulator import SimReport, StaleRead, TransferEvent, TransferLog  # noqa: E402

_SPACE = {0: Space.HOST.value, 1: Space.DEVICE.value}


def _p(a):
    return C.c_void_p(a.ctypes.data)


def oracle_report(prog) -> SimReport:
    L = _oracle.lib()
    L.oracle_sim_run.restype = C.c_int
    n_ops = prog.ops.shape[0]
    n_vars = max(1, prog.n_vars)
    cap_ev = cap_st = 1 << 12
    while True:
        ev = np.zeros(3 * cap_ev, dtype=np.int64)
        st = np.zeros(4 * cap_st, dtype=np.int64)
        warn = np.zeros(len(prog.warnings) + 1, dtype=np.int32)
        order = np.zeros(n_vars, dtype=np.int32)
        ref = np.zeros(n_vars, dtype=np.int64)
        hv = np.zeros(n_vars, dtype=np.uint8)
        dv = np.zeros(n_vars, dtype=np.uint8)
        n_ev, n_st = C.c_int64(0), C.c_int64(0)
        n_warn, n_order = C.c_int32(0), C.c_int32(0)
        ops = np.ascontiguousarray(prog.ops, dtype=np.int32)
        a64 = np.ascontiguousarray(prog.arg64, dtype=np.int64)
        oev = np.ascontiguousarray(prog.op_ev, dtype=np.int32)
        rc = L.oracle_sim_run(_p(ops), _p(a64), _p(oev), C.c_int32(n_ops), C.c_int32(prog.n_vars),
                              C.c_int32(len(prog.warnings)), _p(ev), C.c_int64(cap_ev), C.byref(n_ev),
                              _p(st), C.c_int64(cap_st), C.byref(n_st), _p(warn), C.byref(n_warn),
                              _p(order), C.byref(n_order), _p(ref), _p(hv), _p(dv))
        if rc == -3:
            cap_ev, cap_st = max(cap_ev, n_ev.value), max(cap_st, n_st.value)
            continue
        assert rc == 0, "oracle_sim_run failed (%d)" % rc
        break
    events = []
    for d, e, cnt in ev[:3 * n_ev.value].reshape(-1, 3).tolist():
        name, nbytes, line = prog.events[e]
        events.append(TransferEvent("htod" if d == 0 else "dtoh", name, nbytes, line, cnt))
    stale = [StaleRead(prog.var_names[v], _SPACE[sp], prog.sites[site], cnt)
             for v, sp, site, cnt in st[:4 * n_st.value].reshape(-1, 4).tolist()]
    warnings = [prog.warnings[k] for k in warn[:n_warn.value].tolist()]
    refs = {}
    for v in order[:n_order.value].tolist():
        if ref[v]:
            refs[prog.var_names[v]] = int(ref[v])
    return SimReport(prog.mode, list(prog.entries), TransferLog(events, stale), warnings, refs)


def exact_fields(rep: SimReport):
    """Everything of a report, in order (oracle vs reference)."""
    log = rep.log
    return (rep.mode, list(rep.entries),
            [(e.direction, e.var, e.bytes_per_call, e.line, e.count) for e in log.events],
            [(s.var, s.space, s.line, s.count) for s in log.stale_reads],
            list(rep.warnings), dict(rep.final_refs))


def aggregate_fields(rep: SimReport):
    """What the CUDA simulator reproduces: totals, stale reads aggregated per
    (line, variable, space), warnings as a set, final reference counts."""
    log = rep.log
    agg = {}
    for s in log.stale_reads:
        k = (s.line, s.var, s.space)
        agg[k] = agg.get(k, 0) + s.count
    return (rep.mode, list(rep.entries), log.htod_calls, log.htod_bytes, log.dtoh_calls,
            log.dtoh_bytes, log.stale_count, sorted(agg.items()), sorted(set(rep.warnings)),
            dict(rep.final_refs))


def sim_cases(seeds, n_stmts=(8, 30), **over):
    """(name, ProgramModel, SimConfig) for generated programs in both modes:
    the original (implicit) and its reference transform (annotated)."""
    import random
    from dartomp.pipeline import load, program_model, transform
    from dartomp.simulator import SimConfig
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    for seed in seeds:
        r = random.Random(seed)
        kw = dict(n_funcs=r.randrange(0, 3), n_stmts=r.randrange(*n_stmts), p_jump=0.0)
        kw.update(over)
        text = generate(seed, GenConfig(**kw))
        try:
            a = load(path="g%d.c" % seed, text=text)
            res, _ = transform(a)
            t = load(path="g%d.c (transformed)" % seed, text=res.text)
        except Exception:      # noqa: BLE001 -- programs the reference refuses
            continue
        trip = [1, 2, 3, 7][seed % 4]
        yield ("g%d/implicit" % seed, program_model(a), SimConfig(mode="implicit", default_trip=trip))
        yield ("g%d/annotated" % seed, program_model(t), SimConfig(mode="annotated", default_trip=trip))
