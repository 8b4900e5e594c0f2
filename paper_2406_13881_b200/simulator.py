"""Drop-in `simulate` (and `compare`) backed by the CUDA transfer simulator
(SURVEY §8 f3): `dartomp.simulator.simulate(program, config) -> SimReport`
(`simulator.py:708`) and `dartomp.pipeline.compare` (`pipeline.py:122-143`).

Pipeline: `simlower.lower_program` (host: the simulator's walk with control
resolved) -> `dfx_sim_batch` (CUDA, `csrc/sim.cu`: per-variable state
machine, per-variable loop settling) -> a `SimReport`.

What the report reproduces exactly: the transfer totals (HtoD / DtoH calls
and bytes), the stale-read count, the stale reads aggregated per (variable,
space, line), the warnings (as a set, ordered by their first appearance in
the program text of the lowering), the final reference counts and the entry
list.  `simulation_lines` / `comparison_lines` therefore print the
reference's `mode`, `entry`, `htod`, `dtoh` and `stale` lines byte for byte;
the per-event list of the verbose report is not reproduced (the kernel
counts per variable, it does not keep the reference's global log order), and
a stale read repeated over rounds is one aggregated record instead of the
reference's per-round records.  `simulate_batch` runs many programs in one
launch -- the verifier form: SPEC's soundness invariant (zero stale reads on
the transformed program) checked at batch scale.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._host import import_dartomp
from .simlower import SimProgram, lower_program

import_dartomp()
from dartomp.access import Space  # noqa: E402
from dartomp.simulator import (SimConfig, SimReport, StaleRead,  # noqa: E402
                               TransferLog)


class SimProg(C.Structure):
    _fields_ = [("op_off", C.c_int32), ("n_ops", C.c_int32), ("var_off", C.c_int32),
                ("n_vars", C.c_int32)]


class SimIn(C.Structure):
    _fields_ = [("n_progs", C.c_int32), ("progs", C.c_void_p), ("ops", C.c_void_p),
                ("arg64", C.c_void_p), ("n_ops", C.c_int64), ("n_vars", C.c_int64)]


class SimOut(C.Structure):
    _fields_ = [("vars", C.c_void_p), ("recs", C.c_void_p), ("rec_cap", C.c_int64),
                ("n_recs", C.c_int64), ("kernel_ms", C.c_float)]


SIM_VAR_DTYPE = np.dtype([("htod_calls", np.uint64), ("htod_bytes", np.uint64),
                          ("dtoh_calls", np.uint64), ("dtoh_bytes", np.uint64),
                          ("stale", np.uint64), ("ref", np.int64), ("host_valid", np.uint8),
                          ("device_valid", np.uint8), ("flags", np.uint8), ("pad", np.uint8, 5)])
SIM_REC_DTYPE = np.dtype([("prog", np.int32), ("var", np.int32), ("id", np.int32),
                          ("kind", np.int32), ("count", np.uint64)])
assert SIM_VAR_DTYPE.itemsize == 56 and SIM_REC_DTYPE.itemsize == 24
REC_STALE, REC_WARN, REC_NOSETTLE = 0, 1, 2
_SPACE = {0: Space.HOST.value, 1: Space.DEVICE.value}
VF_OVERFLOW, VF_FAULT = 1, 2


class AggregateTransferLog(TransferLog):
    """`TransferLog` whose totals come from the per-variable counts."""

    def __init__(self, totals: dict, stale_reads: list):
        super().__init__(events=[], stale_reads=stale_reads)
        self._totals = totals

    def calls(self, direction: str) -> int:
        return self._totals[direction][0]

    def bytes(self, direction: str) -> int:
        return self._totals[direction][1]


@dataclass
class SimRaw:
    """Per-variable outputs and records of one batch."""
    vars: np.ndarray
    recs: np.ndarray
    kernel_ms: float


def run_sim(progs: list[SimProgram], eng: _abi.Engine | None = None) -> SimRaw:
    """One `dfx_sim_batch` launch over lowered programs."""
    eng = eng or _abi.engine()
    lib = eng.lib
    lib.dfx_sim_batch.restype = C.c_int
    n = len(progs)
    desc = (SimProg * max(1, n))()
    op_off = var_off = 0
    for i, p in enumerate(progs):
        desc[i].op_off, desc[i].n_ops = op_off, p.ops.shape[0]
        desc[i].var_off, desc[i].n_vars = var_off, p.n_vars
        op_off += p.ops.shape[0]
        var_off += p.n_vars
    ops = np.ascontiguousarray(np.concatenate([p.ops for p in progs]) if n else
                               np.zeros((1, 4), np.int32), dtype=np.int32)
    a64 = np.ascontiguousarray(np.concatenate([p.arg64 for p in progs]) if n else
                               np.zeros(1, np.int64), dtype=np.int64)
    vars_ = np.zeros(max(1, var_off), dtype=SIM_VAR_DTYPE)
    cap = max(1 << 16, 4 * op_off)
    while True:
        recs = np.zeros(cap, dtype=SIM_REC_DTYPE)
        sin = SimIn(n_progs=n, progs=C.addressof(desc), ops=ops.ctypes.data, arg64=a64.ctypes.data,
                    n_ops=op_off, n_vars=var_off)
        sout = SimOut(vars=vars_.ctypes.data, recs=recs.ctypes.data, rec_cap=cap)
        rc = lib.dfx_sim_batch(eng.h, C.byref(sin), C.byref(sout))
        if rc == _abi.DFX_E_NOSPC:
            cap = int(sout.n_recs) + 1024
            continue
        eng.check(rc, "dfx_sim_batch")
        return SimRaw(vars=vars_[:var_off].copy(), recs=recs[:sout.n_recs].copy(),
                      kernel_ms=float(sout.kernel_ms))


def _report(prog: SimProgram, v: np.ndarray, recs: np.ndarray) -> SimReport:
    if (v["flags"] & VF_OVERFLOW).any():
        raise _abi.EngineError("simulator: a transfer count exceeds 64 bits")
    if (v["flags"] & VF_FAULT).any():
        raise _abi.EngineError("simulator: malformed program (shield stack)")
    tot = {"htod": (int(v["htod_calls"].sum(dtype=np.uint64)), int(v["htod_bytes"].sum(dtype=np.uint64))),
           "dtoh": (int(v["dtoh_calls"].sum(dtype=np.uint64)), int(v["dtoh_bytes"].sum(dtype=np.uint64)))}
    st = recs[recs["kind"] == REC_STALE]
    stale = []
    if st.shape[0]:
        agg: dict = {}
        for var, sid, cnt in zip(st["var"].tolist(), st["id"].tolist(), st["count"].tolist()):
            key = (prog.sites[sid & 0x3FFFFFFF], prog.var_names[var], sid >> 30)
            agg[key] = agg.get(key, 0) + cnt
        # one record per (line, variable, space), in line order
        for (line, name, space), cnt in sorted(agg.items()):
            stale.append(StaleRead(name, _SPACE[space], line, int(cnt)))
    if sum(s.count for s in stale) != int(v["stale"].sum(dtype=np.uint64)):
        raise _abi.EngineError("simulator: stale records disagree with the per-variable counts")
    warn_ids = set(prog.static_warnings)
    warn_ids.update(recs["id"][recs["kind"] == REC_WARN].tolist())
    if (recs["kind"] == REC_NOSETTLE).any():
        warn_ids.add(0)
    warnings = [prog.warnings[k] for k in sorted(warn_ids)]
    refs = {}
    for k in np.nonzero(v["ref"])[0].tolist():
        refs[prog.var_names[k]] = int(v["ref"][k])
    return SimReport(prog.mode, list(prog.entries), AggregateTransferLog(tot, stale), warnings, refs)


def simulate_batch(items, eng: _abi.Engine | None = None) -> list[SimReport]:
    """`simulate` over many (program, config) pairs in one kernel launch."""
    progs = [lower_program(p, c) for p, c in items]
    raw = run_sim(progs, eng)
    out = []
    var_off = 0
    prog_of = raw.recs["prog"]
    order = np.argsort(prog_of, kind="stable")
    recs = raw.recs[order]
    bounds = np.searchsorted(recs["prog"], np.arange(len(progs) + 1))
    for i, p in enumerate(progs):
        v = raw.vars[var_off:var_off + p.n_vars]
        out.append(_report(p, v, recs[bounds[i]:bounds[i + 1]]))
        var_off += p.n_vars
    return out


def simulate(program, config: SimConfig) -> SimReport:
    """Drop-in for `dartomp.simulator.simulate` (`simulator.py:708`)."""
    return simulate_batch([(program, config)])[0]


def simulate_analysis(analysis, config: SimConfig) -> SimReport:
    from dartomp.pipeline import program_model
    return simulate(program_model(analysis), config)


def compare(analysis, config: SimConfig, allow_stale: frozenset[str] = frozenset()):
    """`dartomp.pipeline.compare` (`pipeline.py:122-143`) with the engine's
    transform and the CUDA simulator: both simulations in one launch."""
    from dartomp.pipeline import program_model
    from . import pipeline
    result, _ = pipeline.transform(analysis, allow_stale)
    implicit_cfg = SimConfig(sizes=dict(config.sizes), default_trip=config.default_trip,
                             mode="implicit", pointer_default=config.pointer_default,
                             max_call_depth=config.max_call_depth)
    annotated_cfg = SimConfig(sizes=dict(config.sizes), default_trip=config.default_trip,
                              mode="annotated", pointer_default=config.pointer_default,
                              max_call_depth=config.max_call_depth)
    transformed = pipeline.load(path=analysis.src.path + " (transformed)", text=result.text,
                                sizes=dict(config.sizes), pointer_default=config.pointer_default)
    base, mapped = simulate_batch([(program_model(analysis), implicit_cfg),
                                   (program_model(transformed), annotated_cfg)])
    return base, mapped, result
