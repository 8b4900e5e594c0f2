"""Configuration C4: batches of independent functions through the E1 replay
engine, sharded across GPUs.

Functions come from the native generator (`csrc/c4gen.cpp`, exported as
`dfx_gen_c4`), which emits replay programs directly -- 100k functions need no
C front end.  Sharding is longest-processing-time-first over a cost model of
the generator's cheap shapes (N_f statement nodes x ceil(V_f/32) warps); no
collective touches the data path (functions are independent).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .dataflow import PackedBatch, RawResult


@dataclass
class C4Config:
    """BASELINE.json configs[3]: 100k functions, 64-2k nodes, 32-512 vars."""
    n_funcs: int = 100_000
    n_min: int = 64
    n_max: int = 2048
    var_choices: tuple = (32, 64, 128, 256, 512)
    seed: int = 0


def _lib():
    lib = _abi.load_lib()
    lib.dfx_gen_c4.restype = C.c_int
    lib.dfx_gen_c4_shapes.restype = C.c_int
    for n in ("dfx_replay_create", "dfx_replay_run", "dfx_replay_fetch", "dfx_replay_destroy"):
        getattr(lib, n).restype = C.c_int
    return lib


def c4_shapes(cfg: C4Config):
    """(N_f, V_f) of every function of the batch (host only)."""
    lib = _lib()
    N = np.zeros(cfg.n_funcs, dtype=np.int32)
    V = np.zeros(cfg.n_funcs, dtype=np.int32)
    ch = np.array(cfg.var_choices, dtype=np.int32)
    lib.dfx_gen_c4_shapes(C.c_uint64(cfg.seed), C.c_int32(cfg.n_funcs), C.c_int32(cfg.n_min),
                          C.c_int32(cfg.n_max), C.c_void_p(ch.ctypes.data), C.c_int32(len(ch)),
                          C.c_void_p(N.ctypes.data), C.c_void_p(V.ctypes.data))
    return N, V


def lpt_shards(cost: np.ndarray, world: int) -> list[np.ndarray]:
    """Longest-processing-time-first assignment of items to `world` bins;
    each shard is returned sorted (generation order)."""
    order = np.argsort(-cost, kind="stable")
    load = np.zeros(world, dtype=np.float64)
    owner = np.empty(cost.shape[0], dtype=np.int32)
    import heapq
    heap = [(0.0, r) for r in range(world)]
    for i in order:
        l, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (l + float(cost[i]), r))
    return [np.nonzero(owner == r)[0].astype(np.int32) for r in range(world)]


def c4_cost(N: np.ndarray, V: np.ndarray) -> np.ndarray:
    return N.astype(np.float64) * np.ceil(V / 32.0)


def c4_generate(cfg: C4Config, fids: np.ndarray, alloc=np.zeros) -> tuple[PackedBatch, int]:
    """Generate the listed functions as one packed replay batch; `alloc(shape,
    dtype)` lets callers place the arrays in pinned host memory."""
    lib = _lib()
    fids = np.ascontiguousarray(fids, dtype=np.int32)
    ch = np.array(cfg.var_choices, dtype=np.int32)
    sizes = np.zeros(5, dtype=np.int64)
    facts = C.c_int64(0)
    common = (C.c_uint64(cfg.seed), C.c_void_p(fids.ctypes.data), C.c_int32(len(fids)),
              C.c_int32(cfg.n_min), C.c_int32(cfg.n_max), C.c_void_p(ch.ctypes.data),
              C.c_int32(len(ch)))
    lib.dfx_gen_c4(*common, None, None, None, None, None, None,
                   C.c_void_p(sizes.ctypes.data), C.byref(facts))
    n_ops, n_vars, n_stmts, n_sites, n_arms = (int(x) for x in sizes)
    fns = alloc((len(fids),), _abi.FN_DESC_DTYPE)
    ops = alloc((n_ops, 4), np.int32)
    vf = alloc((n_vars,), np.int32)
    span = alloc((n_stmts, 2), np.int32)
    sites = alloc((max(1, n_sites),), np.int32)
    arms = alloc((max(1, 2 * n_arms),), np.int32)
    p = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
    lib.dfx_gen_c4(*common, p(fns), p(ops), p(vf), p(span), p(sites), p(arms), None, None)
    return PackedBatch(fns=fns, ops=ops, var_flags=vf, stmt_span=span, sites=sites[:n_sites],
                       arms=arms[:2 * n_arms]), int(facts.value)


def program_visits(batch: PackedBatch) -> np.ndarray:
    """Dynamic op visits of every function (`dfx_program_visits`): ops the
    reference schedule executes, loops twice (dataflow.py:566-590)."""
    lib = _lib()
    out = np.zeros(batch.fns.shape[0], dtype=np.int64)
    fns = np.ascontiguousarray(batch.fns)
    ops = np.ascontiguousarray(batch.ops)
    rc = lib.dfx_program_visits(C.c_void_p(fns.ctypes.data), C.c_int32(fns.shape[0]),
                                C.c_void_p(ops.ctypes.data), C.c_void_p(out.ctypes.data))
    if rc != 0:
        raise _abi.EngineError("dfx_program_visits failed (%d)" % rc)
    return out


class ReplayBatch:
    """A packed batch resident in HBM (`dfx_replay_create`)."""

    def __init__(self, batch: PackedBatch, event_cap: int | None = None,
                 eng: _abi.Engine | None = None):
        self.eng = eng or _abi.engine()
        _lib()
        self.batch = batch
        self.cap = event_cap or max(1 << 20, 4 * int(batch.ops.shape[0]) // 10)
        rin = batch.replay_in()
        self._keep = rin
        self.h = C.c_void_p()
        self.eng.check(self.eng.lib.dfx_replay_create(self.eng.h, C.byref(rin), C.c_int64(self.cap),
                                                      C.byref(self.h)), "dfx_replay_create")

    def run(self) -> tuple[int, float]:
        n = C.c_int64(0)
        ms = C.c_float(0.0)
        rc = self.eng.lib.dfx_replay_run(self.eng.h, self.h, C.byref(n), C.byref(ms))
        if rc == _abi.DFX_E_NOSPC:
            raise _abi.EngineError("event capacity %d too small (%d events)" % (self.cap, n.value))
        self.eng.check(rc, "dfx_replay_run")
        return int(n.value), float(ms.value)

    def fetch(self) -> RawResult:
        n_vars = self.batch.n_vars
        events = np.zeros(self.cap, dtype=_abi.EVENT_DTYPE)
        var_out = np.zeros(max(1, n_vars), dtype=np.uint8)
        out = _abi.ReplayOut()
        out.events = events.ctypes.data
        out.event_cap = self.cap
        out.var_out = var_out.ctypes.data
        self.eng.check(self.eng.lib.dfx_replay_fetch(self.eng.h, self.h, C.byref(out)),
                       "dfx_replay_fetch")
        return RawResult(events=events[:out.n_events].copy(), var_out=var_out[:n_vars].copy(),
                         kernel_ms=0.0)

    def close(self):
        if self.h:
            self.eng.lib.dfx_replay_destroy(self.eng.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
