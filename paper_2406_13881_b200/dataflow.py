"""Drop-in `analyze_function` backed by the E1 replay engine.

`analyze_function(src, cfg, accesses, table, allow_stale)` keeps the reference
signature and return type (`dartomp/dataflow.py:737-740`): a
`dartomp.dataflow.FunctionPlan` whose anchors are the very `AstNode` objects
of the caller's AST, so `dartomp.rewriter.apply_plans` and
`dartomp.report.plan_lines` consume it unchanged.  `analyze_functions` is the
batched form (one engine launch for many functions; SURVEY §8 b).

Pipeline per batch: host lowering (`lower.py`) -> pack into flat arrays ->
`dfx_replay_batch` (CUDA, `csrc/replay.cu`) -> events sorted by visit key ->
`_finish` restated on name sets (`dataflow.py:678-711`).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import gc

import numpy as np

from . import _abi
from ._host import import_dartomp
from .lower import FnProgram, lower_function

import_dartomp()
from dartomp.access import Storage  # noqa: E402
from dartomp.dataflow import (AFTER, BEFORE, BODY_END, KERNEL,  # noqa: E402
                              DirectivePlan, FunctionPlan, PlanKind,
                              TargetDataRegion)
from dartomp.diagnostics import DeclPlacementError, PreconditionError  # noqa: E402

_POS = {_abi.POS_BEFORE: BEFORE, _abi.POS_AFTER: AFTER,
        _abi.POS_BODY_END: BODY_END, _abi.POS_KERNEL: KERNEL}


@dataclass
class PackedBatch:
    fns: np.ndarray        # FN_DESC_DTYPE
    ops: np.ndarray
    var_flags: np.ndarray
    stmt_span: np.ndarray
    sites: np.ndarray
    arms: np.ndarray

    @property
    def n_vars(self) -> int:
        return int(self.var_flags.shape[0])

    def replay_in(self) -> _abi.ReplayIn:
        r = _abi.ReplayIn()
        r.n_funcs = int(self.fns.shape[0])
        r.fns = _abi.ptr(self.fns)
        r.ops = _abi.ptr(self.ops)
        r.var_flags = _abi.ptr(self.var_flags)
        r.stmt_span = _abi.ptr(self.stmt_span)
        r.sites = _abi.ptr(self.sites)
        r.arms = _abi.ptr(self.arms)
        r.n_ops = int(self.ops.shape[0])
        r.n_vars = int(self.var_flags.shape[0])
        r.n_stmts = int(self.stmt_span.shape[0])
        r.n_sites = int(self.sites.shape[0])
        r.n_arms = int(self.arms.shape[0]) // 2     # units of (kind, node) pairs
        return r


def pack(progs: list[FnProgram]) -> PackedBatch:
    """Concatenate lowered programs into the flat arrays of `dfx_replay_in`."""
    n = len(progs)
    fns = np.zeros(n, dtype=_abi.FN_DESC_DTYPE)
    op_off = var_off = stmt_off = site_off = arm_off = 0
    for i, p in enumerate(progs):
        d = fns[i]
        d["op_off"], d["n_ops"] = op_off, p.ops.shape[0]
        d["var_off"], d["n_vars"] = var_off, p.var_flags.shape[0]
        d["stmt_off"], d["n_stmts"] = stmt_off, p.stmt_span.shape[0]
        d["site_off"], d["arm_off"] = site_off, arm_off
        d["region_begin_start"] = p.region_begin_start
        d["n_slots"] = p.n_slots
        d["max_loop_depth"] = p.max_loop_depth
        d["max_br_depth"] = p.max_br_depth
        d["max_arms"] = p.max_arms
        d["flags"] = p.fn_flags
        op_off += p.ops.shape[0]
        var_off += p.var_flags.shape[0]
        stmt_off += p.stmt_span.shape[0]
        site_off += p.sites.shape[0]
        arm_off += p.arms.shape[0] // 2

    def cat(arrs, shape_tail, dtype=np.int32):
        arrs = [a.reshape((-1,) + shape_tail) for a in arrs]
        if not arrs:
            return np.zeros((0,) + shape_tail, dtype=dtype)
        return np.ascontiguousarray(np.concatenate(arrs).astype(dtype, copy=False))

    return PackedBatch(
        fns=fns,
        ops=cat([p.ops for p in progs], (4,)),
        var_flags=cat([p.var_flags for p in progs], ()),
        stmt_span=cat([p.stmt_span for p in progs], (2,)),
        sites=cat([p.sites for p in progs], ()),
        arms=cat([p.arms for p in progs], ()),
    )


def concat_batches(batches: list[PackedBatch]) -> PackedBatch:
    """One packed batch holding the functions of several, in order (each
    function's offsets shifted by the sizes of the batches before it)."""
    fns, offs = [], np.zeros(5, dtype=np.int64)
    for b in batches:
        f = b.fns.copy()
        for k, name in enumerate(("op_off", "var_off", "stmt_off", "site_off", "arm_off")):
            f[name] += offs[k]
        fns.append(f)
        offs += (b.ops.shape[0], b.var_flags.shape[0], b.stmt_span.shape[0],
                 b.sites.shape[0], b.arms.shape[0] // 2)
    cat = lambda k: np.ascontiguousarray(np.concatenate([getattr(b, k) for b in batches]))  # noqa: E731
    return PackedBatch(fns=np.concatenate(fns), ops=cat("ops"), var_flags=cat("var_flags"),
                       stmt_span=cat("stmt_span"), sites=cat("sites"), arms=cat("arms"))


def pack_ops(ops: np.ndarray) -> np.ndarray | None:
    """16-byte replay ops [n, 4] -> the 8-byte form of `dfx_replay_batch_packed`
    ([n, 2] uint32, include/dfx.h), or None when a field does not fit (then
    the batch goes through `dfx_replay_batch`)."""
    o = ops.astype(np.int64)
    x, y, z, w = o[:, 0], o[:, 1], o[:, 2], o[:, 3]
    code, fl = x & 0xFF, x >> 8
    a = np.zeros_like(y)
    b = np.zeros_like(y)
    c = np.zeros_like(y)
    kept = np.zeros((o.shape[0], 3), dtype=bool)         # which of y, z, w the form keeps
    acc = (code == _abi.OP_HR) | (code == _abi.OP_DR)
    ab = acc | (code == _abi.OP_HW) | (code == _abi.OP_DW) | (code == _abi.OP_ERR)
    a[ab], b[ab] = y[ab], z[ab]
    kept[ab, 0] = kept[ab, 1] = True
    c[acc] = w[acc]
    kept[acc, 2] = True
    m = code == _abi.OP_BR_END
    c[m], b[m] = y[m], z[m]
    kept[m, 0] = kept[m, 1] = True
    m = code == _abi.OP_LOOP_BEGIN
    a[m] = y[m]
    kept[m, 0] = True
    m = code == _abi.OP_LOOP_END
    c[m] = y[m]
    kept[m, 0] = True
    dropped = np.where(kept, 0, o[:, 1:])
    if ((code > 15).any() or (fl < 0).any() or (fl > 31).any() or (dropped != 0).any()
            or (a < 0).any() or (a > 0xFFFF).any() or (b < 0).any() or (b > 0xFFFF).any()
            or (c < 0).any() or (c >= 1 << 23).any()):
        return None
    out = np.empty((o.shape[0], 2), dtype=np.uint32)
    out[:, 0] = (code | (fl << 4) | (c << 9)).astype(np.uint32)
    out[:, 1] = (a | (b << 16)).astype(np.uint32)
    return out


def unpack_ops(packed: np.ndarray) -> np.ndarray:
    """`pack_ops` inverse (the device's unpack, restated for tests)."""
    p = packed.astype(np.int64)
    code, fl, c = p[:, 0] & 15, (p[:, 0] >> 4) & 31, p[:, 0] >> 9
    a, b = p[:, 1] & 0xFFFF, p[:, 1] >> 16
    o = np.zeros((p.shape[0], 4), dtype=np.int64)
    o[:, 0] = code | (fl << 8)
    acc = (code == _abi.OP_HR) | (code == _abi.OP_DR)
    ab = acc | (code == _abi.OP_HW) | (code == _abi.OP_DW) | (code == _abi.OP_ERR)
    o[ab, 1], o[ab, 2] = a[ab], b[ab]
    o[acc, 3] = c[acc]
    m = code == _abi.OP_BR_END
    o[m, 1], o[m, 2] = c[m], b[m]
    m = code == _abi.OP_LOOP_BEGIN
    o[m, 1] = a[m]
    m = code == _abi.OP_LOOP_END
    o[m, 1] = c[m]
    return o.astype(np.int32)


@dataclass
class RawResult:
    events: np.ndarray     # EVENT_DTYPE, all functions
    var_out: np.ndarray    # uint8 per packed variable
    kernel_ms: float


def run_replay(batch: PackedBatch, runner=None, event_cap: int | None = None) -> RawResult:
    """Execute a packed batch.  `runner(in, out) -> rc` defaults to the CUDA
    engine's `dfx_replay_batch`; tests pass the CPU oracle's entry point."""
    if runner is None:
        eng = _abi.engine()

        def runner(rin, rout):
            return eng.check(eng.lib.dfx_replay_batch(eng.h, C.byref(rin), C.byref(rout)),
                             "dfx_replay_batch")
    cap = event_cap if event_cap is not None else max(1024, 4 * int(batch.ops.shape[0]))
    while True:
        events = np.zeros(cap, dtype=_abi.EVENT_DTYPE)
        var_out = np.zeros(max(1, batch.n_vars), dtype=np.uint8)
        rin = batch.replay_in()
        rout = _abi.ReplayOut()
        rout.events = _abi.ptr(events)
        rout.event_cap = cap
        rout.var_out = _abi.ptr(var_out)
        rc = runner(rin, rout)
        if rc == _abi.DFX_E_NOSPC or rout.n_events > cap:
            cap = int(rout.n_events) + 16
            continue
        if rc != 0:
            raise _abi.EngineError("replay failed with status %d" % rc)
        return RawResult(events=events[:rout.n_events].copy(),
                         var_out=var_out[:batch.n_vars].copy(),
                         kernel_ms=float(rout.kernel_ms))


class ReplaySession:
    """Reference-facing host-buffer path of E1 (`dfx_replay_batch`) with
    output buffers reused across calls (optionally pinned, so the library's
    chunked H2D / replay / D2H pipeline overlaps).  Results are views into
    the session's buffers, valid until the next call."""

    def __init__(self, eng: _abi.Engine | None = None, alloc=np.empty, event_cap: int = 0):
        self.eng = eng or _abi.engine()
        self.alloc = alloc
        self.cap = event_cap
        self._ev = None
        self._vout = None

    def run(self, batch: PackedBatch, packed_ops: np.ndarray | None = None) -> RawResult:
        """`packed_ops`: the batch's ops in the 8-byte form (`pack_ops`), sent
        through `dfx_replay_batch_packed` (half the ops' host->device bytes)."""
        if self.cap <= 0:
            self.cap = max(1024, 4 * int(batch.ops.shape[0]) // 10)
        while True:
            if self._ev is None or self._ev.shape[0] < self.cap:
                self._ev = self.alloc((self.cap,), _abi.EVENT_DTYPE)
            if self._vout is None or self._vout.shape[0] < max(1, batch.n_vars):
                self._vout = self.alloc((max(1, batch.n_vars),), np.uint8)
            rin = batch.replay_in()
            call = self.eng.lib.dfx_replay_batch
            if packed_ops is not None:
                assert packed_ops.dtype == np.uint32 and packed_ops.shape == (batch.ops.shape[0], 2)
                rin.ops = _abi.ptr(packed_ops)
                call = self.eng.lib.dfx_replay_batch_packed
            rout = _abi.ReplayOut()
            rout.events = _abi.ptr(self._ev)
            rout.event_cap = self._ev.shape[0]
            rout.var_out = _abi.ptr(self._vout)
            rc = call(self.eng.h, C.byref(rin), C.byref(rout))
            if rc == _abi.DFX_E_NOSPC:
                self.cap = int(rout.n_events) + 16
                continue
            self.eng.check(rc, "dfx_replay_batch")
            return RawResult(events=self._ev[:rout.n_events], var_out=self._vout[:batch.n_vars],
                             kernel_ms=float(rout.kernel_ms))


# ---- decoding --------------------------------------------------------------

def _raise_error(prog: FnProgram, src, ev) -> None:
    kind = int(ev["kind"])
    if kind == _abi.EV_ERR_DATAMAP:
        stmt = prog.stmts[int(ev["node"])]
        raise PreconditionError(
            "input already contains a '%s' directive; analysis expects "
            "unmapped offload regions" % stmt.omp.kind.value,
            path=src.path, line=src.line_of(stmt.span.start))
    if kind == _abi.EV_ERR_BRACES_LOOP:
        node = prog.stmts[int(ev["node"])]
        raise PreconditionError.at(
            src, node.span.start,
            "braces are required around this loop body to place an "
            "update directive")
    if kind == _abi.EV_ERR_BRACES_ARM:
        node = prog.stmts[int(ev["node"])]
        raise PreconditionError.at(
            src, node.span.start,
            "braces are required around this branch arm to place an "
            "update directive")
    if kind == _abi.EV_ERR_DECL:
        var = prog.vars[int(ev["var"])]
        begin = prog.region[1]
        begin_line = src.line_of(begin.span.start)
        decl_line = src.line_of(var.decl.span.start)
        raise DeclPlacementError(
            "'%s' needs a device mapping but is declared at line %d, "
            "after the data region opening at line %d; move the "
            "declaration above the region" % (var.name, decl_line, begin_line),
            path=src.path, line=decl_line)
    raise _abi.EngineError("replay engine resource limit hit in %s (event kind %d)"
                           % (prog.fn.name, kind))


_PLAN_KIND = {_abi.EV_UPDATE_FROM: PlanKind.UPDATE_FROM,
              _abi.EV_UPDATE_TO: PlanKind.UPDATE_TO,
              _abi.EV_FIRSTPRIVATE: PlanKind.FIRSTPRIVATE}


def decode(prog: FnProgram, src, accesses, events: np.ndarray,
           var_out: np.ndarray, presorted: bool = False) -> FunctionPlan:
    """Events of one function (any order, or key order with `presorted`) +
    per-variable bits -> FunctionPlan."""
    if events.shape[0] and not presorted:
        events = events[np.argsort(events["key"], kind="stable")]
    return _decode_cols(prog, src, accesses, events, events["kind"].tolist(),
                        events["var"].tolist(), events["node"].tolist(),
                        events["pos"].tolist(), var_out)


def _decode_cols(prog: FnProgram, src, accesses, events, kinds, vis, nis, pis,
                 var_out, presorted_unique: bool = False) -> FunctionPlan:
    """`decode` on the event columns as lists (key order); `events` (the same
    events as a structured array, or a callable returning it) is read only to
    raise an error.  `presorted_unique`: repeated records were already dropped."""
    updates: list = []
    firstprivates: list = []
    suppressed: list[str] = []
    if kinds:
        if max(kinds) >= _abi.EV_ERR_DATAMAP:
            if callable(events):            # the batch path passes the rows lazily
                events = events()
            errs = events[events["kind"] >= _abi.EV_ERR_DATAMAP]
            _raise_error(prog, src, errs[0])
        keys: set = set()
        pstmts = prog.stmts
        names = [v.name for v in prog.vars]
        name1 = [(n,) for n in names]       # one names tuple per variable
        # the batch path drops repeated (variable, node, kind, position)
        # records before decoding (`_first_occurrences`), so the key set is
        # needed only where two variables share a name (shadowing)
        dedup = not presorted_unique or len(set(names)) != len(names)
        suppress, fp = _abi.EV_SUPPRESS, _abi.EV_FIRSTPRIVATE
        new, DP = object.__new__, DirectivePlan
        for kind, vi, ni, pi in zip(kinds, vis, nis, pis):
            name = names[vi]
            if kind == suppress:
                if name not in suppressed:
                    suppressed.append(name)
                continue
            # `_add_plan`'s key (`dataflow.py:264`): kind, name, anchor
            # identity (one statement per node index), position
            if dedup:
                key = (kind, name, ni, pi)
                if key in keys:
                    continue
                keys.add(key)
            # DirectivePlan(kind, (name,), anchor, position), built without
            # the frozen dataclass's per-field object.__setattr__ (the same
            # object: fields live in its __dict__; eq/hash read them)
            plan = new(DP)
            pd = plan.__dict__
            pd["kind"] = _PLAN_KIND[kind]
            pd["names"] = name1[vi]
            pd["anchor"] = pstmts[ni]
            pd["position"] = _POS[pi]
            (firstprivates if kind == fp else updates).append(plan)
    # sets (`dataflow.py:214-216`) and `_escape_liveness` (`:671-676`)
    presence, to_comp, from_comp = set(), set(), set()
    for i, var in enumerate(prog.vars):
        o = int(var_out[i])
        if o & _abi.OUT_PRESENCE:
            presence.add(var)
            if (o & _abi.OUT_D) and not (o & _abi.OUT_H) \
                    and var.storage is not Storage.LOCAL:
                from_comp.add(var)
        if o & _abi.OUT_TO:
            to_comp.add(var)
        if o & _abi.OUT_FROM:
            from_comp.add(var)
    return _finish(prog, src, accesses, presence, to_comp, from_comp,
                   updates, firstprivates, suppressed)


def _finish(prog, src, accesses, presence, to_comp, from_comp, updates,
            firstprivates, suppressed) -> FunctionPlan:
    """`_Analyzer._finish` (`dataflow.py:678-711`)."""
    fn = prog.fn
    if not prog.kernel_stmts:
        return FunctionPlan(fn, None, [], [], suppressed)
    block, begin, end = prog.region
    to_names = {v.name for v in to_comp}
    from_names = {v.name for v in from_comp}
    tofrom = sorted(to_names & from_names)
    to_only = sorted(to_names - from_names)
    from_only = sorted(from_names - to_names)
    alloc = sorted({v.name for v in presence} - to_names - from_names)
    kernel_clauses = list(firstprivates)
    single = (len(prog.kernel_stmts) == 1
              and begin is prog.kernel_stmts[0]
              and end is prog.kernel_stmts[0]
              and not updates)
    region = None
    if single:
        k = prog.kernel_stmts[0]
        for kind, names in ((PlanKind.MAP_TO, to_only),
                            (PlanKind.MAP_TOFROM, tofrom),
                            (PlanKind.MAP_FROM, from_only),
                            (PlanKind.MAP_ALLOC, alloc)):
            if names:
                kernel_clauses.append(DirectivePlan(kind, tuple(names), k, KERNEL))
    elif presence or updates:
        if prog.scoping_error is not None:      # `_check_region_scoping` (`:713-734`)
            raise DeclPlacementError.at(src, *prog.scoping_error)
        region = TargetDataRegion(block=block, begin=begin, end=end,
                                  map_to=tuple(to_only), map_from=tuple(from_only),
                                  map_tofrom=tuple(tofrom), map_alloc=tuple(alloc))
    return FunctionPlan(fn, region, kernel_clauses, updates, suppressed)


# ---- public API --------------------------------------------------------------

class _Deferred:
    """Per-function result: a FunctionPlan or the exception the reference raises."""

    def __init__(self, plan=None, error=None):
        self.plan = plan
        self.error = error

    def get(self):
        if self.error is not None:
            raise self.error
        return self.plan


# ---- parallel lowering -------------------------------------------------------
# The lowering (the static half of `_Analyzer`) is pure Python and, once the
# solve runs on the GPU, the host-side Amdahl limit for many functions
# (SURVEY §8f rank 1).  Functions are independent, so large batches are
# lowered by forked worker processes that see the parsed translation unit
# copy-on-write.  Objects cannot cross processes, so a worker returns the
# program's arrays with node and variable references as indices (the CFG
# node id of a statement that is one, else a child-index path from the
# function's AST root; index of an access naming the variable), and the
# parent maps them back to its own objects -- the FunctionPlan anchors stay
# the caller's AstNodes.
_FORK_ITEMS: list = []
_FORK_ALLOW: frozenset = frozenset()


def _path(node, root) -> tuple:
    """Child indices leading from `root` to `node`."""
    steps = []
    while node is not root:
        p = node.parent
        steps.append(next(i for i, c in enumerate(p.children) if c is node))
        node = p
    return tuple(reversed(steps))


def _follow(root, path):
    for i in path:
        root = root.children[i]
    return root


def _ref(node, root, cfg):
    """A node reference that survives the process boundary: the id of the
    CFG node it is the statement of (most statements), else its child path."""
    cn = cfg.node_of_ast.get(node)
    if cn is not None and cn.ast is node and cfg.nodes[cn.id] is cn:
        return cn.id
    return _path(node, root)


def _deref(ref, root, cfg):
    return cfg.nodes[ref].ast if isinstance(ref, int) else _follow(root, ref)


def _lower_portable(i: int):
    src, cfg, accs, table = _FORK_ITEMS[i]
    try:
        prog = lower_function(src, cfg, accs, table, _FORK_ALLOW)
    except Exception as e:      # noqa: BLE001 -- re-raised by the parent's serial retry
        return ("error", repr(e))
    root = cfg.function
    first = {}
    for j, a in enumerate(accs):
        first.setdefault(id(a.var), j)
    try:
        stmts = [_ref(n, root, cfg) for n in prog.stmts]
        kstmts = [_ref(n, root, cfg) for n in prog.kernel_stmts]
        region = None if prog.region is None else [_ref(n, root, cfg) for n in prog.region]
        vars_ = [first[id(v)] for v in prog.vars]
        premapped = None if prog.premapped is None else _ref(prog.premapped, root, cfg)
    except (KeyError, AttributeError, StopIteration):
        return ("serial", None)  # a reference not reachable this way: lower in the parent
    fields = {k: getattr(prog, k) for k in ("ops", "var_flags", "stmt_span", "sites", "arms",
                                            "region_begin_start", "n_slots", "max_loop_depth",
                                            "max_br_depth", "max_arms", "fn_flags",
                                            "scoping_error")}
    return ("ok", (fields, stmts, kstmts, region, vars_, premapped))


def _fork_tree_map(n: int, workers: int, timeout: float):
    """`_lower_portable` over range(n) in `workers` forked processes, or None
    (a worker failed or the deadline passed: the caller lowers serially).

    Forking a process whose heap holds a large parse costs milliseconds per
    fork (page tables), so the workers start as a two-level tree: the parent
    forks ~sqrt(workers) group leaders, each leader forks the rest of its
    group in parallel with the others.  Worker w lowers functions w,
    w + workers, ... and sends its results through its own pipe, pickled
    once.  A group is one process group, so a stalled one is killed whole."""
    import math
    import os
    import pickle
    import select
    import signal
    import time
    fan = max(1, math.isqrt(workers))
    groups = [list(range(g, workers, fan)) for g in range(fan)]
    pipes = [os.pipe() for _ in range(workers)]

    def in_child(body, keep_write):
        """Run `body` in this (forked) process and exit; only the write ends
        in `keep_write` stay open."""
        code = 1
        try:
            for x, (r, wfd) in enumerate(pipes):
                os.close(r)
                if x not in keep_write:
                    os.close(wfd)
            body()
            code = 0
        finally:
            os._exit(code)

    def run_worker(w):
        out = pickle.dumps([_lower_portable(i) for i in range(w, n, workers)], protocol=5)
        view = memoryview(out)
        while view:
            view = view[os.write(pipes[w][1], view):]
        os.close(pipes[w][1])

    def lead(grp):
        os.setpgid(0, 0)
        subs = []
        for w in grp[1:]:
            pid = os.fork()
            if pid == 0:                # the leader holds only its group's write ends
                code = 1
                try:
                    for x in grp:
                        if x != w:
                            os.close(pipes[x][1])
                    run_worker(w)
                    code = 0
                finally:
                    os._exit(code)
            subs.append(pid)
        for w in grp[1:]:
            os.close(pipes[w][1])
        run_worker(grp[0])
        if not all(os.waitpid(pid, 0)[1] == 0 for pid in subs):
            raise RuntimeError("a lowering worker failed")

    import warnings
    leaders = []
    with warnings.catch_warnings():     # the children run pure Python, no CUDA, no locks
        warnings.filterwarnings("ignore", message=".*multi-threaded.*fork.*",
                                category=DeprecationWarning)
        for grp in groups:
            pid = os.fork()
            if pid == 0:
                in_child(lambda grp=grp: lead(grp), set(grp))  # never returns
            leaders.append(pid)
    for _, wfd in pipes:
        os.close(wfd)
    bufs = {r: [] for r, _ in pipes}
    open_fds = set(bufs)
    deadline = time.monotonic() + timeout
    failed = False
    while open_fds:
        left = deadline - time.monotonic()
        if left <= 0:
            failed = True
            break
        ready, _, _ = select.select(list(open_fds), [], [], left)
        for fd in ready:
            chunk = os.read(fd, 1 << 22)
            if chunk:
                bufs[fd].append(chunk)
            else:
                open_fds.discard(fd)
    if failed:
        for pid in leaders:
            try:
                os.killpg(pid, signal.SIGKILL)
            except OSError:
                pass
    for pid in leaders:
        failed |= os.waitpid(pid, 0)[1] != 0
    for r, _ in pipes:
        os.close(r)
    if failed:
        return None
    res: list = [None] * n
    for w, (r, _) in enumerate(pipes):
        items = pickle.loads(b"".join(bufs[r])) if bufs[r] else []
        if len(items) != len(range(w, n, workers)):
            return None
        for k, item in enumerate(items):
            res[w + k * workers] = item
    return res


def lower_functions(items, allow_stale: frozenset = frozenset(), workers: int | None = None):
    """`lower_function` over a batch; forked workers for large batches
    (`workers` or $DFX_LOWER_WORKERS, default min(16, cores); serial below
    64 functions or with one worker)."""
    import multiprocessing as mp
    import os
    if workers is None:
        workers = int(os.environ.get("DFX_LOWER_WORKERS", "0")) or min(16, os.cpu_count() or 1)
    if workers <= 1 or len(items) < 64 or "fork" not in mp.get_all_start_methods():
        return [lower_function(src, cfg, accs, table, allow_stale)
                for src, cfg, accs, table in items]
    global _FORK_ITEMS, _FORK_ALLOW
    _FORK_ITEMS, _FORK_ALLOW = list(items), allow_stale
    try:
        # the workers run pure Python on the copied parse (no CUDA, no locks
        # of the parent's other threads); a bounded wait falls back to the
        # serial lowering if a worker ever stalls
        res = _fork_tree_map(len(items), workers, 60 + 0.05 * len(items))
    finally:
        _FORK_ITEMS, _FORK_ALLOW = [], frozenset()
    if res is None:
        return [lower_function(src, cfg, accs, table, allow_stale)
                for src, cfg, accs, table in items]
    progs = []
    for (src, cfg, accs, table), (tag, r) in zip(items, res):
        if tag != "ok":         # errors and unmappable programs: the serial path decides
            progs.append(lower_function(src, cfg, accs, table, allow_stale))
            continue
        fields, stmts, kstmts, region, vars_, premapped = r
        root = cfg.function
        cfg_nodes = cfg.nodes
        progs.append(FnProgram(fn=root, **fields,
                               vars=[accs[j].var for j in vars_],
                               stmts=[cfg_nodes[q].ast if q.__class__ is int else _follow(root, q)
                                      for q in stmts],
                               kernel_stmts=[_deref(q, root, cfg) for q in kstmts],
                               region=None if region is None else tuple(_deref(q, root, cfg) for q in region),
                               premapped=None if premapped is None else _deref(premapped, root, cfg)))
    return progs


def _event_order(evs: np.ndarray) -> np.ndarray:
    """Order of the events by function, then visit key.  One 64-bit sort on
    a combined key when the function index and the key fit beside each other
    (always at C4 scale: 17 + 55 bits), else a two-key lexsort."""
    if evs.shape[0] < 2:
        return np.arange(evs.shape[0])
    fn = evs["fn"]
    key = evs["key"]
    fb = max(1, int(fn.max()).bit_length())
    if fn.min() >= 0 and int(key.max()) < (1 << (64 - fb)):
        return np.argsort((fn.astype(np.uint64) << np.uint64(64 - fb)) | key)
    return np.lexsort((key, fn))


def _first_occurrences(fn, var, node, kind, pos) -> np.ndarray:
    """Mask of the events (columns, sorted by function, then visit key) that
    are the first of their (function, kind, variable, node, position): a
    repeat (a plan re-planned in a later loop round) is dropped by
    `_add_plan`'s dedup (`dataflow.py:259-268`) and a repeated suppression by
    name, so `decode` need not see it.  Error events are always kept."""
    n = fn.shape[0]
    if n < 2:
        return np.ones(n, dtype=bool)
    fn = fn.astype(np.int64)
    var = var.astype(np.int64) + 1          # -1 (function-level errors) -> 0
    node = node.astype(np.int64)
    kind64, pos64 = kind.astype(np.int64), pos.astype(np.int64)
    if (fn.min() >= 0 and fn.max() < (1 << 27) and var.max() < (1 << 15) and node.min() >= 0
            and node.max() < (1 << 16)):
        key = (fn << 36) | (var << 21) | (node << 5) | (kind64 << 2) | pos64
        _, first = np.unique(key, return_index=True)
    else:
        order = np.lexsort((pos64, kind64, node, var, fn))
        k = np.stack([fn[order], var[order], node[order], kind64[order], pos64[order]])
        new = np.ones(order.shape[0], dtype=bool)
        new[1:] = (k[:, 1:] != k[:, :-1]).any(axis=0)
        # first occurrence in event order of each distinct record
        grp = np.cumsum(new) - 1
        first = np.full(int(grp[-1]) + 1, np.iinfo(np.int64).max)
        np.minimum.at(first, grp, order)
    keep = np.zeros(n, dtype=bool)
    keep[first] = True
    keep |= kind >= _abi.EV_ERR_DATAMAP
    return keep


def analyze_functions(items, allow_stale: frozenset[str] = frozenset(),
                      runner=None, precheck=None) -> list[_Deferred]:
    """Batched `analyze_function`: `items` is a list of
    `(src, cfg, accesses, table)`; one engine launch for all of them.
    Returns one deferred result per item (`.get()` returns the
    `FunctionPlan` or raises the reference's exception).  `precheck(progs)`
    runs after the lowering and before the launch (the unit-level input
    checks of `plan_transform`, fed by the per-function lowering)."""
    # The batch allocates a few objects per event on top of the caller's
    # parse (millions of long-lived AST objects), so the cyclic collector's
    # full passes -- each a walk of that whole heap -- would cost more than
    # the analysis; it is paused for the call (nothing built here is cyclic
    # garbage) and restored as it was.
    gc_was = gc.isenabled()
    gc.disable()
    try:
        return _analyze_functions(items, allow_stale, runner, precheck)
    finally:
        if gc_was:
            gc.enable()


def _analyze_functions(items, allow_stale, runner, precheck) -> list[_Deferred]:
    progs = lower_functions(items, allow_stale)
    if precheck is not None:
        precheck(progs)
    batch = pack(progs)
    raw = run_replay(batch, runner=runner)
    # by function, then visit key; gathered column by column (a gather of
    # the 24-byte records costs about three times as much)
    order = _event_order(raw.events)
    cols = {c: raw.events[c][order] for c in ("fn", "var", "node", "kind", "pos")}
    keep = _first_occurrences(cols["fn"], cols["var"], cols["node"], cols["kind"], cols["pos"])
    idx = order[keep]                       # into raw.events, for the error path
    cols = {c: v[keep] for c, v in cols.items()}
    bounds = np.searchsorted(cols["fn"], np.arange(len(progs) + 1)).tolist()
    # columns once, as lists; per function a slice of each
    kinds, vis = cols["kind"].tolist(), cols["var"].tolist()
    nis, pis = cols["node"].tolist(), cols["pos"].tolist()
    var_off, n_vars = batch.fns["var_off"].tolist(), batch.fns["n_vars"].tolist()
    events = raw.events
    out = []
    for i, (p, (src, cfg, accs, table)) in enumerate(zip(progs, items)):
        a, b = bounds[i], bounds[i + 1]
        vo = raw.var_out[var_off[i]:var_off[i] + n_vars[i]]
        try:
            out.append(_Deferred(plan=_decode_cols(
                p, src, accs, lambda a=a, b=b: events[idx[a:b]], kinds[a:b], vis[a:b],
                nis[a:b], pis[a:b], vo, True)))
        except Exception as e:  # the reference's ToolError subclasses
            out.append(_Deferred(error=e))
    return out


def analyze_function(src, cfg, accesses, table,
                     allow_stale: frozenset[str] = frozenset()) -> FunctionPlan:
    """Drop-in for `dartomp.dataflow.analyze_function` (`dataflow.py:737`)."""
    return analyze_functions([(src, cfg, accesses, table)], allow_stale)[0].get()
