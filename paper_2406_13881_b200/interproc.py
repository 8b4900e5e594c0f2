"""Drop-in `summarize_all` backed by kernel (c), plus `apply_call_effects`.

Reference: `dartomp/interproc.py:90-144`.  A function summary maps each
pointer parameter and each global to an `Effect(kind, spaces)`.  Kinds join
as bit sets ({R}, {W}, {R,W}: `access.py:35-44`) and spaces as sets, and
UNKNOWN never survives into a summary (`interproc.py:31-33,79-80`), so a
summary is exactly 4 bits per slot -- R, W, HOST, DEVICE -- and the fixpoint
is an OR-propagation over the call graph:

    S[f] = D[f]  |  OR_{call sites f->g, g defined}  T_cs(S[g])

D[f] folds the function's own accesses (`_direct_effects`, `:75-87`) and every
call to an undeclared external or a declared-but-undefined function (whose
summaries are constants: `:109-120`, `pessimistic_summary` `:50-58`).  T_cs
binds the callee's parameter slots to the caller's slot of each argument's
root (`_classify_bound`, `:147-156`), copies global slots by name, and on a
call made from inside a kernel replaces the spaces by {DEVICE} (`:113-114`).
The least fixpoint is unique, so processing strongly connected components in
reverse topological order (levels) gives the reference's result.

The dict insertion order of `param_effects` / `global_effects` is part of
the output (`apply_call_effects` turns it into access order, hence into the
order of planned directives), and the reference's final orders are those of
its last Gauss-Seidel pass -- not an order fixpoint.  So the engine replays
the reference's pass schedule exactly: passes in dict order until no set
changes, each function rebuilt from its sources in order, carrying an
insertion-order list beside the bits; functions that do not read a
same-pass result run in parallel (waves).

Host lowering (this module) -> `dfx_summaries` (CUDA, `csrc/summ.cu`) ->
`CallSummary` objects.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._host import import_dartomp

import_dartomp()
from dartomp.access import AccessKind, Space, Storage  # noqa: E402
from dartomp.interproc import (CallSummary, Effect,  # noqa: E402
                               apply_call_effects, pessimistic_summary)
from dartomp.nodes import declared_functions, defined_functions  # noqa: E402

__all__ = ["summarize_all", "apply_call_effects", "lower_call_graph", "CallGraph",
           "solve_call_graph", "summaries_from_result"]

BIT_R, BIT_W, BIT_H, BIT_D = 1, 2, 4, 8
_KIND_BITS = {AccessKind.READ: BIT_R, AccessKind.WRITE: BIT_W,
              AccessKind.READWRITE: BIT_R | BIT_W,
              AccessKind.UNKNOWN: BIT_R | BIT_W}   # `_norm`: unknown -> readwrite


_KIND_BITS_ID = {id(k): v for k, v in _KIND_BITS.items()}


def _eff_bits(kind, spaces) -> int:
    b = _KIND_BITS[kind]
    for sp in spaces:
        b |= BIT_H if sp is Space.HOST else BIT_D
    return b


def _kind_of(b: int):
    r, w = b & BIT_R, b & BIT_W
    if r and w:
        return AccessKind.READWRITE
    return AccessKind.READ if r else AccessKind.WRITE


def _spaces_of(b: int) -> frozenset:
    s = set()
    if b & BIT_H:
        s.add(Space.HOST)
    if b & BIT_D:
        s.add(Space.DEVICE)
    return frozenset(s)


_KIND_OF = [_kind_of(b) for b in range(16)]
_SPACES_OF = [_spaces_of(b) for b in range(16)]


def _bits_kind(b: int):
    return _KIND_OF[b & 15]


def _bits_spaces(b: int) -> frozenset:
    return _SPACES_OF[b & 15]


def _force_dev(b: int) -> int:
    return (b & (BIT_R | BIT_W)) | BIT_D if b & (BIT_R | BIT_W) else 0


SRC_STATIC = 0   # constant slot list (direct effects, external/prototype calls)
SRC_CALL = 1     # call to a defined function: bound from the callee's summary


@dataclass
class CallGraph:
    """Lowered summary problem (the inputs of `dfx_summaries`)."""
    names: list                     # defined functions, reference dict order
    fns: list                       # their AstNodes
    n_params: int                   # parameter slots (max over functions)
    globals: list                   # global names, slot n_params + i
    init_bits: np.ndarray           # uint8 [n_funcs, n_slots]  S_0 = _direct_effects
    init_len: np.ndarray            # int32 [n_funcs]
    init_list: np.ndarray           # int16 [n_funcs, n_slots]  S_0 insertion order
    direct: np.ndarray              # uint8 [n_funcs, n_slots]  accesses + constant call sites
    src_off: np.ndarray             # int32 [n_funcs+1]
    src: np.ndarray                 # int32 [n_src, 4] (kind|dev<<8, a, b, c)
    slist: np.ndarray               # int16 static slot lists
    bind: np.ndarray                # int32 [n_bind, 2] (callee param, caller slot)
    wave_off: np.ndarray            # int32 [n_waves+1]
    wave_fns: np.ndarray            # int32 functions grouped by wave
    pess: dict = field(default_factory=dict)   # name -> pessimistic CallSummary

    @property
    def n_slots(self) -> int:
        return self.n_params + len(self.globals)

    @property
    def n_funcs(self) -> int:
        return len(self.names)


def lower_call_graph(src, tu, cfgs, accesses, table) -> CallGraph:
    """Static half of `summarize_all` (`interproc.py:90-144`).

    Each defined function becomes an ordered list of *sources* that rebuild
    its summary in the reference's order: its own accesses
    (`_direct_effects`), then every call site in order -- a constant slot
    list for undeclared externals and declared-but-undefined functions, or a
    binding from the callee's current summary for defined callees.  `wave`
    numbers order the Gauss-Seidel dependencies inside one pass (a callee
    earlier in dict order is read from the same pass: `:105-107`)."""
    from dartomp.access import _Classifier   # the reference's arg-root resolver
    helper = _Classifier(src, table)
    defined = defined_functions(tu)
    declared = declared_functions(tu)
    pess = {name: pessimistic_summary(fn) for name, fn in declared.items() if name not in defined}
    names = list(defined)
    index = {n: i for i, n in enumerate(names)}
    params = {n: defined[n].params for n in names}      # `params` rescans children: once
    n_params = max([len(params[n]) for n in names] + [0])
    gidx: dict[str, int] = {}

    def classify(fn_pidx, root):
        """`_classify_bound` target: ("p", i) / ("g", name) / None."""
        var = table.for_ref(root)
        d = var.decl
        if d is not None and d in fn_pidx and d.type_info.is_pointerish:
            return ("p", fn_pidx[d])
        if var.storage is Storage.GLOBAL:
            return ("g", var.name)
        return None

    per_fn = []
    for name in names:
        fn = defined[name]
        pidx = {p: i for i, p in enumerate(params[name])}
        items = []
        unknown, host, glob = AccessKind.UNKNOWN, Space.HOST, Storage.GLOBAL
        for acc in accesses[name]:                 # `_direct_effects` (:75-87)
            kind = acc.kind
            if kind is unknown:
                continue
            # `_eff_bits(kind, (space,))` (Enum.__hash__ is Python-level: id-keyed)
            b = _KIND_BITS_ID[id(kind)] | (BIT_H if acc.space is host else BIT_D)
            var = acc.var
            d = var.decl
            if d is not None and d in pidx and d.type_info.is_pointerish:
                items.append((("p", pidx[d]), b))
            elif var.storage is glob:
                items.append((("g", var.name), b))
        srcs = [("static", items)]
        for cs in cfgs[name].call_sites:
            args = cs.call.children
            dev = cs.on_device
            if cs.callee in index:                 # defined callee (:119-131)
                binds = []
                for i in range(len(params[cs.callee])):
                    if i >= len(args):
                        continue
                    root = helper.pointerish_arg_root(args[i])
                    if root is None:
                        continue
                    t = classify(pidx, root)
                    if t is not None:
                        binds.append((i, t))
                srcs.append(("call", index[cs.callee], dev, binds))
                continue
            callee = pess.get(cs.callee)
            citems = []
            if callee is None:                     # undeclared external (:109-118)
                for arg in args:
                    root = helper.pointerish_arg_root(arg)
                    if root is None:
                        continue
                    t = classify(pidx, root)
                    if t is not None:
                        citems.append((t, (BIT_R | BIT_W) | (BIT_D if dev else BIT_H)))
            else:                                  # pessimistic summary (:119-131)
                for i, eff in callee.param_effects.items():
                    if i >= len(args):
                        continue
                    root = helper.pointerish_arg_root(args[i])
                    if root is None:
                        continue
                    b = _eff_bits(eff.kind, eff.spaces)
                    t = classify(pidx, root)
                    if t is not None:
                        citems.append((t, _force_dev(b) if dev else b))
            srcs.append(("static", citems))
        per_fn.append(srcs)
        for sr in srcs:
            if sr[0] == "static":
                for t, _ in sr[1]:
                    if t[0] == "g" and t[1] not in gidx:
                        gidx[t[1]] = len(gidx)
            else:
                for _, t in sr[3]:
                    if t[0] == "g" and t[1] not in gidx:
                        gidx[t[1]] = len(gidx)
    gnames = list(gidx)
    n_slots = max(1, n_params + len(gnames))
    if n_slots >= 32767:
        raise ValueError("too many summary slots (%d)" % n_slots)

    def slot(t):
        return t[1] if t[0] == "p" else n_params + gidx[t[1]]

    nf = len(names)
    init_bits = np.zeros((nf, n_slots), dtype=np.uint8)
    init_list = np.zeros((nf, n_slots), dtype=np.int16)
    init_len = np.zeros(nf, dtype=np.int32)
    direct = np.zeros((nf, n_slots), dtype=np.uint8)
    src_off = np.zeros(nf + 1, dtype=np.int32)
    src_rows, slist, bind = [], [], []
    wave = [0] * nf
    # the bits go through dicts keyed by (function, slot) and land in the
    # arrays at the end: numpy item assignment per access is the slow part
    dbits: dict = {}
    ibits: dict = {}
    for f, srcs in enumerate(per_fn):
        row = f * n_slots
        for k, sr in enumerate(srcs):
            if sr[0] == "static":
                order, seen = [], set()
                for t, b in sr[1]:
                    sl = slot(t)
                    key = row + sl
                    dbits[key] = dbits.get(key, 0) | b
                    if k == 0:
                        ibits[key] = ibits.get(key, 0) | b
                    if sl not in seen:
                        seen.add(sl)
                        order.append(sl)
                if k == 0:
                    init_len[f] = len(order)
                    init_list[f, :len(order)] = order
                src_rows.append((SRC_STATIC, len(slist), len(order), 0))
                slist.extend(order)
            else:
                _, g, dev, binds = sr
                src_rows.append((SRC_CALL | ((1 if dev else 0) << 8), g, len(bind), len(binds)))
                bind.extend((i, slot(t)) for i, t in binds)
                if g < f:
                    wave[f] = max(wave[f], wave[g] + 1)
        src_off[f + 1] = len(src_rows)
    for arr, bits in ((direct, dbits), (init_bits, ibits)):
        if bits:
            arr.reshape(-1)[np.fromiter(bits.keys(), np.int64, len(bits))] = \
                np.fromiter(bits.values(), np.uint8, len(bits))
    n_waves = max(wave) + 1 if nf else 0
    buckets: list[list[int]] = [[] for _ in range(n_waves)]
    for f in range(nf):
        buckets[wave[f]].append(f)
    wave_off = np.zeros(n_waves + 1, dtype=np.int32)
    for i, bk in enumerate(buckets):
        wave_off[i + 1] = wave_off[i] + len(bk)
    return CallGraph(
        names=names, fns=[defined[n] for n in names], n_params=n_params, globals=gnames,
        init_bits=init_bits, init_len=init_len, init_list=init_list, direct=direct,
        src_off=src_off, src=np.array(src_rows, dtype=np.int32).reshape(-1, 4),
        slist=np.array(slist, dtype=np.int16), bind=np.array(bind, dtype=np.int32).reshape(-1, 2),
        wave_off=wave_off, wave_fns=np.array([f for bk in buckets for f in bk], dtype=np.int32),
        pess=pess)


# ---- engine call ---------------------------------------------------------------

class CgIn(C.Structure):
    _fields_ = [("n_funcs", C.c_int32), ("n_slots", C.c_int32), ("n_params", C.c_int32),
                ("n_waves", C.c_int32), ("max_passes", C.c_int32),
                ("init_bits", C.c_void_p), ("init_list", C.c_void_p), ("init_len", C.c_void_p),
                ("direct", C.c_void_p), ("src_off", C.c_void_p), ("src", C.c_void_p),
                ("slist", C.c_void_p), ("bind", C.c_void_p), ("wave_off", C.c_void_p),
                ("wave_fns", C.c_void_p), ("n_src", C.c_int64), ("n_slist", C.c_int64),
                ("n_bind", C.c_int64)]


class CgOut(C.Structure):
    _fields_ = [("bits", C.c_void_p), ("list", C.c_void_p), ("len", C.c_void_p),
                ("passes", C.c_int32), ("launches", C.c_int32), ("kernel_ms", C.c_float)]


def cg_struct(g: CallGraph, keep: list, max_passes: int) -> CgIn:
    arrs = [np.ascontiguousarray(a) for a in (
        g.init_bits, g.init_list, g.init_len, g.direct, g.src_off, g.src, g.slist, g.bind,
        g.wave_off, g.wave_fns)]
    keep.extend(arrs)
    p = [a.ctypes.data if a.size else None for a in arrs]
    return CgIn(g.n_funcs, g.init_bits.shape[1], g.n_params, g.wave_off.shape[0] - 1,
                max_passes, *p, g.src.shape[0], g.slist.shape[0], g.bind.shape[0])


@dataclass
class CgResult:
    bits: np.ndarray     # uint8 [n_funcs, n_slots]
    list: np.ndarray     # int16 [n_funcs, n_slots]
    len: np.ndarray      # int32 [n_funcs]
    passes: int
    launches: int
    kernel_ms: float


def solve_call_graph(g: CallGraph, runner=None, max_call_depth: int = 16) -> CgResult:
    """Replay the reference's summary passes (`interproc.py:105-143`).
    `runner(cg_in, cg_out) -> rc` defaults to the CUDA engine."""
    keep: list = []
    cin = cg_struct(g, keep, max(max_call_depth, g.n_funcs + 1))
    bits = np.zeros(g.init_bits.shape, dtype=np.uint8)
    lst = np.zeros(g.init_list.shape, dtype=np.int16)
    ln = np.zeros(g.n_funcs, dtype=np.int32)
    cout = CgOut(bits.ctypes.data, lst.ctypes.data, ln.ctypes.data, 0, 0, 0.0)
    if runner is None:
        eng = _abi.engine()
        eng.lib.dfx_summaries.restype = C.c_int
        eng.check(eng.lib.dfx_summaries(eng.h, C.byref(cin), C.byref(cout)), "dfx_summaries")
    else:
        rc = runner(cin, cout)
        if rc != 0:
            raise _abi.EngineError("summary runner failed (%d)" % rc)
    return CgResult(bits, lst, ln, cout.passes, cout.launches, cout.kernel_ms)


# ---- CallSummary reconstruction -----------------------------------------------

def summaries_from_result(g: CallGraph, r: CgResult) -> dict:
    """Engine rows -> `CallSummary` objects with the reference's dict order:
    declared-but-undefined first, then defined (`:102-104`); inside a summary,
    `param_effects` / `global_effects` in insertion order."""
    out: dict[str, CallSummary] = dict(g.pess)
    P = g.n_params
    eff_of = [Effect(_bits_kind(b), _bits_spaces(b)) for b in range(16)]   # frozen: shareable
    lens = r.len.tolist()
    globs = g.globals
    for f, name in enumerate(g.names):
        s = CallSummary(fn=name, defined=True)
        n = lens[f]
        if n:
            slots = r.list[f, :n].tolist()
            bits = r.bits[f].tolist()
            pe, ge = s.param_effects, s.global_effects
            for slot in slots:
                eff = eff_of[bits[slot] & 15]
                if slot < P:
                    pe[slot] = eff
                else:
                    ge[globs[slot - P]] = eff
        out[name] = s
    return out


def summarize_all(src, tu, cfgs, accesses, table, max_call_depth: int = 16,
                  runner=None) -> dict:
    """Drop-in for `dartomp.interproc.summarize_all` (`interproc.py:90`)."""
    g = lower_call_graph(src, tu, cfgs, accesses, table)
    r = solve_call_graph(g, runner=runner, max_call_depth=max_call_depth)
    return summaries_from_result(g, r)
