"""Batched directive emission on the native emitter
(`csrc/emit.cpp`, `dfx_emit_batch`): drop-ins for the reference's
`rewriter.apply_plans` (`dartomp/rewriter.py:255-274`) and
`report.plan_lines` (`dartomp/report.py:13-39`), plus `emit_batch` for many
translation units in one native call.

Output is byte-identical to the reference's, errors included:
`PreconditionError` for a loop without a braced body, `InternalError` for
conflicting update directions at one point and for plan positions the
rewriter does not place.  `report.plan_lines` has no entry for an AFTER
update (`report.py:35`) and raises `KeyError('after')`; `plan_lines` keeps
that behaviour by default (`on_after="raise"`) and, with `on_after="line"`,
reports the update as `update\\tfrom(x)\\tafter line N` instead.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._host import import_dartomp

import_dartomp()
from dartomp.dataflow import AFTER, BEFORE, BODY_END, KERNEL, PlanKind  # noqa: E402
from dartomp.diagnostics import InternalError, PreconditionError  # noqa: E402
from dartomp.nodes import NodeKind  # noqa: E402
from dartomp.rewriter import RewriteResult  # noqa: E402

_POS = {BEFORE: _abi.POS_BEFORE, AFTER: _abi.POS_AFTER, BODY_END: _abi.POS_BODY_END,
        KERNEL: _abi.POS_KERNEL}
_POS_NAME = {v: k for k, v in _POS.items()}
_UPD = {PlanKind.UPDATE_TO: 0, PlanKind.UPDATE_FROM: 1}
_KCL = {PlanKind.MAP_TO: 0, PlanKind.MAP_TOFROM: 1, PlanKind.MAP_FROM: 2, PlanKind.MAP_ALLOC: 3,
        PlanKind.FIRSTPRIVATE: 4}
EMIT_REPORT, EMIT_AFTER_LINES = 1, 2
ERR_BRACES, ERR_CLASH, ERR_POSITION = 1, 2, 3


class EmitIn(C.Structure):
    _fields_ = [("n_units", C.c_int32), ("text", C.c_void_p), ("text_off", C.c_void_p),
                ("unit_len", C.c_void_p), ("unit_text", C.c_void_p), ("unit_off", C.c_void_p),
                ("n_fns", C.c_int32), ("fn_unit", C.c_void_p), ("fn_region", C.c_void_p),
                ("fn_clause", C.c_void_p), ("fn_name", C.c_void_p), ("fn_supp_off", C.c_void_p),
                ("supp_idx", C.c_void_p), ("n_plans", C.c_int32), ("plan", C.c_void_p),
                ("plan_pos", C.c_void_p), ("plan_names_off", C.c_void_p), ("name_idx", C.c_void_p),
                ("str_off", C.c_void_p), ("strpool", C.c_void_p), ("flags", C.c_int32)]


class EmitOut(C.Structure):
    _fields_ = [("text", C.c_void_p), ("text_cap", C.c_int64), ("text_off", C.c_void_p),
                ("ins", C.c_void_p), ("ins_cap", C.c_int64), ("ins_off", C.c_void_p),
                ("report", C.c_void_p), ("report_cap", C.c_int64), ("report_off", C.c_void_p),
                ("err_kind", C.c_void_p), ("err_offset", C.c_void_p), ("report_err", C.c_void_p),
                ("text_need", C.c_int64), ("ins_need", C.c_int64), ("report_need", C.c_int64)]


class _Rewrite(RewriteResult):
    """`RewriteResult` whose `placed` list is built on first use from the
    native (start, length) pairs."""

    def __init__(self, original: str, text: str, ins: np.ndarray):
        self.original = original
        self.text = text
        self._ins = ins

    def __getattr__(self, name):
        if name == "placed":
            t = self.text
            self.placed = [(s0, t[s0:s0 + n]) for s0, n in self._ins.tolist()]
            return self.placed
        raise AttributeError(name)


def _u32(s: str) -> np.ndarray:
    return np.frombuffer(s.encode("utf-32-le"), dtype=np.uint32)


class _Strings:
    def __init__(self):
        self.ids: dict[str, int] = {}
        self.items: list[str] = []

    def id(self, s: str) -> int:
        k = self.ids.get(s)
        if k is None:
            k = self.ids[s] = len(self.items)
            self.items.append(s)
        return k


def _ptr(a):
    return a.ctypes.data if a.size else None


def emit_batch(units, report: bool = True, rewrite: bool = True, on_after: str = "raise"):
    """`units`: list of (src, plans, indent_unit or None).  Returns, per unit,
    (RewriteResult | exception, report lines | exception)."""
    strs = _Strings()
    text_parts, text_off = [], [0]
    unit_len, unit_parts, unit_off = [], [], [0]
    fn_unit, fn_region, fn_clause, fn_name, supp_off, supp = [], [], [], [], [0], []
    plan, plan_pos, names_off, names = [], [], [0], []
    plan_src = []                      # plan objects, for error messages
    ids, items = strs.ids, strs.items
    pos_get, kcl_get, upd_get = _POS.get, _KCL.get, _UPD.get
    plan_app, pos_app, names_app, noff_app = plan.append, plan_pos.append, names.append, names_off.append
    body_end, compound = _abi.POS_BODY_END, NodeKind.COMPOUND_STMT
    for u, (src, plans, indent_unit) in enumerate(units):
        t = _u32(src.text)
        text_parts.append(t)
        text_off.append(text_off[-1] + t.shape[0])
        if indent_unit is None:
            unit_len.append(-1)
            unit_off.append(unit_off[-1])
        else:
            w = _u32(indent_unit)
            unit_parts.append(w)
            unit_len.append(w.shape[0])
            unit_off.append(unit_off[-1] + w.shape[0])
        for fp in plans:
            f = len(fn_unit)
            fn_unit.append(u)
            r = fp.region
            if r is None:
                fn_region += [-1, -1]
                fn_clause.append(strs.id(""))
            else:
                fn_region += [r.begin.span.start, r.end.span.end]
                fn_clause.append(strs.id(r.clause_text()))
            fn_name.append(strs.id(fp.function.name))
            for nme in fp.suppressed:
                supp.append(strs.id(nme))
            supp_off.append(len(supp))
            groups: dict[int, int] = {}
            for cls, lst in ((1, fp.kernel_clauses), (0, fp.updates)):
                for p in lst:
                    a = p.anchor
                    sp = a.span
                    pos = pos_get(p.position, 99)
                    brace = -1
                    if cls:
                        kind = kcl_get(p.kind, 4)
                        grp = groups.setdefault(id(a), len(groups))
                    else:
                        kind = upd_get(p.kind, 0)
                        grp = 0
                        if pos == body_end:
                            body = getattr(a, "body", None)
                            if body is not None and body.kind is compound:
                                brace = body.span.end - 1
                    plan_app((f, cls, kind, pos, grp, 0))
                    pos_app((sp.start, sp.end, brace))
                    for nme in p.names:
                        k = ids.get(nme)
                        if k is None:
                            k = ids[nme] = len(items)
                            items.append(nme)
                        names_app(k)
                    noff_app(len(names))
                    plan_src.append(p)
    if not strs.items:
        strs.id("")
    pool_parts = [_u32(s) for s in strs.items]
    str_off = np.zeros(len(pool_parts) + 1, dtype=np.int64)
    str_off[1:] = np.cumsum([x.shape[0] for x in pool_parts])
    arr = {
        "text": np.concatenate(text_parts) if text_parts else np.zeros(0, np.uint32),
        "text_off": np.array(text_off, dtype=np.int64),
        "unit_len": np.array(unit_len, dtype=np.int32),
        "unit_text": np.concatenate(unit_parts) if unit_parts else np.zeros(0, np.uint32),
        "unit_off": np.array(unit_off, dtype=np.int64),
        "fn_unit": np.array(fn_unit, dtype=np.int32),
        "fn_region": np.array(fn_region, dtype=np.int64),
        "fn_clause": np.array(fn_clause, dtype=np.int32),
        "fn_name": np.array(fn_name, dtype=np.int32),
        "fn_supp_off": np.array(supp_off, dtype=np.int64),
        "supp_idx": np.array(supp, dtype=np.int32),
        "plan": np.array(plan, dtype=np.int32).reshape(-1, 6),
        "plan_pos": np.array(plan_pos, dtype=np.int64).reshape(-1, 3),
        "plan_names_off": np.array(names_off, dtype=np.int64),
        "name_idx": np.array(names, dtype=np.int32),
        "str_off": str_off,
        "strpool": np.concatenate(pool_parts) if pool_parts else np.zeros(0, np.uint32),
    }
    flags = (EMIT_REPORT if report else 0) | (EMIT_AFTER_LINES if on_after == "line" else 0)
    ein = EmitIn(n_units=len(units), n_fns=len(fn_unit), n_plans=len(plan), flags=flags,
                 **{k: _ptr(v) for k, v in arr.items()})
    lib = _abi.load_lib()
    lib.dfx_emit_batch.restype = C.c_int
    nu = len(units)
    # capacities from the inputs (a retry after DFX_E_NOSPC reruns the whole
    # emission): insertions <= covered lines + plans (+2 per region), report
    # <= a line per plan / function with its names
    n_lines = int(sum(src.text.count("\n") for src, _, _ in units)) + nu
    name_chars = int(str_off[-1])
    caps = [arr["text"].shape[0] + 64 * (len(plan) + 4 * len(fn_unit)) + name_chars * 4 + 1024,
            n_lines + len(plan) + 2 * len(fn_unit) + 64,
            96 * (len(plan) + 4 * len(fn_unit) + nu) + name_chars * 4 + 1024]
    while True:
        o = {"text": np.zeros(caps[0], np.uint32), "text_off": np.zeros(nu + 1, np.int64),
             "ins": np.zeros(2 * caps[1], np.int64), "ins_off": np.zeros(nu + 1, np.int64),
             "report": np.zeros(caps[2], np.uint32), "report_off": np.zeros(nu + 1, np.int64),
             "err_kind": np.zeros(max(1, nu), np.int32), "err_offset": np.zeros(max(1, nu), np.int64),
             "report_err": np.zeros(max(1, nu), np.int32)}
        eout = EmitOut(text_cap=caps[0], ins_cap=caps[1], report_cap=caps[2],
                       **{k: v.ctypes.data for k, v in o.items()})
        rc = lib.dfx_emit_batch(C.byref(ein), C.byref(eout))
        if rc == _abi.DFX_E_NOSPC:
            caps = [int(eout.text_need) + 16, int(eout.ins_need) + 16, int(eout.report_need) + 16]
            continue
        if rc != 0:
            raise _abi.EngineError("dfx_emit_batch failed (%d)" % rc)
        break
    text_all = o["text"]
    results = []
    for u, (src, plans, _) in enumerate(units):
        a, b = int(o["text_off"][u]), int(o["text_off"][u + 1])
        body = text_all[a:b].tobytes().decode("utf-32-le")
        ek = int(o["err_kind"][u])
        if ek == ERR_BRACES:
            res = PreconditionError.at(src, int(o["err_offset"][u]),
                                       "braces are required around this loop body to place an "
                                       "update directive")
        elif ek == ERR_CLASH:
            res = InternalError("conflicting update directions at one point for %s" % body)
        elif ek == ERR_POSITION:
            k = int(o["err_offset"][u])
            what = "kernel clause plan" if arr["plan"][k, 1] == 1 else "unexpected update"
            res = InternalError("%s position %r" % (what, plan_src[k].position)
                                if what == "unexpected update" else
                                "kernel clause plan with position %r" % plan_src[k].position)
        else:
            i0, i1 = int(o["ins_off"][u]), int(o["ins_off"][u + 1])
            res = _Rewrite(src.text, body, o["ins"][2 * i0:2 * i1].reshape(-1, 2))
        if not report:
            lines = None
        elif int(o["report_err"][u]):
            lines = KeyError(AFTER)
        else:
            r0, r1 = int(o["report_off"][u]), int(o["report_off"][u + 1])
            lines = o["report"][r0:r1].tobytes().decode("utf-32-le").split("\n")[:-1]
        results.append((res if rewrite else None, lines))
    return results


def apply_plans(src, plans, indent_unit: str | None = None) -> RewriteResult:
    """Drop-in for `dartomp.rewriter.apply_plans` (`rewriter.py:255-274`)."""
    res, _ = emit_batch([(src, plans, indent_unit)], report=False)[0]
    if isinstance(res, Exception):
        raise res
    return res


def plan_lines(src, plans, on_after: str = "raise") -> list[str]:
    """Drop-in for `dartomp.report.plan_lines` (`report.py:13-39`)."""
    _, lines = emit_batch([(src, plans, None)], rewrite=False, on_after=on_after)[0]
    if isinstance(lines, Exception):
        raise lines
    return lines
