"""Syntax-directed CSR of a monotone-subset function, and the reference's own
in-states at every planning visit (TEST INFRASTRUCTURE).

SURVEY F5: on programs with loops and no branches (and no update hoisted in
front of a loop), the reference analysis' state at each `record=True` visit
equals the greatest fixpoint of the AND-meet gen/kill system on the
syntax-directed graph.  This module builds that graph -- one node per
planning visit, in the reference's visit order (loop conditions split into
the entry edge and the back edge, D7) -- with the host/kernel node encoding
of kernel (a) (A = R|W, B = W, S = firstprivate-eligible scalars), and
instruments `dartomp.dataflow._Analyzer` to snapshot (H, D) of every
variable at those same visits.
"""
from __future__ import annotations

import numpy as np

from paper_2406_13881_b200._host import import_dartomp

import_dartomp()
from dartomp.access import AccessKind, Space, kernel_rw_sets, reads, writes  # noqa: E402
from dartomp.bounds import find_indexing_var  # noqa: E402
from dartomp.dataflow import _Analyzer  # noqa: E402
from dartomp.nodes import NodeKind  # noqa: E402

from paper_2406_13881_b200.lower import _clause_names, _Lowerer  # noqa: E402


class Unsupported(Exception):
    pass


class _Walker:
    def __init__(self, src, cfg, accesses, table):
        self.lw = _Lowerer(src, cfg, accesses, table)
        self.nodes: list[dict] = []
        self.cur: list[int] = []
        self.var_index: dict[int, int] = {}
        self.vars: list = []

    def vid(self, var):
        k = id(var)
        if k not in self.var_index:
            self.var_index[k] = len(self.vars)
            self.vars.append(var)
        return self.var_index[k]

    def node(self, kind):
        n = {"kind": kind, "R": set(), "W": set(), "S": set(), "preds": list(self.cur)}
        self.nodes.append(n)
        self.cur = [len(self.nodes) - 1]
        return n

    def host(self, stmt, accs):
        n = self.node(0)
        inside = self.lw.in_region(stmt)
        for acc in accs:
            if acc.kind is AccessKind.UNKNOWN:
                continue
            space = acc.space
            if space is Space.DEVICE and not inside:
                space = Space.HOST
            if space is Space.DEVICE:
                raise Unsupported("device access in a host statement")
            v = self.vid(acc.var)
            if reads(acc.kind):
                n["R"].add(v)
            if writes(acc.kind):
                n["W"].add(v)

    def omp(self, stmt):
        lw = self.lw
        node = lw.cfg.node_of_ast.get(stmt)
        if node is None or node.sub_cfg is None:
            if stmt.children:
                self.stmt(stmt.children[0])
            return
        entry_reads, kernel_writes = kernel_rw_sets(lw.accesses, node.id, stmt)
        kw = set(kernel_writes)
        info = stmt.omp
        if _clause_names(info, "firstprivate"):
            raise Unsupported("firstprivate clause")
        private = _clause_names(info, "private") | _clause_names(info, "linear")
        for f in stmt.find_all(NodeKind.FOR_STMT):
            v = find_indexing_var(f)
            if v is not None:
                private.add(v)
        if lw.group(stmt):
            raise Unsupported("host accesses on a kernel statement")
        n = self.node(1)
        for var in entry_reads:
            if var.name in private:
                continue
            v = self.vid(var)
            n["R"].add(v)
            if var.is_scalar and var not in kw:
                n["S"].add(v)
        for var in kernel_writes:
            if var.name in private:
                continue
            n["W"].add(self.vid(var))

    def block(self, b):
        for s in b.children:
            self.stmt(s)

    def loop_body(self, stmt, fwd_first, tail):
        mark = len(self.nodes)
        self.stmt(stmt.body)
        tail()
        back = len(self.nodes) - 1
        # the first node of the loop (body, or the tail when the body is
        # empty) also receives the back edge
        self.nodes[mark]["preds"].append(back)
        return back

    def stmt(self, s):
        k = s.kind
        lw = self.lw
        if k is NodeKind.COMPOUND_STMT:
            self.block(s)
        elif k is NodeKind.OMP_DIRECTIVE:
            self.omp(s)
        elif k in (NodeKind.IF_STMT, NodeKind.SWITCH_STMT):
            raise Unsupported("branch")
        elif k is NodeKind.FOR_STMT:
            self.stmt(s.for_init)
            cond = lw.accs_in(s, s.for_cond)
            inc = lw.accs_in(s, s.for_inc)
            self.host(s, cond)
            fwd = self.cur[0]

            def tail():
                self.host(s, inc)
                self.host(s, cond)
            back = self.loop_body(s, fwd, tail)
            self.cur = [fwd, back]
        elif k is NodeKind.WHILE_STMT:
            cond = lw.accs_in(s, s.cond)
            self.host(s, cond)
            fwd = self.cur[0]
            back = self.loop_body(s, fwd, lambda: self.host(s, cond))
            self.cur = [fwd, back]
        elif k is NodeKind.DO_STMT:
            cond = lw.accs_in(s, s.cond)
            back = self.loop_body(s, None, lambda: self.host(s, cond))
            self.cur = [back]
        else:
            self.host(s, lw.group(s))


def build_graph(src, cfg, accesses, table):
    """-> (row_ptr, col, kind, R, W, S, vars) in the kernel-(a) encoding."""
    w = _Walker(src, cfg, accesses, table)
    if cfg.function.body is not None:
        w.block(cfg.function.body)
    n = len(w.nodes)
    V = max(1, len(w.vars))
    words = ((V + 127) // 128) * 4
    R = np.zeros((n, words), dtype=np.uint32)
    W = np.zeros_like(R)
    S = np.zeros(words, dtype=np.uint32)
    row_ptr = np.zeros(n + 1, dtype=np.int32)
    col = []
    kind = np.zeros(n, dtype=np.uint8)
    for i, nd in enumerate(w.nodes):
        kind[i] = nd["kind"]
        for v in nd["R"]:
            R[i, v >> 5] |= np.uint32(1 << (v & 31))
        for v in nd["W"]:
            W[i, v >> 5] |= np.uint32(1 << (v & 31))
        for v in nd["S"]:
            S[v >> 5] |= np.uint32(1 << (v & 31))
        col.extend(nd["preds"])
        row_ptr[i + 1] = len(col)
    # a variable is a scalar everywhere or nowhere; firstprivate eligibility
    # additionally needs "read, not written by this kernel" = A & ~B, which
    # the kernel-node transfer applies
    for v, var in enumerate(w.vars):
        if var.is_scalar:
            S[v >> 5] |= np.uint32(1 << (v & 31))
    return row_ptr, np.array(col, dtype=np.int32), kind, R, W, S, w.vars


class _Snap(_Analyzer):
    """The reference analyzer, snapshotting (H, D) at every planning visit."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.snaps = []
        self._in_omp = False

    def _snap(self):
        self.snaps.append(self.state.copy())

    def process_accesses(self, stmt, accs, record, anchor_override=None):
        if record and not self._in_omp:
            self._snap()
        return super().process_accesses(stmt, accs, record, anchor_override)

    def exec_omp(self, stmt, record):
        node = self.cfg.node_of_ast.get(stmt)
        kern = node is not None and node.sub_cfg is not None
        if kern and record:
            self._snap()
        prev = self._in_omp
        self._in_omp = kern
        try:
            return super().exec_omp(stmt, record)
        finally:
            self._in_omp = prev


def reference_states(src, cfg, accesses, table, vars_):
    """[(H bits, D bits)] per planning visit, over the graph's variable order,
    plus the plan the reference produced."""
    an = _Snap(src, cfg, accesses, table)
    plan = an.run()
    out = []
    for st in an.snaps:
        h = np.ones(len(vars_), dtype=bool)
        d = np.zeros(len(vars_), dtype=bool)
        for i, v in enumerate(vars_):
            s = st.vars.get(v)
            if s is not None:
                h[i], d[i] = s.host_valid, s.device_valid
        out.append((h, d))
    return out, plan


def in_states(row_ptr, col, OH, OD, n_vars):
    """IN = AND over predecessors' OUT (boundary (1,0) without preds)."""
    n = row_ptr.shape[0] - 1
    res = []
    for i in range(n):
        a, b = row_ptr[i], row_ptr[i + 1]
        if a == b:
            ih = np.full(OH.shape[1], 0xFFFFFFFF, dtype=np.uint32)
            idd = np.zeros(OH.shape[1], dtype=np.uint32)
        else:
            ih = np.bitwise_and.reduce(OH[col[a:b]], axis=0)
            idd = np.bitwise_and.reduce(OD[col[a:b]], axis=0)
        bits = lambda w: np.unpackbits(w.view(np.uint8), bitorder="little")[:n_vars].astype(bool)  # noqa: E731
        res.append((bits(ih), bits(idd)))
    return res
