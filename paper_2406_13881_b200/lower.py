"""Host lowering: compile one function into an E1 replay program.

The reference analysis (`dartomp/dataflow.py:194-734`, `_Analyzer`) is a
syntax-directed abstract interpreter: it walks the AST in execution order,
forks and re-joins per-variable (host-valid, device-valid) state at branches,
and runs every loop body twice (dry round, weaken, planning round).  The
traversal order, the branch/loop structure and every per-access decision that
does not depend on run-time state are *static*; only the validity flags and
the two provenance maps (`device_producer`, `last_host_write`) are dynamic.

This module performs that static part once, on the host, and emits a compact
structured bytecode (one op per access, plus branch/loop control ops).  The
dynamic part -- per-variable state, slot aliasing (D4), the 2^depth loop
replay (F4), reconcile joins (D1), firstprivate (D2), the zero-trip skip merge
(D3), and the in-kernel Algorithm-1 hoisting against the dynamic `loc_lim`
(`bounds.py:134-193`) -- is executed by the replay engine (CUDA kernel in
`csrc/replay.cu`; CPU restatement in `oracle/replay_oracle.c`), one lane per
variable, which is exact because the analysis separates per variable
(SURVEY F3).

Opcode set (each op is four int32 words: ``op|flags<<8, a, b, c``):

=============  =========================================================
HR  var stmt site|anchor   host_read   (`dataflow.py:299-324`)
HW  var stmt               host_write  (`dataflow.py:326-330`)
DR  var stmt site|anchor   device_read (`dataflow.py:332-368`)
DW  var stmt               device_write (`dataflow.py:370-378`)
BR_BEGIN                   push branch frame, saved = cur
ARM_FORK                   cur = copy(saved); F_CAPTURE: arms += [cur]
ARM_CLOSE                  arms += [cur]  (switch: arm = slot at group end)
ARM_PASSIVE                arms += [copy(saved)] (absent else / default)
BR_END   armtab n          `_merge_arms` (`dataflow.py:525-564`); cur = arm0
LOOP_BEGIN loopstmt        `_loop_rounds` (`dataflow.py:566-590`) entry
LOOP_END  bodypc           dry->plan round switch, skip merge
ERR  kind node             statically-known error at this visit
=============  =========================================================
"""
from __future__ import annotations

import bisect
import operator
from dataclasses import dataclass, field

import numpy as np

from ._host import import_dartomp

import_dartomp()
from dartomp.access import AccessKind, Space, Storage  # noqa: E402
from dartomp.bounds import (enclosing_for_loops, find_indexing_var,  # noqa: E402
                            subscript_index_vars)
from dartomp.dataflow import compute_region_extent  # noqa: E402
from dartomp.nodes import NodeKind  # noqa: E402
from dartomp.omp import DATA_MAPPING_KINDS, KERNEL_KINDS  # noqa: E402

# ---- opcodes (must match include/dfx.h) ----------------------------------
OP_END = 0
OP_HR = 1
OP_HW = 2
OP_DR = 3
OP_DW = 4
OP_BR_BEGIN = 5
OP_ARM_FORK = 6
OP_ARM_CLOSE = 7
OP_ARM_PASSIVE = 8
OP_BR_END = 9
OP_LOOP_BEGIN = 10
OP_LOOP_END = 11
OP_ERR = 12

F_AFTER_REGION = 1 << 8   # HR: statement lies after the data region
F_OVR = 1 << 9            # HR/DR: anchor override (BODY_END, c = loop stmt)
F_FP = 1 << 10            # DR: firstprivate-eligible (scalar, not kernel-written, kernel stmt)
F_CAPTURE = 1 << 11       # ARM_FORK: the forked slot itself is the arm (if-arms, D4)
F_MAY_SKIP = 1 << 12      # LOOP_BEGIN: for/while (zero-trip skip merge, D3)

# ---- per-variable flags ----------------------------------------------------
V_SCALAR = 1
V_ALLOW_STALE = 2
V_DECL_LATE = 4           # check_decl_placement would raise (`dataflow.py:242-255`)
V_NONLOCAL = 8            # storage is not LOCAL (`_escape_liveness`, `dataflow.py:671-676`)

# function flags (dfx_fn_desc.flags)
FN_NO_ERR_SITES = 1       # no anchor of the function can raise a braces error

# ---- anchor codes (hoist tables and arm anchors) ---------------------------
AC_NODE_MASK = (1 << 20) - 1
AC_ERR = 1 << 20          # the node is the one `_normalize_anchor` failed at
AC_QUAL = 1 << 21         # loop's induction variable indexes the subscript
AC_CLEAN = 1 << 22        # no write to the variable in [loop.start, read)

# arm anchor kinds
ARM_BEFORE = 0
ARM_AFTER = 1
ARM_ERR_ARM = 2           # "braces are required around this branch arm"
ARM_ERR_LOOP = 3          # `_normalize_anchor` failed ("... loop body ...")

# static error kinds (OP_ERR) and event kinds (must match include/dfx.h)
ERR_DATAMAP = 1

POS_BEFORE = 0
POS_AFTER = 1
POS_BODY_END = 2
POS_KERNEL = 3

# statement ids: functions with fewer than 0xFFFF statements replay with 16-bit
# provenance ids (replay.cu Narrow), larger ones with 32-bit ids (Wide); the
# hoist table's 20-bit node field (DFX_AC_NODE_MASK) is the hard bound
MAX_STMTS = (1 << 20) - 2


class LoweringError(Exception):
    pass


def _clause_names(info, clause: str) -> set[str]:
    """Names listed in one clause kind (restates `dataflow.py:145-155`)."""
    names: set[str] = set()
    for cl in info.clauses:
        if cl.name != clause:
            continue
        for arg in cl.args:
            if ":" in arg:
                arg = arg.split(":", 1)[1]
            if arg.strip():
                names.add(arg.strip())
    return names


_JUMPS = (NodeKind.RETURN_STMT, NodeKind.BREAK_STMT, NodeKind.CONTINUE_STMT)
_ARRAY_SUBSCRIPT = NodeKind.ARRAY_SUBSCRIPT
# `access.reads` / `access.writes` (`access.py:44-49`) as tuples (identity tests)
_UNKNOWN = AccessKind.UNKNOWN
_by_name = operator.attrgetter("name")
_READ_KINDS = (AccessKind.READ, AccessKind.READWRITE, AccessKind.UNKNOWN)
_WRITE_KINDS = (AccessKind.WRITE, AccessKind.READWRITE, AccessKind.UNKNOWN)


@dataclass
class FnProgram:
    """One function's lowered replay program plus what the host needs to
    turn engine events back into a `FunctionPlan`."""

    fn: object
    ops: np.ndarray                      # [n_ops, 4] int32
    var_flags: np.ndarray                # [n_vars] int32 (flags | name_rank << 16)
    stmt_span: np.ndarray                # [n_stmts, 2] int32 (start, end)
    sites: np.ndarray                    # flat int32 hoist tables
    arms: np.ndarray                     # flat int32 (kind, node) pairs
    region_begin_start: int              # -1 when the function has no kernels
    n_slots: int
    max_loop_depth: int
    max_br_depth: int
    max_arms: int
    fn_flags: int = 0                    # dfx_fn_desc.flags (FN_NO_ERR_SITES)
    scoping_error: tuple | None = None   # (decl offset, message): see region_scoping_error
    vars: list = field(default_factory=list)
    stmts: list = field(default_factory=list)
    kernel_stmts: list = field(default_factory=list)
    region: tuple | None = None          # (block, begin, end)
    premapped: object = None             # first pre-annotated directive (see below)

    @property
    def n_vars(self) -> int:
        return len(self.vars)


_STMT_KINDS = frozenset({
    NodeKind.EXPR_STMT, NodeKind.DECL_STMT, NodeKind.RETURN_STMT,
    NodeKind.IF_STMT, NodeKind.SWITCH_STMT, NodeKind.FOR_STMT,
    NodeKind.WHILE_STMT, NodeKind.DO_STMT, NodeKind.OMP_DIRECTIVE,
    NodeKind.BREAK_STMT, NodeKind.CONTINUE_STMT,
})
_STMT_KIND_IDS = frozenset(id(k) for k in _STMT_KINDS)   # Enum.__hash__ is Python-level


def _enclosing_statement(ast):
    """`access.enclosing_statement` (`access.py:147-160`) with its statement-
    kind set built once instead of per call."""
    node = ast
    kinds = _STMT_KIND_IDS
    while node is not None:
        if id(node.kind) in kinds:
            return node
        node = node.parent
    return ast


def _for_stmts(root):
    """`root.find_all(NodeKind.FOR_STMT)` in the same (pre-)order, iteratively
    (expression subtrees, which hold no statement, are not entered)."""
    out, stack = [], [root]
    for_kind, leaf = NodeKind.FOR_STMT, _NO_STMT_BELOW_IDS
    while stack:
        n = stack.pop()
        k = n.kind
        if k is for_kind:
            out.append(n)
        elif id(k) in leaf:
            continue
        stack.extend(reversed(n.children))
    return out


class _Lowerer:
    """Static half of `_Analyzer` (`dataflow.py:194-734`)."""

    def __init__(self, src, cfg, accesses, table, allow_stale=frozenset()):
        self.src = src
        self.cfg = cfg
        self.fn = cfg.function
        self.accesses = accesses
        self.table = table
        self.allow_stale = allow_stale
        # `dataflow.py:204-212`
        self.kernel_node_ids = {n.id for n in cfg.kernel_nodes()}
        self.kernel_stmts = [cfg.node(i).ast for i in sorted(self.kernel_node_ids)]
        self.kernel_stmts.sort(key=lambda n: n.span.start)
        self.stmt_groups: dict = {}
        for acc in accesses:
            if acc.space is Space.DEVICE and acc.cfg_node in self.kernel_node_ids:
                continue
            stmt = _enclosing_statement(acc.ast)
            self.stmt_groups.setdefault(stmt, []).append(acc)
        self.region_block = self.region_begin = self.region_end = None
        if self.kernel_stmts:
            self.region_block, self.region_begin, self.region_end = \
                compute_region_extent(self.fn, self.kernel_stmts)
        # write positions per variable, for the static `writes_between`
        # (`bounds.py:160-165`) queries of Algorithm-1 finalisation
        self._write_pos: dict[int, list[int]] = {}
        for acc in accesses:
            if acc.kind in _WRITE_KINDS:
                self._write_pos.setdefault(id(acc.var), []).append(acc.ast.span.start)
        for v in self._write_pos.values():
            v.sort()
        self.ops: list[tuple[int, int, int, int]] = []
        self.sites: list[int] = []
        self.arms: list[int] = []
        self.var_index: dict[int, int] = {}
        self.vars: list = []
        self.stmt_index: dict[int, int] = {}
        self.stmts: list = []
        self._site_cache: dict = {}
        self._dev_read_sub: dict | None = None
        self._dev_by_node: dict | None = None
        self._fiv_cache: dict = {}
        self._norm_cache: dict = {}
        self._levels_cache: dict = {}
        self._loops_cache: dict = {}
        self._idx_cache: dict = {}
        self._decl_anc: dict = {}
        # structural bounds for engine resources
        self.loop_depth = 0
        self.max_loop_depth = 0
        self.br_depth = 0
        self.max_br_depth = 0
        self.max_arms = 0
        self.may_err = False    # some anchor can raise a braces error
        self.live = 1       # slot references held (cur)
        self.max_live = 1

    # ---- interning ------------------------------------------------------
    def sid(self, node) -> int:
        k = id(node)
        i = self.stmt_index.get(k)
        if i is None:
            i = len(self.stmts)
            if i >= MAX_STMTS:
                raise LoweringError("function has more than %d statements" % MAX_STMTS)
            self.stmt_index[k] = i
            self.stmts.append(node)
        return i

    def vid(self, var) -> int:
        k = id(var)
        i = self.var_index.get(k)
        if i is None:
            i = len(self.vars)
            self.var_index[k] = i
            self.vars.append(var)
        return i

    def emit(self, op: int, a: int = 0, b: int = 0, c: int = 0) -> int:
        self.ops.append((op, a, b, c))
        return len(self.ops) - 1

    # ---- region geometry (`dataflow.py:231-240`) ------------------------
    def in_region(self, stmt) -> bool:
        if self.region_begin is None:
            return False
        return (stmt.span.start >= self.region_begin.span.start
                and stmt.span.end <= self.region_end.span.end)

    def after_region(self, stmt) -> bool:
        if self.region_end is None:
            return False
        return stmt.span.start > self.region_end.span.end

    # ---- anchors ---------------------------------------------------------
    def norm_code(self, anchor) -> int:
        """`_normalize_anchor` (`dataflow.py:278-295`) as a static code."""
        k = id(anchor)
        if k in self._norm_cache:
            return self._norm_cache[k]
        node = anchor
        code = None
        while node.parent is not None:
            p = node.parent
            if p.kind in (NodeKind.COMPOUND_STMT, NodeKind.FUNCTION_DEF):
                code = self.sid(node)
                break
            if p.kind in (NodeKind.IF_STMT, NodeKind.OMP_DIRECTIVE, NodeKind.SWITCH_STMT):
                node = p
                continue
            if p.kind is NodeKind.FOR_STMT and node is not p.body:
                node = p
                continue
            code = self.sid(node) | AC_ERR
            self.may_err = True
            break
        if code is None:
            code = self.sid(node)
        self._norm_cache[k] = code
        return code

    def writes_between(self, var, begin: int, end: int) -> bool:
        pos = self._write_pos.get(id(var))
        if not pos:
            return False
        i = bisect.bisect_left(pos, begin)
        return i < len(pos) and pos[i] < end

    def site(self, access_stmt, subscript, var) -> int:
        """Static Algorithm-1 table for one (read site, variable).

        `_hoist` = `find_update_insert_loc` (`bounds.py:134-157`) +
        `finalize_update_anchor` (`bounds.py:168-193`) + `_normalize_anchor`;
        only `loc_lim` is dynamic, so per enclosing for-level we store the
        loop start, whether its induction variable indexes the subscript, and
        whether the variable is written in [loop.start, read) -- the engine
        picks the level from `loc_lim` at run time.
        """
        key = (id(access_stmt), id(subscript), id(var))
        off = self._site_cache.get(key)
        if off is not None:
            return off
        off = len(self.sites)
        acc_code = self.norm_code(access_stmt)
        if subscript is None:
            self.sites.extend([0, acc_code])
        else:
            # per (statement, index text), not per variable: each enclosing
            # for-level's start and anchor code with its qualification bit.
            # The index variables depend only on the subscript's index
            # expressions, so subscripts with the same index text (`x[i]`,
            # `y[i]`) share one entry.
            base = subscript
            while base.kind is _ARRAY_SUBSCRIPT:
                base = base.children[0]
            itext = self.src.text[base.span.end:subscript.span.end]
            k2 = (id(access_stmt), itext)
            levels = self._levels_cache.get(k2)
            if levels is None:
                k = id(access_stmt)         # per statement: loop start, code, indexing var
                loops = self._loops_cache.get(k)
                if loops is None:
                    loops = self._loops_cache[k] = [
                        (f.span.start, self.norm_code(f), self.find_indexing_var(f))
                        for f in enclosing_for_loops(access_stmt, stop_at=self.fn)]
                idx_vars = self._idx_cache.get(itext)
                if idx_vars is None:
                    idx_vars = self._idx_cache[itext] = subscript_index_vars(subscript)
                levels = self._levels_cache[k2] = [
                    (start, code | AC_QUAL if v is not None and v in idx_vars else code)
                    for start, code, v in loops]
            read_pos = access_stmt.span.start
            sites = self.sites
            sites.extend([len(levels), acc_code])
            pos = self._write_pos.get(id(var))
            for start, code in levels:
                # `writes_between(var, loop start, read)` (bounds.py:160-165)
                if pos:
                    i = bisect.bisect_left(pos, start)
                    if not (i < len(pos) and pos[i] < read_pos):
                        code |= AC_CLEAN
                else:
                    code |= AC_CLEAN
                sites.extend([start, code])
        self._site_cache[key] = off
        return off

    def find_indexing_var(self, f):
        """`bounds.find_indexing_var`, memoised per loop statement."""
        k = id(f)
        if k not in self._fiv_cache:
            self._fiv_cache[k] = find_indexing_var(f)
        return self._fiv_cache[k]

    def kernel_rw_sets(self, node_id, kernel_ast):
        """`access.kernel_rw_sets` (`access.py:405-427`) over the kernel
        node's device accesses only (grouped once per function, in access
        order) instead of a scan of every access per kernel."""
        by = self._dev_by_node
        if by is None:
            by = self._dev_by_node = {}
            for acc in self.accesses:
                if acc.space is Space.DEVICE:
                    by.setdefault(acc.cfg_node, []).append(acc)
        # the reference's loop (`access.py:405-427`) with `decl_is_inside`
        # (`access.py:163-166`, an ancestor walk) answered once per variable
        written: set = set()
        seen_reads: set = set()
        entry_reads: list = []
        writes_out: list = []
        inside: dict = {}
        anc = self._decl_anc
        kid = id(kernel_ast)
        ks, ke = kernel_ast.span.start, kernel_ast.span.end
        for acc in by.get(node_id, ()):
            var = acc.var
            k = id(var)
            ins = inside.get(k)
            if ins is None:
                d = var.decl
                if d is None:
                    ins = False
                elif d.span.start < ks or d.span.end > ke:
                    ins = False     # a descendant's span nests in its ancestors'
                else:
                    a = anc.get(id(d))
                    if a is None:      # the declaration and its ancestors' ids, once per function
                        a = anc[id(d)] = {id(x) for x in d.ancestors()} | {id(d)}
                    ins = kid in a
                inside[k] = ins
            if ins:
                continue
            kind = acc.kind
            if kind in _READ_KINDS and var not in written and var not in seen_reads:
                entry_reads.append(var)
                seen_reads.add(var)
            if kind in _WRITE_KINDS:
                if var not in written:
                    writes_out.append(var)
                written.add(var)
        return entry_reads, writes_out

    def device_read_subscript(self, var, kernel_stmt):
        """`_device_read_subscript` (`dataflow.py:380-390`): the subscript of
        the first device read of `var` at the kernel's node, in access order
        (indexed once per function instead of a scan per call)."""
        node = self.cfg.node_of_ast.get(kernel_stmt)
        if node is None:
            return None
        idx = self._dev_read_sub
        if idx is None:
            idx = self._dev_read_subscripts()
        return idx.get((node.id, id(var)))

    def _dev_read_subscripts(self) -> dict:
        idx = self._dev_read_sub = {}
        for acc in self.accesses:
            if (acc.space is Space.DEVICE and acc.kind in _READ_KINDS
                    and acc.subscript is not None):
                idx.setdefault((acc.cfg_node, id(acc.var)), acc.subscript)
        return idx

    # ---- access ops ------------------------------------------------------
    def op_hr(self, var, stmt, subscript, override):
        flags = OP_HR
        if self.after_region(stmt):
            flags |= F_AFTER_REGION
        if override is not None:
            flags |= F_OVR
            c = self.sid(override)
        else:
            c = self.site(stmt, subscript, var)
        self.emit(flags, self.vid(var), self.sid(stmt), c)

    def op_dr(self, var, stmt, kernel_writes, override):
        flags = OP_DR
        if (var.is_scalar and var not in kernel_writes
                and stmt.kind is NodeKind.OMP_DIRECTIVE):
            flags |= F_FP
        if override is not None:
            flags |= F_OVR
            c = self.sid(override)
        else:
            c = self.site(stmt, self.device_read_subscript(var, stmt), var)
        self.emit(flags, self.vid(var), self.sid(stmt), c)

    def op_hw(self, var, stmt):
        self.emit(OP_HW, self.vid(var), self.sid(stmt), 0)

    def op_dw(self, var, stmt):
        self.emit(OP_DW, self.vid(var), self.sid(stmt), 0)

    # ---- traversal (mirrors `dataflow.py:394-667`) -------------------------
    def run(self) -> None:
        body = self.fn.body
        if body is not None:
            self.exec_block(body)
        self.emit(OP_END)

    def exec_block(self, block) -> None:
        for stmt in block.children:
            self.exec_stmt(stmt)

    def group(self, stmt):
        return self.stmt_groups.get(stmt, [])

    def accs_in(self, stmt, sub):
        return [a for a in self.group(stmt)
                if sub.span.start <= a.ast.span.start < sub.span.end]

    def process_accesses(self, stmt, accs, override=None) -> None:
        inside = self.in_region(stmt)
        for acc in accs:
            kind = acc.kind
            if kind is _UNKNOWN:
                continue
            if acc.space is Space.HOST or not inside:
                if kind in _READ_KINDS:
                    self.op_hr(acc.var, stmt, acc.subscript, override)
                if kind in _WRITE_KINDS:
                    self.op_hw(acc.var, stmt)
            else:
                if kind in _READ_KINDS:
                    self.op_dr(acc.var, stmt, frozenset(), override)
                if kind in _WRITE_KINDS:
                    self.op_dw(acc.var, stmt)

    def exec_stmt(self, stmt) -> None:
        kind = stmt.kind
        if kind is NodeKind.COMPOUND_STMT:
            self.exec_block(stmt)
        elif kind is NodeKind.OMP_DIRECTIVE:
            self.exec_omp(stmt)
        elif kind is NodeKind.IF_STMT:
            self.exec_if(stmt)
        elif kind is NodeKind.FOR_STMT:
            self.exec_for(stmt)
        elif kind is NodeKind.WHILE_STMT:
            self.exec_while(stmt)
        elif kind is NodeKind.DO_STMT:
            self.exec_do(stmt)
        elif kind is NodeKind.SWITCH_STMT:
            self.exec_switch(stmt)
        else:
            self.process_accesses(stmt, self.group(stmt))

    def exec_omp(self, stmt) -> None:
        info = stmt.omp
        if info.kind in DATA_MAPPING_KINDS:
            self.emit(OP_ERR, ERR_DATAMAP, self.sid(stmt), 0)
            return
        node = self.cfg.node_of_ast.get(stmt)
        if node is None or node.sub_cfg is None:
            if stmt.children:
                self.exec_stmt(stmt.children[0])
            return
        entry_reads, kernel_writes = self.kernel_rw_sets(node.id, stmt)
        kw = set(kernel_writes)
        captured = _clause_names(info, "firstprivate")
        private = _clause_names(info, "private") | _clause_names(info, "linear")
        for f in _for_stmts(stmt):
            v = self.find_indexing_var(f)
            if v is not None:
                private.add(v)
        # `op_dr` / `op_dw` inline: the subscript of each variable's first
        # device read at this kernel node (`_device_read_subscript`)
        sub = self._dev_read_sub
        if sub is None:
            sub = self._dev_read_subscripts()
        nid = node.id
        s_stmt = self.sid(stmt)
        ops, vid, site = self.ops, self.vid, self.site
        for var in sorted(entry_reads, key=_by_name):
            name = var.name
            if name in private:
                continue
            if name in captured:
                self.op_hr(var, stmt, None, None)
                continue
            flags = OP_DR | F_FP if (var.is_scalar and var not in kw) else OP_DR
            ops.append((flags, vid(var), s_stmt, site(stmt, sub.get((nid, id(var))), var)))
        for var in sorted(kernel_writes, key=_by_name):
            name = var.name
            if name in private or name in captured:
                continue
            ops.append((OP_DW, vid(var), s_stmt, 0))
        extra = list(self.group(stmt))
        if extra:
            self.process_accesses(stmt, extra)

    # -- branches --
    def _br_begin(self):
        self.emit(OP_BR_BEGIN)
        self.br_depth += 1
        self.max_br_depth = max(self.max_br_depth, self.br_depth)
        self.live += 1                      # saved

    def _hold(self, n=1):
        self.live += n
        self.max_live = max(self.max_live, self.live + 1)

    def _br_end(self, anchors) -> None:
        off = len(self.arms)
        for a in anchors:
            self.arms.extend(a)
        self.emit(OP_BR_END, off // 2, len(anchors), 0)
        self.br_depth -= 1
        self.max_arms = max(self.max_arms, len(anchors))
        self.live -= 1 + len(anchors)       # saved + arms released, cur kept

    def arm_anchor(self, arm, branch_stmt):
        """`_arm_anchor` (`dataflow.py:512-523`) with the `None` case already
        resolved to `(BEFORE, normalize(branch))` (`dataflow.py:551-552`)."""
        if arm is None:
            return self._none_anchor(branch_stmt)
        if arm.kind is NodeKind.COMPOUND_STMT:
            if not arm.children:
                return self._none_anchor(branch_stmt)
            last = arm.children[-1]
            if last.kind in _JUMPS:
                return (ARM_BEFORE, self.sid(last))
            return (ARM_AFTER, self.sid(last))
        if arm.kind in _JUMPS:
            return self._none_anchor(branch_stmt)
        self.may_err = True
        return (ARM_ERR_ARM, self.sid(arm))

    def _none_anchor(self, branch_stmt):
        code = self.norm_code(branch_stmt)
        if code & AC_ERR:
            return (ARM_ERR_LOOP, code & AC_NODE_MASK)
        return (ARM_BEFORE, code)

    def group_anchor(self, group, branch_stmt):
        """`_group_anchor` (`dataflow.py:661-667`)."""
        if not group:
            return self._none_anchor(branch_stmt)
        last = group[-1]
        if last.kind in _JUMPS:
            return (ARM_BEFORE, self.sid(last))
        return (ARM_AFTER, self.sid(last))

    def exec_if(self, stmt) -> None:
        self.process_accesses(stmt, self.group(stmt))
        self._br_begin()
        self.emit(OP_ARM_FORK | F_CAPTURE)
        self._hold(2)                       # arm0 + new cur
        self.exec_stmt(stmt.then_branch)
        anchors = [self.arm_anchor(stmt.then_branch, stmt)]
        if stmt.else_branch is not None:
            self.emit(OP_ARM_FORK | F_CAPTURE)
            self._hold(2)
            self.exec_stmt(stmt.else_branch)
            anchors.append(self.arm_anchor(stmt.else_branch, stmt))
            self.live -= 1
        else:
            self.emit(OP_ARM_PASSIVE)
            self._hold(1)
            anchors.append(self._none_anchor(stmt))
        self.live -= 1
        self._br_end(anchors)

    def exec_switch(self, stmt) -> None:
        self.process_accesses(stmt, self.group(stmt))
        body = stmt.body
        if body is None or body.kind is not NodeKind.COMPOUND_STMT:
            if body is not None:
                self.exec_stmt(body)
            return
        groups: list[list] = []
        has_default = False
        for child in body.children:
            if child.kind is NodeKind.CASE_LABEL:
                groups.append([])
                if child.value is None:
                    has_default = True
                continue
            if not groups:
                groups.append([])
            groups[-1].append(child)
        if not groups and has_default:     # unreachable: has_default implies a group
            return
        self._br_begin()
        anchors = []
        for group in groups:
            self.emit(OP_ARM_FORK)
            self._hold(1)
            for s in group:
                self.exec_stmt(s)
            self.emit(OP_ARM_CLOSE)
            self._hold(1)
            self.live -= 1                  # cur reference transferred to arm
            anchors.append(self.group_anchor(group, stmt))
        if not has_default:
            self.emit(OP_ARM_PASSIVE)
            self._hold(1)
            anchors.append(self._none_anchor(stmt))
        self._br_end(anchors)

    # -- loops --
    def _loop(self, stmt, may_skip: bool, body_fn) -> None:
        flags = OP_LOOP_BEGIN | (F_MAY_SKIP if may_skip else 0)
        begin = self.emit(flags, self.sid(stmt), 0, 0)
        self.loop_depth += 1
        self.max_loop_depth = max(self.max_loop_depth, self.loop_depth)
        self._hold(2)                       # entry/weakened + a stale round-0 cur
        body_fn()
        self.emit(OP_LOOP_END, begin + 1, 0, 0)
        self.live -= 2
        self.loop_depth -= 1

    def exec_for(self, stmt) -> None:
        self.exec_stmt(stmt.for_init)
        cond_accs = self.accs_in(stmt, stmt.for_cond)
        inc_accs = self.accs_in(stmt, stmt.for_inc)
        self.process_accesses(stmt, cond_accs)

        def body():
            self.exec_stmt(stmt.body)
            self.process_accesses(stmt, inc_accs)
            self.process_accesses(stmt, cond_accs, override=stmt)
        self._loop(stmt, True, body)

    def exec_while(self, stmt) -> None:
        cond_accs = self.accs_in(stmt, stmt.cond)
        self.process_accesses(stmt, cond_accs)

        def body():
            self.exec_stmt(stmt.body)
            self.process_accesses(stmt, cond_accs, override=stmt)
        self._loop(stmt, True, body)

    def exec_do(self, stmt) -> None:
        cond_accs = self.accs_in(stmt, stmt.cond)

        def body():
            self.exec_stmt(stmt.body)
            self.process_accesses(stmt, cond_accs, override=stmt)
        self._loop(stmt, False, body)

    # ---- packing ---------------------------------------------------------
    def finish(self) -> FnProgram:
        # name ranks: the reference sorts by name in `_merge_arms`
        order = sorted(range(len(self.vars)), key=lambda i: (self.vars[i].name, i))
        rank = [0] * len(self.vars)
        for r, i in enumerate(order):
            rank[i] = r
        flags = []
        for i, v in enumerate(self.vars):
            f = 0
            if v.is_scalar:
                f |= V_SCALAR
            if v.name in self.allow_stale:
                f |= V_ALLOW_STALE
            if (v.storage is Storage.LOCAL and v.decl is not None
                    and self.region_begin is not None
                    and v.decl.span.start >= self.region_begin.span.start):
                f |= V_DECL_LATE
            if v.storage is not Storage.LOCAL:
                f |= V_NONLOCAL
            flags.append(f | (rank[i] << 16))
        span = np.array([[s.span.start, s.span.end] for s in self.stmts],
                        dtype=np.int32).reshape(-1, 2)
        ops = np.array(self.ops, dtype=np.int32).reshape(-1, 4)
        n_slots = self.max_live + 2 * self.max_loop_depth + 2
        return FnProgram(
            fn=self.fn, ops=ops, var_flags=np.array(flags, dtype=np.int32),
            stmt_span=span, sites=np.array(self.sites, dtype=np.int32),
            arms=np.array(self.arms, dtype=np.int32),
            region_begin_start=(self.region_begin.span.start
                                if self.region_begin is not None else -1),
            n_slots=n_slots, max_loop_depth=self.max_loop_depth,
            max_br_depth=self.max_br_depth, max_arms=self.max_arms,
            fn_flags=0 if self.may_err else FN_NO_ERR_SITES,
            scoping_error=(region_scoping_error(self.src, self.accesses, self.region_begin,
                                               self.region_end)
                           if self.region_begin is not None else None),
            vars=self.vars, stmts=self.stmts, kernel_stmts=self.kernel_stmts,
            region=((self.region_block, self.region_begin, self.region_end)
                    if self.region_begin is not None else None))


def region_scoping_error(src, accesses, begin, end):
    """`_Analyzer._check_region_scoping` (`dataflow.py:713-734`) as data: the
    DeclPlacementError it raises for a region over [begin, end] -- (offset,
    message) -- or None.  Static (declarations and accesses only), so the
    lowering computes it and `_finish` raises it only if the plan opens a
    region."""
    lo = begin.span.start
    hi = end.span.end
    inside = {}
    for acc in accesses:
        d = acc.var.decl
        if d is None or not (lo <= d.span.start < hi):
            continue
        if acc.ast.span.start >= hi and acc.ast is not d:
            inside.setdefault(acc.var, acc)
    for var, acc in sorted(inside.items(), key=lambda kv: kv[0].name):
        return (var.decl.span.start,
                "'%s' is declared at line %d inside the new data region "
                "(lines %d..%d) but used at line %d after it; move the "
                "declaration above the region" % (
                    var.name, src.line_of(var.decl.span.start),
                    src.line_of(lo), src.line_of(hi - 1),
                    src.line_of(acc.ast.span.start)))
    return None


def premapped_directive(root):
    """First OpenMP directive under `root`, in the pre-order of
    `AstNode.walk` (`nodes.py:108-111`), that `check_transform_preconditions`
    (`pipeline.py:65-82`) refuses: a data-mapping construct, or an offload
    directive that already has a `map` clause.  None if there is none.
    Iterative, so the batched lowering can run the check per function in its
    workers instead of one recursive generator walk over the whole unit."""
    omp_kind = NodeKind.OMP_DIRECTIVE
    leaf = _NO_STMT_BELOW_IDS
    stack = [root]
    while stack:
        node = stack.pop()
        kind = node.kind
        if kind is omp_kind and node.omp is not None:
            info = node.omp
            if info.kind in DATA_MAPPING_KINDS or (
                    info.kind in KERNEL_KINDS and info.clause("map") is not None):
                return node
        if id(kind) in leaf:
            continue
        ch = node.children
        if ch:
            stack.extend(reversed(ch))
    return None


# node kinds whose subtrees hold expressions and declarators only: no
# statement -- in particular no pragma (`parser.py:293-298`) and no loop --
# lies below them, so the pre-order walks for directives and for-statements
# need not enter them
_NO_STMT_BELOW = frozenset({
    NodeKind.EXPR_STMT, NodeKind.DECL_STMT, NodeKind.RETURN_STMT, NodeKind.VAR_DECL,
    NodeKind.PARAM_DECL, NodeKind.STRUCT_DECL, NodeKind.BINARY_OP, NodeKind.UNARY_OP,
    NodeKind.ASSIGN_OP, NodeKind.ARRAY_SUBSCRIPT, NodeKind.MEMBER_ACCESS, NodeKind.CALL,
    NodeKind.DECL_REF, NodeKind.INT_LITERAL, NodeKind.FLOAT_LITERAL, NodeKind.STRING_LITERAL,
    NodeKind.INIT_LIST, NodeKind.CAST, NodeKind.EMPTY,
})
_NO_STMT_BELOW_IDS = frozenset(id(k) for k in _NO_STMT_BELOW)   # Enum.__hash__ is Python-level


def lower_function(src, cfg, accesses, table, allow_stale=frozenset()) -> FnProgram:
    lw = _Lowerer(src, cfg, accesses, table, allow_stale)
    lw.run()
    prog = lw.finish()
    prog.premapped = premapped_directive(cfg.function)
    return prog
