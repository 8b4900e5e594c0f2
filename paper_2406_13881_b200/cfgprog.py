"""North-star lowering of real programs into kernels (a)+(b).

`north_star`: the front end lowers each program into packed CSR graphs -- the
CFG and its predecessor lists -- and each node's GEN/KILL and access sets into
uint32 bitplanes over the variable dimension, which hand-written kernels solve.
This module is that path for parsed translation units of the reference:

- the graph is the reference's own AST-CFG (`astcfg.py:507`, `AstCfg.edges`):
  one node per CFG node, predecessors from its edges, kernel nodes where the
  CFG has a sub-CFG (`AstCfg.kernel_nodes`);
- a node's accesses are the reference's `MemoryAccess` list grouped by
  `cfg_node` with the analysis' own op rules (`dataflow.py:412-494`): a device
  access outside the data region counts as a host access, `UNKNOWN` is
  skipped, READWRITE is read then write, and a kernel node carries its
  whole-object entry reads and writes (`access.kernel_rw_sets`) without its
  private / linear / loop-index variables; a scalar read and not written by
  the kernel is firstprivate-eligible (the S plane);
- many functions (of one or many units) go into ONE block-diagonal problem:
  each function's variables get function-local slots, scalars first, so one
  S plane (slots [0, max scalars)) serves every function;
- `solve_program` runs kernel (a) (fixpoint) and kernel (b) (per-node
  requirements) in one call through the access-list entry point
  (`dfx_mfp_acc`: H2D of CSR + lists, expansion, kernels, D2H of lists).

What it computes is the monotone-framework solution the north star names
(`dataflow.py:299-378` op effects, `:130-134` AND meet) over the CFG.  It
equals the reference analysis' state at every planning visit on the monotone
subset (loops, no branches, no update hoisted in front of a loop),
which `tests/test_cfgprog.py` checks against the reference itself; outside
that subset the reference's reconcile joins, dry rounds and provenance (D1,
D3, D8, D9) are not an MFP, and the directive plans come from E1 (DESIGN.md
§13).  A statement that mixes host and device ops (a firstprivate capture at
a kernel, a call whose callee offloads inside the region) becomes a chain of
graph nodes.  The one shape the two-plane encoding cannot express -- a scalar
read on the device outside a kernel's own entry reads, which the kernel-node
transfer would make firstprivate-eligible -- marks the function unsupported;
it is reported, not approximated.
"""
from __future__ import annotations

import functools
from dataclasses import dataclass, field

import numpy as np

from ._host import import_dartomp
from .csr import ACC_READ, ACC_WRITE, REQ_FP_FLAG, AccSession, CsrProblem
from .frontend import paused_gc
from .lower import (_clause_names, _enclosing_statement, _for_stmts, _Lowerer,
                    _READ_KINDS, _WRITE_KINDS)

import_dartomp()
from dartomp.access import AccessKind, Space  # noqa: E402


class Unsupported(Exception):
    """An op the host/kernel two-plane encoding cannot express."""


@dataclass
class FnGraph:
    """One function's part of a batch: graph nodes [node0, node0 + n_nodes)
    are its CFG nodes' chains in reverse postorder (`first[c]` is CFG node
    c's first graph node); slot s of the batch's variable dimension is
    `vars[s]` (None: unused by this function)."""
    name: str
    cfg: object
    node0: int = 0
    n_nodes: int = 0
    vars: list = field(default_factory=list)
    status: str = "ok"
    first: list = field(default_factory=list)   # CFG node id -> its first graph node


@dataclass
class CfgProgram:
    row_ptr: np.ndarray      # int32 [N+1] predecessor CSR
    col: np.ndarray          # int32 [nnz]
    kind: np.ndarray         # uint8 [N]: 0 host node, 1 kernel node
    acc_off: np.ndarray      # int64 [N+1]
    acc: np.ndarray          # uint16: slot | kind << 14 (1 read, 2 write, 3 both)
    S: np.ndarray            # uint32 [words]: firstprivate-eligible scalar slots
    words: int
    fns: list                # FnGraph per input function (unsupported: n_nodes 0)
    node_cfg: np.ndarray = None   # int32 [N]: the CFG node id each graph node belongs to

    @property
    def n_nodes(self) -> int:
        return int(self.row_ptr.shape[0]) - 1

    @property
    def facts(self) -> int:
        """Nodes x variables of the supported functions (the metric's facts)."""
        return sum(f.n_nodes * sum(v is not None for v in f.vars) for f in self.fns)


_HOST, _DEV = 0, 1


def _node_chain(seqs):
    """Per-variable op sequences of one CFG node -> a chain of graph nodes.

    `seqs`: {var id: (var, [(space, read, write, fp_ok)])} in op order.  A
    node carries one run per variable: consecutive ops of one space, reads
    before writes (a read after a write starts a new run, so the node's USE
    bit means "the first H/D-affecting op is a read", `dataflow.py:299-368`).
    Different variables are independent, so each variable's runs
    go to successive chain nodes of the matching kind and only its own order
    is kept.  Returns [(kind, {var id: (var, read, write)})]."""
    chain: list = []
    for k, (var, ops) in seqs.items():
        runs = []
        for sp, r, w, fp_ok in ops:
            if runs and runs[-1][0] == sp and not (r and runs[-1][2]):
                last = runs[-1]
                runs[-1] = (sp, last[1] or r, last[2] or w, last[3] and fp_ok)
            else:
                runs.append((sp, r, w, fp_ok))
        pos = 0
        for sp, r, w, fp_ok in runs:
            if sp == _DEV and r and not w and var.is_scalar and not fp_ok:
                # the kernel-node transfer would make it firstprivate-eligible
                raise Unsupported("scalar device read outside a kernel's entry reads")
            while pos < len(chain) and chain[pos][0] != sp:
                pos += 1
            if pos == len(chain):
                chain.append((sp, {}))
            chain[pos][1][k] = (var, r, w)
            pos += 1
    return chain


def _function_graph(src, cfg, accesses, table):
    """(chains per CFG node, preds per CFG node): the analysis' per-statement
    op sequences (`dataflow.py:412-494`) as graph-node chains."""
    lw = _Lowerer(src, cfg, accesses, table)
    n = len(cfg.nodes)
    preds = [[] for _ in range(n)]
    for e in cfg.edges:
        preds[e.dst].append(e.src)
    kernel_ids = lw.kernel_node_ids
    seqs: list = [dict() for _ in range(n)]

    def add(nid, var, sp, r, w, fp_ok=False):
        d = seqs[nid]
        ent = d.get(id(var))
        if ent is None:
            ent = d[id(var)] = (var, [])
        ent[1].append((sp, r, w, fp_ok))

    # kernel nodes first in each node's order: `exec_omp` (dataflow.py:456-494)
    # runs the kernel's entry reads and writes, then the statement's own
    # accesses (`process_accesses(stmt, extra)`)
    for nid in sorted(kernel_ids):
        stmt = cfg.nodes[nid].ast
        info = stmt.omp
        entry_reads, kernel_writes = lw.kernel_rw_sets(nid, stmt)
        captured = _clause_names(info, "firstprivate")
        private = _clause_names(info, "private") | _clause_names(info, "linear")
        for f in _for_stmts(stmt):
            v = lw.find_indexing_var(f)
            if v is not None:
                private.add(v)
        for var in entry_reads:
            if var.name in private:
                continue
            if var.name in captured:
                add(nid, var, _HOST, True, False)     # host_read at the kernel
            else:
                add(nid, var, _DEV, True, False, True)
        for var in kernel_writes:
            if var.name not in private and var.name not in captured:
                add(nid, var, _DEV, False, True)
    # statements' accesses (`process_accesses`, dataflow.py:412-435), in order
    for acc in accesses:
        kind = acc.kind
        if kind is AccessKind.UNKNOWN:
            continue
        if acc.space is Space.DEVICE and acc.cfg_node in kernel_ids:
            continue           # folded into the kernel's read/write sets
        sp = _HOST
        if acc.space is Space.DEVICE and lw.in_region(_enclosing_statement(acc.ast)):
            sp = _DEV
        r, w = kind in _READ_KINDS, kind in _WRITE_KINDS
        if r:
            add(acc.cfg_node, acc.var, sp, True, False)
        if w:
            add(acc.cfg_node, acc.var, sp, False, True)
    chains = [_node_chain(d) if d else [] for d in seqs]
    return chains, preds


def lower_program(items) -> CfgProgram:
    """`items`: (name, src, cfg, accesses, table) per function.  Returns one
    block-diagonal problem over all supported functions.  A CFG node becomes
    a chain of graph nodes when its statement mixes host and device ops
    (a call whose callee offloads, a firstprivate capture at a kernel): the
    chain's first node takes the CFG node's predecessors, its last node
    feeds the CFG node's successors.  The cyclic collector is paused for the
    call (`frontend.paused_gc`)."""
    with paused_gc():
        return _lower_program(items)


def _lower_program(items) -> CfgProgram:
    parts = []
    for name, src, cfg, accesses, table in items:
        fg = FnGraph(name=name, cfg=cfg)
        try:
            parts.append((fg, _function_graph(src, cfg, accesses, table)))
        except Unsupported as e:
            fg.status = "unsupported: %s" % e
            parts.append((fg, None))
    # slots: per function, scalars then the rest, in first-occurrence order
    n_sc = n_ot = 0
    split: dict = {}                  # id(FnGraph) -> (scalars, others)
    for fg, g in parts:
        if g is None:
            continue
        sc, ot = {}, {}
        for chain in g[0]:
            for _, ents in chain:
                for var, _, _ in ents.values():
                    (sc if var.is_scalar else ot).setdefault(id(var), var)
        split[id(fg)] = (list(sc.values()), list(ot.values()))
        n_sc, n_ot = max(n_sc, len(sc)), max(n_ot, len(ot))
    V = max(1, n_sc + n_ot)
    if V > 0x3FFF:
        raise ValueError("more than %d variables in one function" % 0x3FFF)
    words = ((V + 127) // 128) * 4
    bits = np.zeros(words * 32, dtype=np.uint8)
    bits[:n_sc] = 1
    S = np.packbits(bits, bitorder="little").view(np.uint32).copy()
    row_ptr, col, kind, acc_off, acc, node_cfg = [0], [], [], [0], [], []
    node0 = 0
    for fg, g in parts:
        if g is None:
            continue
        chains, preds = g
        scalars, others = split[id(fg)]
        slot = {id(v): i for i, v in enumerate(scalars)}
        slot.update({id(v): n_sc + i for i, v in enumerate(others)})
        fg.vars = [None] * V
        for v in scalars + others:
            fg.vars[slot[id(v)]] = v
        # graph node ids: every CFG node gets at least one (empty chains: a
        # host node without accesses), numbered in reverse postorder so that
        # kernel (a)'s in-order sweep meets most predecessors already final
        # and a statement's fall-through predecessor is the node before it
        order = _reverse_postorder(preds)
        first, last, nxt = [0] * len(chains), [0] * len(chains), node0
        for c_id in order:
            first[c_id] = nxt
            nxt += max(1, len(chains[c_id]))
            last[c_id] = nxt - 1
        fg.node0, fg.n_nodes = node0, nxt - node0
        fg.first = first
        for c_id in order:
            c = chains[c_id]
            nodes = c if c else [(_HOST, {})]
            for j, (sp, ents) in enumerate(nodes):
                if j == 0:
                    col.extend(last[p] for p in preds[c_id])
                else:
                    col.append(first[c_id] + j - 1)
                row_ptr.append(len(col))
                kind.append(sp)
                node_cfg.append(c_id)
                acc.extend(sorted(slot[k] | (((ACC_READ if r else 0) | (ACC_WRITE if w else 0)) << 14)
                                  for k, (var, r, w) in ents.items()))
                acc_off.append(len(acc))
        node0 = nxt
    return CfgProgram(row_ptr=np.array(row_ptr, dtype=np.int32),
                      col=np.array(col, dtype=np.int32),
                      kind=np.array(kind, dtype=np.uint8),
                      acc_off=np.array(acc_off, dtype=np.int64),
                      acc=np.array(acc, dtype=np.uint16), S=S, words=words,
                      fns=[fg for fg, _ in parts],
                      node_cfg=np.array(node_cfg, dtype=np.int32))


def _reverse_postorder(preds):
    """CFG node ids in reverse postorder from the entry (node 0); nodes the
    entry does not reach follow in id order."""
    n = len(preds)
    succ = [[] for _ in range(n)]
    for d, ps in enumerate(preds):
        for p in ps:
            succ[p].append(d)
    seen = [False] * n
    post = []
    if n:
        seen[0] = True
        stack = [(0, iter(succ[0]))]
        while stack:
            v, it = stack[-1]
            for w in it:
                if not seen[w]:
                    seen[w] = True
                    stack.append((w, iter(succ[w])))
                    break
            else:
                stack.pop()
                post.append(v)
    post.reverse()
    return post + [v for v in range(n) if not seen[v]]


def lower_analysis(analysis, names=None) -> CfgProgram:
    """`lower_program` over the functions of a `dartomp.pipeline.Analysis`."""
    names = list(analysis.cfgs) if names is None else names
    return lower_program([(n, analysis.src, analysis.cfgs[n], analysis.accesses[n],
                           analysis.table) for n in names])


class FnRequirements:
    """Kernel (b)'s answer for one function, per CFG node id: the variables
    needing a device -> host transfer before a host read (`update_from`),
    a host -> device transfer before a device read (`update_to` / map to),
    and a kernel's firstprivate captures.  Held as entry arrays (CFG node,
    variable slot, what); the per-node dicts are built when first read."""

    UPDATE_FROM, UPDATE_TO, FIRSTPRIVATE = 0, 1, 2

    def __init__(self, name, vars_, cfg_node, slot, what):
        self.name = name
        self.vars = vars_
        self.cfg_node = cfg_node        # int32 [entries]
        self.slot = slot                # int32 [entries]
        self.what = what                # uint8 [entries]

    def _by_node(self, w) -> dict:
        m = self.what == w
        out: dict = {}
        vs = self.vars
        for c, sl in zip(self.cfg_node[m].tolist(), self.slot[m].tolist()):
            out.setdefault(c, []).append(vs[sl])
        return out

    @functools.cached_property
    def update_from(self) -> dict:
        return self._by_node(self.UPDATE_FROM)

    @functools.cached_property
    def update_to(self) -> dict:
        return self._by_node(self.UPDATE_TO)

    @functools.cached_property
    def firstprivate(self) -> dict:
        return self._by_node(self.FIRSTPRIVATE)


def solve_program(prog: CfgProgram, session: AccSession | None = None):
    """Kernels (a)+(b) on the whole batch in one `dfx_mfp_acc` call.
    Returns ([FnRequirements] for the supported functions, CsrStats)."""
    sess = session or AccSession()
    rl = sess.run(prog.row_ptr, prog.col, prog.kind, prog.acc_off, prog.acc, prog.S,
                  prog.words)
    counts = np.diff(rl.row_off)
    node = np.repeat(np.arange(prog.n_nodes, dtype=np.int32), counts)   # graph node per entry
    e = rl.vars
    what = np.where(e & REQ_FP_FLAG, FnRequirements.FIRSTPRIVATE,
                    prog.kind[node].astype(np.int64)).astype(np.uint8)   # host node: from, kernel: to
    slot = (e & 0x3FFF).astype(np.int32)
    cfg_node = prog.node_cfg[node]
    out = []
    for fg in prog.fns:
        if fg.status != "ok":
            continue
        a, b = np.searchsorted(node, (fg.node0, fg.node0 + fg.n_nodes))
        out.append(FnRequirements(fg.name, fg.vars, cfg_node[a:b], slot[a:b], what[a:b]))
    return out, sess.stats


def fixpoint_planes(prog: CfgProgram):
    """Kernel (a)'s fixpoint OUT planes (H, D) [N, words] of the batch."""
    p = CsrProblem.from_acc(prog.row_ptr, prog.col, prog.kind, prog.acc_off, prog.acc,
                            prog.S, prog.words)
    try:
        p.solve()
        oh, od, _ = p.download(True, True)
    finally:
        p.close()
    return oh, od
