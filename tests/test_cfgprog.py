"""North-star lowering of real programs (paper_2406_13881_b200/cfgprog.py):
the reference's AST-CFG + access lists -> one packed CSR problem -> kernels
(a)+(b).  Pinned to the reference itself on the monotone subset (SURVEY F5:
loops, no branches, no update hoisted in front of a loop): the fixpoint's
IN state at every statement's CFG node equals the reference analyzer's
(H, D) at that statement's planning visit, for every variable.  CUDA ==
oracle bit for bit on whole batches (fixpoint planes and requirement lists),
including programs outside the monotone subset."""
import numpy as np
import pytest

import _oracle
from paper_2406_13881_b200._host import have_dartomp

pytestmark = pytest.mark.skipif(not have_dartomp(), reason="host front end not importable")

MONO = dict(n_funcs=0, p_if=0.0, p_switch=0.0, p_jump=0.0, p_call=0.0, p_fp_clause=0.0,
            p_late_decl=0.0, p_braceless=0.0, p_loop=0.35, max_loop_depth=3, max_depth=4)


def _bits(words_row, n):
    return np.unpackbits(words_row.view(np.uint8), bitorder="little")[:n].astype(bool)


def _oracle_planes(prog):
    from paper_2406_13881_b200.csr import lists_to_planes
    n = prog.n_nodes
    R, W = _acc_planes(prog)
    g = {"row_ptr": prog.row_ptr, "col": prog.col, "kind": prog.kind, "A": R | W, "B": W,
         "USE": R, "S": prog.S}
    OH, OD, _ = _oracle.c3_solve(g)
    REQ, FP = _oracle.c3_requirements(g, OH, OD)
    assert lists_to_planes  # (the CUDA list output is compared as planes)
    return OH, OD, REQ, FP, n


def _acc_planes(prog):
    from paper_2406_13881_b200.csr import lists_to_planes
    acc = prog.acc.astype(np.int64)
    var = acc & 0x3FFF
    k = acc >> 14
    rd = np.where(k & 1, var, 0x3FFF + 1)        # the read entries
    wr = np.where(k & 2, var, 0x3FFF + 1)
    n, words = prog.n_nodes, prog.words

    def planes(sel):
        node = np.repeat(np.arange(n), np.diff(prog.acc_off))
        keep = sel <= 0x3FFF
        bits = np.zeros((n, words * 32), dtype=np.uint8)
        bits[node[keep], sel[keep]] = 1
        return np.packbits(bits, axis=1, bitorder="little").view(np.uint32).reshape(n, words).copy()
    del lists_to_planes
    return planes(rd), planes(wr)


def _in_state(prog, OH, OD, node):
    a, b = prog.row_ptr[node], prog.row_ptr[node + 1]
    if a == b:
        return (np.full(prog.words, 0xFFFFFFFF, dtype=np.uint32),
                np.zeros(prog.words, dtype=np.uint32))
    return (np.bitwise_and.reduce(OH[prog.col[a:b]], axis=0),
            np.bitwise_and.reduce(OD[prog.col[a:b]], axis=0))


def _reference_snapshots(src, cfg, accesses, table):
    """(statement, state copy) at every planning visit of the reference."""
    from dartomp.dataflow import _Analyzer

    class Snap(_Analyzer):
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            self.snaps = []
            self._in_omp = False

        def process_accesses(self, stmt, accs, record, anchor_override=None):
            if record and not self._in_omp:
                self.snaps.append((stmt, self.state.copy()))
            return super().process_accesses(stmt, accs, record, anchor_override)

        def exec_omp(self, stmt, record):
            node = self.cfg.node_of_ast.get(stmt)
            kern = node is not None and node.sub_cfg is not None
            if kern and record:
                self.snaps.append((stmt, self.state.copy()))
            prev = self._in_omp
            self._in_omp = kern
            try:
                return super().exec_omp(stmt, record)
            finally:
                self._in_omp = prev
    an = Snap(src, cfg, accesses, table)
    plan = an.run()
    return an.snaps, plan


def _monotone_cases(seeds):
    import random
    from dartomp.nodes import LOOP_KINDS
    from dartomp.pipeline import load
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    for seed in seeds:
        r = random.Random(seed)
        a = load(path="m%d.c" % seed,
                 text=generate(seed, GenConfig(n_stmts=r.randrange(6, 22), **MONO)))
        snaps, plan = _reference_snapshots(a.src, a.cfgs["main"], a.accesses["main"], a.table)
        if any(u.anchor.kind in LOOP_KINDS for u in plan.updates):
            continue               # D3: an update hoisted in front of a loop
        yield seed, a, snaps


def test_cfg_fixpoint_equals_reference_on_monotone_programs():
    from dartomp.nodes import LOOP_KINDS
    from paper_2406_13881_b200.cfgprog import lower_analysis
    n_fn = n_cmp = 0
    for seed, a, snaps in _monotone_cases(range(200)):
        prog = lower_analysis(a, ["main"])
        fg = prog.fns[0]
        if fg.status != "ok":
            continue
        OH, OD, _, _, _ = _oracle_planes(prog)
        cfg = a.cfgs["main"]
        slots = [(s, v) for s, v in enumerate(fg.vars) if v is not None]
        for stmt, st in snaps:
            if stmt.kind in LOOP_KINDS:
                continue           # loop conditions: entry and back edge visits share a node
            node = cfg.node_of_ast.get(stmt)
            assert node is not None, (seed, stmt.kind)
            ih, idd = _in_state(prog, OH, OD, fg.first[node.id])
            h, d = _bits(ih, prog.words * 32), _bits(idd, prog.words * 32)
            for s, v in slots:
                vs = st.vars.get(v)
                rh, rd = (vs.host_valid, vs.device_valid) if vs is not None else (True, False)
                assert (h[s], d[s]) == (rh, rd), (seed, stmt.kind, v.name)
                n_cmp += 1
        n_fn += 1
    assert n_fn >= 80 and n_cmp > 40_000, (n_fn, n_cmp)


def test_batch_is_block_diagonal():
    """Many functions in one problem solve exactly as each alone."""
    from dartomp.pipeline import load
    from paper_2406_13881_b200.cfgprog import lower_analysis
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    a = load(text=generate(3, GenConfig(n_funcs=12, n_globals=10, n_stmts=25, p_kernel=0.3)))
    names = list(a.cfgs)
    prog = lower_analysis(a, names)
    OH, OD, REQ, FP, _ = _oracle_planes(prog)
    ok = [f for f in prog.fns if f.status == "ok"]
    assert len(ok) >= 4
    for fg in ok:
        one = lower_analysis(a, [fg.name])
        f1 = one.fns[0]
        oh, od, rq, fp, _ = _oracle_planes(one)
        # the single-function problem has its own slot width: compare by variable
        for s, v in enumerate(fg.vars):
            if v is None:
                continue
            s1 = f1.vars.index(v)
            for i in range(fg.n_nodes):
                for big, small in ((OH, oh), (OD, od), (REQ, rq), (FP, fp)):
                    b = (big[fg.node0 + i, s >> 5] >> (s & 31)) & 1
                    t = (small[i, s1 >> 5] >> (s1 & 31)) & 1
                    assert b == t


def test_mixed_nodes_become_chains():
    """A firstprivate capture is a host read at a kernel node: the kernel's
    CFG node lowers to a chain of a host node and a kernel node (in either
    order: only each variable's own op order matters)."""
    from dartomp.pipeline import load
    from paper_2406_13881_b200.cfgprog import lower_analysis
    text = ("void f(int n, double *x) {\n  double a = 2.0;\n"
            "#pragma omp target teams distribute parallel for firstprivate(a)\n"
            "  for (int i = 0; i < n; i++) x[i] = a * x[i];\n}\n")
    a = load(text=text)
    prog = lower_analysis(a)
    fg = prog.fns[0]
    assert fg.status == "ok"
    k = [n.id for n in a.cfgs["f"].kernel_nodes()][0]
    g0 = fg.first[k]
    assert prog.node_cfg[g0] == k and prog.node_cfg[g0 + 1] == k
    assert sorted(prog.kind[g0:g0 + 2].tolist()) == [0, 1]
    assert list(prog.col[prog.row_ptr[g0 + 1]:prog.row_ptr[g0 + 2]]) == [g0]


def test_unsupported_shapes_are_reported():
    """A scalar read on the device outside a kernel's own entry reads (here
    through a call inside the region) would be firstprivate-eligible under
    the kernel-node transfer: reported, not approximated."""
    from dartomp.pipeline import load
    from paper_2406_13881_b200.cfgprog import lower_analysis
    text = ("double s;\ndouble y[64];\n"
            "void g(void) {\n#pragma omp target teams distribute parallel for\n"
            "  for (int i = 0; i < 64; i++) y[i] = s * y[i];\n}\n"
            "int main(void) {\n  s = 2.0;\n"
            "#pragma omp target teams distribute parallel for\n"
            "  for (int i = 0; i < 64; i++) y[i] = 1.0;\n"
            "  g();\n"
            "#pragma omp target teams distribute parallel for\n"
            "  for (int i = 0; i < 64; i++) y[i] = y[i] + 1.0;\n  return 0;\n}\n")
    prog = lower_analysis(load(text=text))
    st = {f.name: f.status for f in prog.fns}
    assert st["g"] == "ok"
    assert st["main"].startswith("unsupported"), st


def _corpus_and_generated():
    import pathlib
    from dartomp.pipeline import load
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    root = pathlib.Path(__file__).parent / "golden" / "corpus" / "transform"
    units = [load(path=str(p), text=p.read_text()) for p in sorted(root.glob("*.c"))]
    units += [load(text=generate(s, GenConfig(n_funcs=8, n_globals=16, n_stmts=30, p_kernel=0.3)))
              for s in range(6)]
    return units


def test_corpus_lowers():
    from paper_2406_13881_b200.cfgprog import lower_program
    items = [(n, a.src, a.cfgs[n], a.accesses[n], a.table)
             for a in _corpus_and_generated() for n in a.cfgs]
    prog = lower_program(items)
    ok = sum(f.status == "ok" for f in prog.fns)
    assert ok >= len(prog.fns) // 2, [f.status for f in prog.fns]
    assert prog.row_ptr[-1] == prog.col.shape[0]
    assert prog.acc_off[-1] == prog.acc.shape[0]
    assert (prog.col >= 0).all() and (prog.col < prog.n_nodes).all()


@pytest.mark.gpu
def test_cuda_cfg_program_equals_oracle():
    """Corpus + generated units (branches included) in ONE problem: CUDA
    fixpoint planes and requirement lists == the C restatement."""
    from paper_2406_13881_b200.cfgprog import fixpoint_planes, lower_program, solve_program
    from paper_2406_13881_b200.csr import AccSession
    items = [(n, a.src, a.cfgs[n], a.accesses[n], a.table)
             for a in _corpus_and_generated() for n in a.cfgs]
    prog = lower_program(items)
    OH, OD, REQ, FP, n = _oracle_planes(prog)
    gh, gd = fixpoint_planes(prog)
    assert np.array_equal(gh, OH) and np.array_equal(gd, OD)
    sess = AccSession()
    reqs, stats = solve_program(prog, sess)
    rl = sess.run(prog.row_ptr, prog.col, prog.kind, prog.acc_off, prog.acc, prog.S, prog.words)
    rq, fp = rl.to_planes()
    assert np.array_equal(rq, REQ) and np.array_equal(fp, FP)
    # the per-function view names the same variables at the same CFG nodes
    n_req = 0
    for fr, fg in zip(reqs, [f for f in prog.fns if f.status == "ok"]):
        for d, kind in ((fr.update_from, 0), (fr.update_to, 1)):
            for c, vs in d.items():
                nodes = [g for g in range(fg.node0, fg.node0 + fg.n_nodes)
                         if prog.node_cfg[g] == c and prog.kind[g] == kind]
                for v in vs:
                    s = fg.vars.index(v)
                    assert any((REQ[g, s >> 5] >> (s & 31)) & 1 for g in nodes)
                    n_req += 1
    assert n_req == int(sum(bin(int(x)).count("1") for x in REQ.ravel()))


@pytest.mark.gpu
def test_cuda_cfg_fixpoint_equals_reference_on_monotone_programs():
    from dartomp.nodes import LOOP_KINDS
    from paper_2406_13881_b200.cfgprog import fixpoint_planes, lower_analysis
    n_fn = 0
    for seed, a, snaps in _monotone_cases(range(200, 280)):
        prog = lower_analysis(a, ["main"])
        fg = prog.fns[0]
        if fg.status != "ok":
            continue
        OH, OD = fixpoint_planes(prog)
        cfg = a.cfgs["main"]
        for stmt, st in snaps:
            if stmt.kind in LOOP_KINDS:
                continue
            ih, idd = _in_state(prog, OH, OD, fg.first[cfg.node_of_ast[stmt].id])
            h, d = _bits(ih, prog.words * 32), _bits(idd, prog.words * 32)
            for s, v in enumerate(fg.vars):
                if v is None:
                    continue
                vs = st.vars.get(v)
                rh, rd = (vs.host_valid, vs.device_valid) if vs is not None else (True, False)
                assert (h[s], d[s]) == (rh, rd), (seed, v.name)
        n_fn += 1
    assert n_fn >= 25


def test_empty_and_trivial_units():
    """A unit whose functions have no accesses, and an empty item list."""
    from dartomp.pipeline import load
    from paper_2406_13881_b200.cfgprog import lower_analysis, lower_program
    prog = lower_program([])
    assert prog.n_nodes == 0 and prog.fns == []
    prog = lower_analysis(load(text="void f(void) { }\nint g(int x) { return 1; }\n"))
    assert all(f.status == "ok" for f in prog.fns)
    assert prog.acc.shape[0] == 0 and prog.n_nodes > 0
