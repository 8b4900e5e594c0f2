"""GPU: kernels (a)+(b) (libdfx.so) against the CPU oracle, bit-exact."""
import numpy as np
import pytest

import _mfp_ref
import _oracle
from paper_2406_13881_b200.csr import AccSession, C3Config, CsrProblem, mfp_csr, planes_to_acc

pytestmark = pytest.mark.gpu


def _check(prob, g, chunk=0):
    st = prob.solve(chunk)
    OH, OD, _ = prob.download(True, True)
    eh, ed, _ = _oracle.c3_solve(g)
    assert np.array_equal(OH, eh), "H planes differ in %d words" % (OH != eh).sum()
    assert np.array_equal(OD, ed), "D planes differ in %d words" % (OD != ed).sum()
    rows = prob.requirements()
    REQ, FP = _oracle.c3_requirements(g, eh, ed)
    rq, rf = rows.to_planes()
    assert np.array_equal(rq, REQ) and np.array_equal(rf, FP)
    # order-preserving compaction: row offsets are the prefix of per-node
    # nonzero-word counts; masks follow node order, requirement words first
    cnt = (REQ != 0).sum(axis=1) + (FP != 0).sum(axis=1)
    assert np.array_equal(np.diff(rows.row_off), cnt) and rows.row_off[0] == 0
    nz = np.concatenate([REQ, FP], axis=1)
    assert np.array_equal(nz[nz != 0], rows.masks)
    return st


@pytest.mark.parametrize("words", [128, 8, 4, 256, 512])
def test_c3_generated_on_device_matches_oracle(words):
    n = 1 << 15 if words >= 256 else 1 << 16
    cfg = C3Config(n_nodes=n, n_vars=32 * words, seed=11, w0=0)
    g = _oracle.c3_generate(cfg.seed, n, cfg.w0, words, cfg.n_scalar)
    prob = CsrProblem.generate_c3(cfg)
    st = _check(prob, g)
    assert st.rounds_h >= 2 and st.rounds_d >= 2


def test_c3_shard_offset_matches_oracle():
    cfg = C3Config(n_nodes=1 << 14, n_vars=4096, seed=5, w0=128)   # rank-1 slab
    g = _oracle.c3_generate(cfg.seed, cfg.n_nodes, cfg.w0, cfg.words, cfg.n_scalar)
    _check(CsrProblem.generate_c3(cfg), g)


@pytest.mark.parametrize("chunk", [1, 7, 32, 33, 256, 4096])
def test_chunk_sizes_same_fixpoint(chunk):
    g = _oracle.c3_generate(2, 1 << 14, 0, 128, 82)
    prob = CsrProblem.from_arrays(g["row_ptr"], g["col"], g["kind"], g["USE"], g["B"], g["S"])
    _check(prob, g, chunk)


@pytest.mark.parametrize("seed", range(8))
def test_random_graphs_entries_selfloops_duplicates(seed):
    rng = np.random.default_rng(100 + seed)
    words = [4, 8, 128, 132][seed % 4]
    row_ptr, col, kind, R, W, S = _mfp_ref.random_graph(rng, 700, words)
    g = {"row_ptr": row_ptr, "col": col, "kind": kind, "A": R | W, "B": W, "USE": R, "S": S}
    prob = CsrProblem.from_arrays(row_ptr, col, kind, R, W, S)
    _check(prob, g, chunk=[1, 16, 64, 500][seed % 4])


def test_all_in_one_host_call():
    g = _oracle.c3_generate(9, 1 << 14, 0, 128, 82)
    rows, stats = mfp_csr(g["row_ptr"], g["col"], g["kind"], g["USE"], g["B"], g["S"])
    eh, ed, _ = _oracle.c3_solve(g)
    REQ, FP = _oracle.c3_requirements(g, eh, ed)
    rq, rf = rows.to_planes()
    assert np.array_equal(rq, REQ) and np.array_equal(rf, FP)
    assert stats.solve_ms > 0


def test_full_size_c3_properties():
    """1M x 4096 on the device == the oracle on ALL 128 variable words: the
    fixpoint planes OUT_H / OUT_D, kernel (b)'s requirement and firstprivate
    planes and its per-node list form (the e2e output shape), checked block
    by block (variables are independent); then idempotence."""
    cfg = C3Config()
    prob = CsrProblem.generate_c3(cfg)
    st = prob.solve()
    OH, OD, _ = prob.download(True, True)
    rq, rf = prob.requirements().to_planes()
    bad = _oracle.c3_verify(cfg.seed, cfg.n_nodes, cfg.w0, cfg.words, cfg.n_scalar,
                            OH, OD, rq, rf)
    assert bad == {"OUT_H": 0, "OUT_D": 0, "REQ": 0, "FP": 0}, bad
    lq, lf = prob.requirements_list().to_planes()
    assert np.array_equal(lq, rq) and np.array_equal(lf, rf)
    assert st.rounds_h >= 2
    # idempotence: a second solve from scratch reproduces the same fixpoint
    prob.solve()
    OH2, OD2, _ = prob.download(True, True)
    assert np.array_equal(OH2, OH) and np.array_equal(OD2, OD)


# ---- list forms (dfx_csr_create_acc / dfx_csr_requirements_list / dfx_mfp_acc)

def _check_lists(rl, g, eh, ed):
    REQ, FP = _oracle.c3_requirements(g, eh, ed)
    rq, rf = rl.to_planes()
    assert np.array_equal(rq, REQ) and np.array_equal(rf, FP)
    # per-node order: requirement vars ascending, then firstprivate ascending
    cnt = np.unpackbits(REQ.view(np.uint8), axis=1).sum(axis=1) + \
        np.unpackbits(FP.view(np.uint8), axis=1).sum(axis=1)
    assert np.array_equal(np.diff(rl.row_off), cnt)
    for n in np.nonzero(cnt)[0][:200]:
        e = rl.vars[rl.row_off[n]:rl.row_off[n + 1]].astype(np.int64)
        key = (e & 0x8000) * 4 + (e & 0x3FFF)
        assert np.all(np.diff(key) > 0)


@pytest.mark.parametrize("seed", range(4))
def test_acc_lists_random_graphs(seed):
    rng = np.random.default_rng(300 + seed)
    words = [4, 8, 128, 132][seed]
    row_ptr, col, kind, R, W, S = _mfp_ref.random_graph(rng, 600, words)
    g = {"row_ptr": row_ptr, "col": col, "kind": kind, "A": R | W, "B": W, "USE": R, "S": S}
    off, acc = planes_to_acc(R, W)
    shuffled = acc.copy()
    for i in range(0, len(off) - 1, 7):         # order inside a node is free
        rng.shuffle(shuffled[off[i]:off[i + 1]])
    prob = CsrProblem.from_acc(row_ptr, col, kind, off, shuffled, S, words)
    prob.solve()
    eh, ed, _ = _oracle.c3_solve(g)
    OH, OD, _ = prob.download(True, True)
    assert np.array_equal(OH, eh) and np.array_equal(OD, ed)
    _check_lists(prob.requirements_list(), g, eh, ed)
    # export round trip: planes -> lists on the device == numpy lists
    eoff, eacc = prob.export_acc()
    assert np.array_equal(eoff, off) and np.array_equal(eacc, acc)


def test_acc_all_in_one_matches_plane_path():
    g = _oracle.c3_generate(9, 1 << 14, 0, 128, 82)
    off, acc = planes_to_acc(g["USE"], g["B"])
    sess = AccSession()
    rl = sess.run(g["row_ptr"], g["col"], g["kind"], off, acc, g["S"], 128)
    eh, ed, _ = _oracle.c3_solve(g)
    _check_lists(rl, g, eh, ed)
    rl2 = sess.run(g["row_ptr"], g["col"], g["kind"], off, acc, g["S"], 128)   # cached buffers
    assert np.array_equal(rl2.vars, rl.vars) and np.array_equal(rl2.row_off, rl.row_off)
    assert sess.stats.solve_ms > 0


def test_acc_rejects_bad_entries():
    g = _oracle.c3_generate(3, 256, 0, 4, 8)
    off, acc = planes_to_acc(g["USE"], g["B"])
    bad = acc.copy()
    bad[0] = 200 | (1 << 14)                      # var 200 >= V = 128
    with pytest.raises(RuntimeError):
        CsrProblem.from_acc(g["row_ptr"], g["col"], g["kind"], off, bad, g["S"], 4)
    bad = acc.copy()
    bad[0] = bad[0] & 0x3FFF                      # kind 0
    with pytest.raises(RuntimeError):
        CsrProblem.from_acc(g["row_ptr"], g["col"], g["kind"], off, bad, g["S"], 4)


def test_async_solves_back_to_back_reach_the_fixpoint():
    """dfx_csr_solve_async: several solves enqueued without host sync (each
    restarts from top and decides convergence on the device) end at the
    same fixpoint as the synchronous call."""
    g = _oracle.c3_generate(4, 1 << 14, 0, 128, 82)
    prob = CsrProblem.from_arrays(g["row_ptr"], g["col"], g["kind"], g["USE"], g["B"], g["S"])
    for _ in range(4):
        prob.solve_async()
    OH, OD, _ = prob.download(True, True)
    eh, ed, _ = _oracle.c3_solve(g)
    assert np.array_equal(OH, eh) and np.array_equal(OD, ed)
    st = prob.solve()
    assert st.rounds_h >= 2


def test_long_backward_propagation_hundreds_of_rounds():
    """A reversed chain (pred of n is n+1) propagates one node per round
    against the sweep order: ~N rounds.  Exercises the unbounded round loop
    and the wrap of the per-edge seen bytes (> 255 rounds)."""
    n, words = 700, 4
    rng = np.random.default_rng(1)
    row_ptr = np.zeros(n + 1, dtype=np.int32)
    row_ptr[1:] = np.arange(1, n + 1, dtype=np.int32)
    row_ptr[n] = n - 1                       # the last node is the entry
    col = np.arange(1, n, dtype=np.int32)    # pred(n) = n + 1
    kind = np.zeros(n, dtype=np.uint8)
    kind[-50:] = 1                           # kernel nodes at the far end write
    W = np.zeros((n, words), dtype=np.uint32)
    W[-50:] = rng.integers(0, 2**32, size=(50, words), dtype=np.uint32)
    R = np.zeros_like(W)
    R[:: 7] = rng.integers(0, 2**32, size=R[:: 7].shape, dtype=np.uint32) & 0x01010101
    S = np.zeros(words, dtype=np.uint32)
    g = {"row_ptr": row_ptr, "col": col, "kind": kind, "A": R | W, "B": W, "USE": R, "S": S}
    prob = CsrProblem.from_arrays(row_ptr, col, kind, R, W, S)
    st = prob.solve()
    OH, OD, _ = prob.download(True, True)
    eh, ed, _ = _oracle.c3_solve(g)
    assert np.array_equal(OH, eh) and np.array_equal(OD, ed)
    assert max(st.rounds_h, st.rounds_d) > 256


def test_acc_lists_edge_cases():
    """List forms at the edges: no accesses at all, the widest variable
    space (V = 16384: 14-bit variable ids, four 4096-variable slices), and a
    too-small output capacity (DFX_E_NOSPC, then the exact size)."""
    rng = np.random.default_rng(5)
    # no accesses: every state stays at its boundary value, no requirements
    row_ptr, col, kind, R, W, S = _mfp_ref.random_graph(rng, 300, 4)
    R[:] = 0
    W[:] = 0
    off, acc = planes_to_acc(R, W)
    assert acc.shape[0] == 0
    prob = CsrProblem.from_acc(row_ptr, col, kind, off, acc, S, 4)
    prob.solve()
    rl = prob.requirements_list()
    assert rl.vars.shape[0] == 0 and not rl.row_off.any()
    # V = 16384
    row_ptr, col, kind, R, W, S = _mfp_ref.random_graph(rng, 200, 512)
    g = {"row_ptr": row_ptr, "col": col, "kind": kind, "A": R | W, "B": W, "USE": R, "S": S}
    off, acc = planes_to_acc(R, W)
    assert int((acc & 0x3FFF).max()) >= 16000
    prob = CsrProblem.from_acc(row_ptr, col, kind, off, acc, S, 512)
    prob.solve()
    eh, ed, _ = _oracle.c3_solve(g)
    OH, OD, _ = prob.download(True, True)
    assert np.array_equal(OH, eh) and np.array_equal(OD, ed)
    _check_lists(prob.requirements_list(capacity=1), g, eh, ed)   # NOSPC, then exact


# ---- malformed graphs: argument errors, never device faults

def _small_graph(seed=3, words=4, n=300):
    rng = np.random.default_rng(seed)
    return _mfp_ref.random_graph(rng, n, words)


@pytest.mark.parametrize("what", ["col_high", "col_neg", "rowptr_dec", "rowptr_start",
                                  "acc_col_high"])
def test_malformed_csr_is_an_argument_error_and_engine_survives(what):
    from paper_2406_13881_b200 import _abi
    row_ptr, col, kind, R, W, S = _small_graph()
    col = col.copy()
    row_ptr = row_ptr.copy()
    n = row_ptr.shape[0] - 1
    if what in ("col_high", "acc_col_high"):
        col[len(col) // 2] = n + 5
    elif what == "col_neg":
        col[3] = -1
    elif what == "rowptr_dec":
        row_ptr[n // 2] = row_ptr[n // 2 + 1] + 1
    elif what == "rowptr_start":
        row_ptr[0] = 1
    with pytest.raises(_abi.EngineError, match="CSR|row_ptr"):
        if what == "acc_col_high":
            off, acc = planes_to_acc(R, W)
            AccSession().run(row_ptr, col, kind, off, acc, S, R.shape[1])
        else:
            CsrProblem.from_arrays(row_ptr, col, kind, R, W, S)
    # the context is intact: a good problem on the same engine solves exactly
    row_ptr, col, kind, R, W, S = _small_graph(seed=4)
    g = {"row_ptr": row_ptr, "col": col, "kind": kind, "A": R | W, "B": W, "USE": R, "S": S}
    _check(CsrProblem.from_arrays(row_ptr, col, kind, R, W, S), g)
    rows, _ = mfp_csr(row_ptr, col, kind, R, W, S)
    assert rows.masks.shape[0] >= 0
