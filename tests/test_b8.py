"""Byte-coded access / requirement lists (include/dfx.h "B8", dfx_mfp_acc8):
the host encoder and decoder round-trip exactly (long gaps, every kind, empty
nodes, the firstprivate restart), and on the GPU the byte-coded call returns
exactly the uint16 list call's answer (which tests/test_lists.py pins to the
oracle), on random graphs and a C3 slab; malformed streams are refused."""
import numpy as np
import pytest

from paper_2406_13881_b200.csr import (B8_FP, B8_REQ, _b8_encode, acc_to_b8, b8_decode,
                                       planes_to_acc, req8_to_lists)


def _planes(rng, n, words, p_r, p_w):
    pk = lambda B: np.packbits(B.astype(np.uint8), axis=1, bitorder="little").view(  # noqa: E731
        np.uint32).reshape(n, words)
    return (pk(rng.random((n, words * 32)) < p_r), pk(rng.random((n, words * 32)) < p_w))


@pytest.mark.parametrize("density", [0.001, 1 / 32, 0.3])
def test_access_lists_round_trip(density):
    rng = np.random.default_rng(int(density * 1000))
    R, W = _planes(rng, 700, 16, density, density / 2)
    off, acc = planes_to_acc(R, W)
    boff, b = acc_to_b8(off, acc)
    assert boff.dtype == np.int32 and b.dtype == np.uint8 and boff[-1] == b.shape[0]
    node, var, kind = b8_decode(boff, b)
    a = acc.astype(np.int64)
    assert np.array_equal(node, np.repeat(np.arange(700), np.diff(off)))
    assert np.array_equal(var, a & 0x3FFF) and np.array_equal(kind, a >> 14)
    if density == 1 / 32:       # C3's access density: about 1.15 bytes per entry
        assert b.shape[0] < 1.25 * acc.shape[0]


def test_gaps_and_kinds():
    node = np.array([0, 0, 0, 2, 2, 2, 2])
    var = np.array([0, 62, 63 + 62 + 126, 3, 7, 4000, 16383])
    kind = np.array([1, 2, 3, 1, 2, 2, 3])
    o, b = _b8_encode(node, var, kind, 3)
    assert o[0] == 0 and o[1] == o[2] and o[3] == b.shape[0]
    n2, v2, k2 = b8_decode(o, b)
    assert list(n2) == list(node) and list(v2) == list(var) and list(k2) == list(kind)
    # every byte of an entry carries its kind; only the last has d < 63
    assert ((b & 63) < 63).sum() == var.shape[0]


def test_requirement_lists_to_uint16_form():
    node = np.array([0, 0, 0, 1])
    var = np.array([5, 900, 2, 77])
    kind = np.array([B8_REQ, B8_REQ, B8_FP, B8_FP])
    restart = np.array([False, False, True, False])
    o, b = _b8_encode(node, var, kind, 2, restart)
    rl = req8_to_lists(o, b, 32)
    assert list(rl.row_off) == [0, 3, 4]
    assert list(rl.vars) == [5, 900, 2 | 0x8000, 77 | 0x8000]


def test_encoder_refuses_unsorted():
    with pytest.raises(ValueError):
        _b8_encode(np.array([0, 0]), np.array([9, 3]), np.array([1, 1]), 1)


def _random_graph(rng, n, words):
    deg = rng.integers(0, 4, n)
    deg[0] = 0
    row_ptr = np.zeros(n + 1, dtype=np.int32)
    row_ptr[1:] = np.cumsum(deg)
    col = rng.integers(0, n, int(row_ptr[-1])).astype(np.int32)
    kind = (rng.random(n) < 0.25).astype(np.uint8)
    S = np.zeros(words, dtype=np.uint32)
    S[0] = 0xFFFF
    return row_ptr, col, kind, S


@pytest.mark.gpu
@pytest.mark.parametrize("n,words,dens", [(5000, 4, 0.05), (20000, 16, 1 / 32), (3000, 128, 0.01),
                                          (1500, 512, 0.004)])
def test_cuda_b8_equals_uint16_lists(n, words, dens):
    from paper_2406_13881_b200.csr import Acc8Session, AccSession
    rng = np.random.default_rng(n + words)
    row_ptr, col, kind, S = _random_graph(rng, n, words)
    R, W = _planes(rng, n, words, dens, dens / 2)
    off, acc = planes_to_acc(R, W)
    ref = AccSession().run(row_ptr, col, kind, off, acc, S, words)
    boff, b = acc_to_b8(off, acc)
    got = Acc8Session().run(row_ptr, col, kind, boff, b, S, words)
    lists = got.to_lists()
    assert np.array_equal(lists.row_off, ref.row_off)
    assert np.array_equal(lists.vars, ref.vars)


@pytest.mark.gpu
def test_cuda_b8_c3_slab():
    """A 64k-node slice of configuration C3 (128 words): byte-coded call ==
    uint16 list call, entry for entry."""
    from paper_2406_13881_b200.csr import (Acc8Session, AccSession, C3Config, CsrProblem,
                                           c3_scalar_mask)
    cfg = C3Config(n_nodes=1 << 16, seed=3)
    prob = CsrProblem.generate_c3(cfg)
    rp, col, kind, R, W = prob.export_inputs()
    off, acc = prob.export_acc()
    S = c3_scalar_mask(cfg)
    ref = AccSession().run(rp, col, kind, off, acc, S, 128)
    boff, b = acc_to_b8(off, acc)
    got = Acc8Session().run(rp, col, kind, boff, b, S, 128).to_lists()
    assert np.array_equal(got.row_off, ref.row_off) and np.array_equal(got.vars, ref.vars)
    assert b.shape[0] < 0.65 * 2 * acc.shape[0]


@pytest.mark.gpu
def test_cuda_b8_refuses_malformed_stream():
    from paper_2406_13881_b200 import _abi
    from paper_2406_13881_b200.csr import Acc8Session
    rng = np.random.default_rng(1)
    row_ptr, col, kind, S = _random_graph(rng, 100, 4)
    boff = np.zeros(101, dtype=np.int32)
    boff[1:] = 1
    b = np.array([(1 << 6) | 63], dtype=np.uint8)       # node 0: an unterminated entry
    with pytest.raises(_abi.EngineError):
        Acc8Session().run(row_ptr, col, kind, boff, b, S, 4)
    b = np.array([(1 << 6) | 62, ], dtype=np.uint8)     # fine: variable 62 < 128
    Acc8Session().run(row_ptr, col, kind, boff, b, S, 4)
    b = np.array([0], dtype=np.uint8)                   # kind 0
    with pytest.raises(_abi.EngineError):
        Acc8Session().run(row_ptr, col, kind, boff, b, S, 4)


@pytest.mark.gpu
def test_cuda_b8_empty_lists_and_single_node():
    """Nodes without accesses, a graph of one node, and a list whose every
    node is empty: the byte-coded call agrees with the uint16 call."""
    from paper_2406_13881_b200.csr import Acc8Session, AccSession
    rng = np.random.default_rng(3)
    for n in (1, 7, 4096):
        row_ptr, col, kind, S = _random_graph(rng, n, 4)
        for dens in (0.0, 0.02):
            R, W = _planes(rng, n, 4, dens, dens)
            off, acc = planes_to_acc(R, W)
            ref = AccSession().run(row_ptr, col, kind, off, acc, S, 4)
            boff, b = acc_to_b8(off, acc)
            got = Acc8Session().run(row_ptr, col, kind, boff, b, S, 4).to_lists()
            assert np.array_equal(got.row_off, ref.row_off) and np.array_equal(got.vars, ref.vars)
