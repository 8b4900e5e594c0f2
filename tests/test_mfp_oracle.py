"""CPU: pin the C oracle of kernels (a)/(b) against an independent numpy
formulation (Jacobi rounds vs the oracle's Gauss-Seidel sweeps) and check
the C3 generator's statistics against its specification."""
import numpy as np
import pytest

import _mfp_ref
import _oracle


def _prob(row_ptr, col, kind, R, W, S):
    return {"row_ptr": row_ptr, "col": col, "kind": kind, "A": R | W, "B": W, "USE": R, "S": S}


@pytest.mark.parametrize("seed", range(6))
def test_oracle_solver_matches_numpy_jacobi(seed):
    rng = np.random.default_rng(seed)
    row_ptr, col, kind, R, W, S = _mfp_ref.random_graph(rng, 300, 4)
    g = _prob(row_ptr, col, kind, R, W, S)
    OH, OD, sweeps = _oracle.c3_solve(g)
    rh, rd = _mfp_ref.solve(row_ptr, col, kind, g["A"], g["B"], S)
    assert np.array_equal(OH, rh) and np.array_equal(OD, rd)
    REQ, FP = _oracle.c3_requirements(g, OH, OD)
    rq, rf = _mfp_ref.requirements(row_ptr, col, kind, g["A"], g["B"], R, S, OH, OD)
    assert np.array_equal(REQ, rq) and np.array_equal(FP, rf)


def test_c3_generator_statistics():
    g = _oracle.c3_generate(7, 1 << 16, 0, 4, 82)
    n = g["kind"].shape[0]
    assert abs(g["nnz"] / n - 2.5) < 0.03                       # avg in-degree 2.5
    assert abs(g["kind"].mean() - 0.2) < 0.01                    # 20% kernel nodes
    acc = np.unpackbits((g["A"]).view(np.uint8)).mean()
    assert abs(acc - 1 / 32) < 0.002                             # access prob 1/32
    assert g["row_ptr"][1] == 0                                  # entry has no preds
    # every non-entry node's first predecessor is its fall-through n-1
    assert np.array_equal(g["col"][g["row_ptr"][1:-1]], np.arange(n - 1))
    assert (g["S"][:2] == 0xFFFFFFFF).all() and g["S"][2] == (1 << 18) - 1 and g["S"][3] == 0


def test_c3_column_block_is_exact_sample():
    """Variables are independent: solving a column block equals the same
    columns of a wider solve."""
    wide = _oracle.c3_generate(3, 4096, 0, 8, 82)
    narrow = _oracle.c3_generate(3, 4096, 4, 4, 82)
    OHw, ODw, _ = _oracle.c3_solve(wide)
    OHn, ODn, _ = _oracle.c3_solve(narrow)
    assert np.array_equal(OHw[:, 4:], OHn) and np.array_equal(ODw[:, 4:], ODn)
