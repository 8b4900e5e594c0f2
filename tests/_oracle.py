"""Test-side loader for the CPU oracle library (oracle/liboracle.so).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg use this module.
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

ROOT = pathlib.Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "liboracle.so"

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_LIB.exists():
            subprocess.run(["make", "-C", str(ORACLE_DIR)], check=True,
                           stdout=subprocess.DEVNULL)
        _lib = C.CDLL(str(ORACLE_LIB))
        _lib.oracle_replay_batch.restype = C.c_int
    return _lib


def replay_runner(rin, rout) -> int:
    return lib().oracle_replay_batch(C.byref(rin), C.byref(rout))


def replay_runner_mt(rin, rout) -> int:
    """All host threads (OpenMP over functions); same output as replay_runner."""
    return lib().oracle_replay_batch_mt(C.byref(rin), C.byref(rout))


# ---- E2 / C3 (oracle/mfp_oracle.c) -------------------------------------------
import numpy as np  # noqa: E402


class CsrProb(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("words", C.c_int),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("kind", C.c_void_p),
                ("A", C.c_void_p), ("B", C.c_void_p), ("S", C.c_void_p)]


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def c3_scalar_mask(w0: int, words: int, n_scalar: int) -> np.ndarray:
    L = lib()
    L.oracle_c3_scalar_word.restype = C.c_uint32
    return np.array([L.oracle_c3_scalar_word(w0 + w, n_scalar) for w in range(words)],
                    dtype=np.uint32)


def c3_generate(seed: int, n_nodes: int, w0: int, words: int, n_scalar: int):
    """C3 inputs for the global word columns [w0, w0+words)."""
    L = lib()
    L.oracle_c3_csr.restype = C.c_int64
    nnz = L.oracle_c3_csr(C.c_uint64(seed), C.c_int64(n_nodes), None, None)
    row_ptr = np.zeros(n_nodes + 1, dtype=np.int32)
    col = np.zeros(max(1, nnz), dtype=np.int32)
    L.oracle_c3_csr(C.c_uint64(seed), C.c_int64(n_nodes), _p(row_ptr), _p(col))
    kind = np.zeros(n_nodes, dtype=np.uint8)
    A = np.zeros((n_nodes, words), dtype=np.uint32)
    B = np.zeros_like(A)
    USE = np.zeros_like(A)
    L.oracle_c3_planes(C.c_uint64(seed), C.c_int64(n_nodes), C.c_int(words), C.c_int(w0),
                       _p(kind), _p(A), _p(B), _p(USE))
    S = c3_scalar_mask(w0, words, n_scalar)
    return {"row_ptr": row_ptr, "col": col[:nnz], "kind": kind, "A": A, "B": B,
            "USE": USE, "S": S, "nnz": nnz}


def c3_solve(g):
    L = lib()
    n = g["kind"].shape[0]
    words = g["A"].shape[1]
    prob = CsrProb(n, words, *(g[k].ctypes.data for k in ("row_ptr", "col", "kind", "A", "B", "S")))
    OH = np.zeros((n, words), dtype=np.uint32)
    OD = np.zeros_like(OH)
    L.oracle_mfp_solve.restype = C.c_int
    sweeps = L.oracle_mfp_solve(C.byref(prob), _p(OH), _p(OD))
    return OH, OD, sweeps


def c3_requirements(g, OH, OD):
    L = lib()
    n = g["kind"].shape[0]
    words = g["A"].shape[1]
    prob = CsrProb(n, words, *(g[k].ctypes.data for k in ("row_ptr", "col", "kind", "A", "B", "S")))
    REQ = np.zeros((n, words), dtype=np.uint32)
    FP = np.zeros_like(REQ)
    L.oracle_mfp_requirements(C.byref(prob), _p(g["USE"]), _p(OH), _p(OD), _p(REQ), _p(FP))
    return REQ, FP


def num_threads() -> int:
    return lib().oracle_num_threads()


def summaries_runner(cin, cout) -> int:
    return lib().oracle_summaries(C.byref(cin), C.byref(cout))


def c3_verify(seed: int, n_nodes: int, w0: int, words: int, n_scalar: int, OH, OD,
              REQ=None, FP=None, block: int = 32) -> dict:
    """Exact check of full-size solve outputs (OUT_H/OUT_D planes, and the
    requirement / firstprivate planes when given) against the oracle, one
    block of `block` variable words at a time (variables are independent, so
    each block is an exact sub-problem; memory stays O(n_nodes x block)).
    Returns the number of differing words per output."""
    bad = {"OUT_H": 0, "OUT_D": 0}
    if REQ is not None:
        bad.update(REQ=0, FP=0)
    for b0 in range(0, words, block):
        nb = min(block, words - b0)
        g = c3_generate(seed, n_nodes, w0 + b0, nb, n_scalar)
        eh, ed, _ = c3_solve(g)
        bad["OUT_H"] += int(np.count_nonzero(OH[:, b0:b0 + nb] != eh))
        bad["OUT_D"] += int(np.count_nonzero(OD[:, b0:b0 + nb] != ed))
        if REQ is not None:
            rq, fp = c3_requirements(g, eh, ed)
            bad["REQ"] += int(np.count_nonzero(REQ[:, b0:b0 + nb] != rq))
            bad["FP"] += int(np.count_nonzero(FP[:, b0:b0 + nb] != fp))
    return bad
