"""Independent numpy formulation of the CSR fixpoint (Jacobi rounds), used to
pin the C oracle (oracle/mfp_oracle.c, Gauss-Seidel) on small graphs."""
from __future__ import annotations

import numpy as np

ALL = np.uint32(0xFFFFFFFF)


def meet(OUT, row_ptr, col, boundary):
    n = row_ptr.shape[0] - 1
    IN = np.empty_like(OUT)
    for i in range(n):
        a, b = row_ptr[i], row_ptr[i + 1]
        if a == b:
            IN[i] = boundary
        else:
            IN[i] = np.bitwise_and.reduce(OUT[col[a:b]], axis=0)
    return IN


def solve(row_ptr, col, kind, A, B, S):
    kind = kind.astype(bool)[:, None]
    OH = np.full_like(A, ALL)
    while True:
        IN = meet(OH, row_ptr, col, ALL)
        new = np.where(kind, IN & ~B, IN | A)
        if np.array_equal(new, OH):
            break
        OH = new
    HIN = meet(OH, row_ptr, col, ALL)
    F = A & ~B & S[None, :]
    OD = np.full_like(A, ALL)
    while True:
        IN = meet(OD, row_ptr, col, np.uint32(0))
        new = np.where(kind, IN | (A & ~(F & HIN)), IN & ~B)
        if np.array_equal(new, OD):
            break
        OD = new
    return OH, OD


def requirements(row_ptr, col, kind, A, B, USE, S, OH, OD):
    k = kind.astype(bool)[:, None]
    IH = meet(OH, row_ptr, col, ALL)
    ID = meet(OD, row_ptr, col, np.uint32(0))
    F = np.where(k, A & ~B & S[None, :], np.uint32(0))
    REQ = np.where(k, (USE & ~F & ~ID) | (F & ~ID & ~IH), USE & ~IH)
    FP = np.where(k, F & ~ID & IH, np.uint32(0))
    return REQ, FP


def random_graph(rng, n, words, max_deg=4, p_entry=0.05, density=0.08):
    degs = rng.integers(0, max_deg + 1, size=n)
    degs[rng.random(n) < p_entry] = 0
    row_ptr = np.zeros(n + 1, dtype=np.int32)
    row_ptr[1:] = np.cumsum(degs)
    col = rng.integers(0, n, size=int(row_ptr[-1])).astype(np.int32)
    kind = (rng.random(n) < 0.3).astype(np.uint8)
    bits = lambda p: (rng.random((n, words, 32)) < p)  # noqa: E731
    pack = lambda b: np.packbits(b, axis=2, bitorder="little").view(np.uint32).reshape(n, words)  # noqa: E731
    R = pack(bits(density))
    W = pack(bits(density))
    S = np.packbits(rng.random((words, 32)) < 0.1, axis=1,
                    bitorder="little").view(np.uint32).reshape(words)
    return row_ptr, col, kind, R, W, S
