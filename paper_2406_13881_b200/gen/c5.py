"""Configuration C5 generator, emitted directly in lowered form.

`gen/callgraph.py` writes the same shape as C source (used for parity with
the reference front end at a few hundred functions); this module builds the
lowered `CallGraph` (the `dfx_summaries` inputs) directly, so 10k-function
graphs cost no parsing: chains of `depth` calls in dict order (callee after
caller), `p_back` back edges to earlier functions of the chain (SCCs, and
same-pass Gauss-Seidel dependencies), `n_params` pointer parameters bound to
caller parameters or globals, calls from inside kernels (device-forced), and
constant external/prototype call sites.
"""
from __future__ import annotations

import random

import numpy as np

from ..interproc import BIT_D, BIT_H, BIT_R, BIT_W, SRC_CALL, SRC_STATIC, CallGraph


def generate_c5(seed: int = 0, n_funcs: int = 10_000, depth: int = 12, n_globals: int = 256,
                n_params: int = 2, p_back: float = 0.10, p_dev: float = 0.06,
                p_const: float = 0.06, globals_per_fn: int = 3) -> CallGraph:
    r = random.Random(seed)
    P = n_params
    ns = P + n_globals
    n_chains = max(1, n_funcs // depth)
    nf = n_chains * depth
    init_bits = np.zeros((nf, ns), dtype=np.uint8)
    init_list = np.zeros((nf, ns), dtype=np.int16)
    init_len = np.zeros(nf, dtype=np.int32)
    direct = np.zeros((nf, ns), dtype=np.uint8)
    src_off = np.zeros(nf + 1, dtype=np.int32)
    src_rows, slist, bind = [], [], []
    wave = [0] * nf

    def eff():
        k = r.choice([BIT_R, BIT_W, BIT_R | BIT_W])
        return k | (BIT_D if r.random() < 0.3 else BIT_H)

    def static_src(f, items, first):
        order = []
        for sl, b in items:
            direct[f, sl] |= b
            if first:
                init_bits[f, sl] |= b
            if sl not in order:
                order.append(sl)
        if first:
            init_len[f] = len(order)
            init_list[f, :len(order)] = order
        src_rows.append((SRC_STATIC, len(slist), len(order), 0))
        slist.extend(order)

    def call_src(f, g):
        dev = r.random() < p_dev
        binds = []
        for i in range(P):
            x = r.random()
            if x < 0.45:
                binds.append((i, r.randrange(P)))
            elif x < 0.9:
                binds.append((i, P + r.randrange(n_globals)))
        src_rows.append((SRC_CALL | ((1 if dev else 0) << 8), g, len(bind), len(binds)))
        bind.extend(binds)
        if g < f:
            wave[f] = max(wave[f], wave[g] + 1)

    for c in range(n_chains):
        for d in range(depth):
            f = c * depth + d
            gl = [P + r.randrange(n_globals) for _ in range(globals_per_fn)]
            items = [(r.choice(list(range(P)) + gl), eff()) for _ in range(r.randrange(1, 4))]
            static_src(f, items, True)
            if d + 1 < depth:
                call_src(f, f + 1)
            if d > 0 and r.random() < p_back:
                call_src(f, c * depth + r.randrange(d))
            if r.random() < p_const:
                static_src(f, [(r.choice(list(range(P)) + gl), BIT_R | BIT_W | BIT_H)], False)
            src_off[f + 1] = len(src_rows)
    n_waves = max(wave) + 1
    buckets = [[] for _ in range(n_waves)]
    for f in range(nf):
        buckets[wave[f]].append(f)
    wave_off = np.zeros(n_waves + 1, dtype=np.int32)
    for i, bk in enumerate(buckets):
        wave_off[i + 1] = wave_off[i] + len(bk)
    return CallGraph(
        names=["f%d" % f for f in range(nf)], fns=[None] * nf, n_params=P,
        globals=["g%d" % i for i in range(n_globals)], init_bits=init_bits, init_len=init_len,
        init_list=init_list, direct=direct, src_off=src_off,
        src=np.array(src_rows, dtype=np.int32).reshape(-1, 4),
        slist=np.array(slist, dtype=np.int16), bind=np.array(bind, dtype=np.int32).reshape(-1, 2),
        wave_off=wave_off, wave_fns=np.array([f for bk in buckets for f in bk], dtype=np.int32))
