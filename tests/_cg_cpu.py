"""CPU restatement of one kernel-(c) wave (TEST INFRASTRUCTURE): used to run
the multi-rank exchange protocol of distributed.ShardedSummaries on gloo."""
from __future__ import annotations

import numpy as np


def _force_dev(b):
    return ((b & 3) | 8) if (b & 3) else 0


def make_cpu_wave(state):
    """wave_impl(prev, cur, w) for a ShardedSummaries on CPU tensors."""
    g = state.g
    P = g.n_params

    def wave(prev, cur, w):
        tp, tc = state.t[prev], state.t[cur]
        pb, pl, pn = tp["bits"].numpy(), tp["list"].numpy(), tp["len"].numpy()
        cb, cl, cn = tc["bits"].numpy(), tc["list"].numpy(), tc["len"].numpy()
        lo, hi = int(g.wave_off[w]), int(g.wave_off[w + 1])
        changed = 0
        for pos in range(lo + state.rank, hi, state.world):
            f = int(g.wave_fns[pos])
            nb = g.direct[f].copy()
            order, seen = [], set()

            def app(s):
                if s not in seen:
                    seen.add(s)
                    order.append(s)
            for k in range(g.src_off[f], g.src_off[f + 1]):
                kind, a, b, c = (int(x) for x in g.src[k])
                if (kind & 0xFF) == 0:
                    for j in range(b):
                        app(int(g.slist[a + j]))
                    continue
                dev = (kind >> 8) & 1
                callee = a
                B, L, N = (cb, cl, cn) if callee < f else (pb, pl, pn)
                glist = [int(x) for x in L[callee, :N[callee]]]
                for x in glist:
                    if x >= P:
                        continue
                    for t in range(b, b + c):
                        if int(g.bind[t, 0]) == x:
                            s = int(g.bind[t, 1])
                            nb[s] |= _force_dev(int(B[callee, x])) if dev else int(B[callee, x])
                            app(s)
                for x in glist:
                    if x < P:
                        continue
                    nb[x] |= _force_dev(int(B[callee, x])) if dev else int(B[callee, x])
                    app(x)
            ns = g.init_bits.shape[1]
            if not np.array_equal(nb, pb[f, :ns]):
                changed = 1
            cb[f, :ns] = nb
            cl[f, :len(order)] = order
            cn[f] = len(order)
        return changed
    return wave
