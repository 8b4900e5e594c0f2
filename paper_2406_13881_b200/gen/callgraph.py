"""Configuration C5: interprocedural call-graph programs (emitted as C).

`n_funcs` functions arranged in chains of `depth` calls (SCC chains when
back edges are present), each with `n_ptr_params` pointer parameters,
touching a random subset of `n_globals` global arrays on the host or in
offloaded kernels; a fraction of call sites go back up the chain (cycles), a
few call undeclared externals and declared-but-undefined prototypes (the
reference's pessimistic summaries, interproc.py:50-58), and some calls are
made from inside kernels (device-forced effects, interproc.py:113-114).
"""
from __future__ import annotations

import random
from dataclasses import dataclass


@dataclass
class CallGraphConfig:
    n_funcs: int = 10_000
    depth: int = 12
    n_globals: int = 256
    n_ptr_params: int = 2
    p_back: float = 0.10         # call sites that go back up the chain (SCCs)
    p_kernel: float = 0.30       # functions with an offloaded kernel
    p_extern: float = 0.03       # calls to an undeclared external
    p_proto: float = 0.03        # calls to a declared, undefined function
    globals_per_fn: int = 3
    size: int = 64


def generate(seed: int, cfg: CallGraphConfig | None = None) -> str:
    cfg = cfg or CallGraphConfig()
    r = random.Random(seed)
    L: list[str] = []
    L.append("#define N %d" % cfg.size)
    for g in range(cfg.n_globals):
        L.append("double g%d[%d];" % (g, cfg.size))
    L.append("void proto_rw(double *a, const double *b);")
    n_chains = max(1, cfg.n_funcs // cfg.depth)
    names = [["f%d_%d" % (c, d) for d in range(cfg.depth)] for c in range(n_chains)]
    P = cfg.n_ptr_params
    params = ", ".join("double *p%d" % i for i in range(P))
    # prototypes first so back edges and out-of-order calls resolve
    for c in range(n_chains):
        for d in range(cfg.depth):
            L.append("void %s(%s);" % (names[c][d], params))
    L.append("")

    def arg(c, d):
        x = r.random()
        if x < 0.5:
            return "p%d" % r.randrange(P)
        return "g%d" % r.randrange(cfg.n_globals)

    for c in range(n_chains):
        for d in range(cfg.depth):
            L.append("void %s(%s) {" % (names[c][d], params))
            gl = ["g%d" % r.randrange(cfg.n_globals) for _ in range(cfg.globals_per_fn)]
            # host effects on params and globals
            for _ in range(r.randrange(1, 4)):
                tgt = r.choice(["p%d" % r.randrange(P)] + gl)
                src = r.choice(["p%d" % r.randrange(P)] + gl)
                op = r.choice(["=", "+="])
                L.append("    %s[%d] %s %s[%d];" % (tgt, r.randrange(4), op, src, r.randrange(4)))
            if r.random() < cfg.p_kernel:
                tgt = r.choice(["p%d" % r.randrange(P)] + gl)
                src = r.choice(["p%d" % r.randrange(P)] + gl)
                L.append("    #pragma omp target teams distribute parallel for")
                L.append("    for (int k = 0; k < N; ++k) {")
                L.append("        %s[k] = %s[k] + 1.0;" % (tgt, src))
                if d + 1 < cfg.depth and r.random() < 0.2:
                    L.append("        %s(%s);" % (names[c][d + 1],
                                                   ", ".join(arg(c, d) for _ in range(P))))
                L.append("    }")
            if d + 1 < cfg.depth:
                L.append("    %s(%s);" % (names[c][d + 1], ", ".join(arg(c, d) for _ in range(P))))
            if d > 0 and r.random() < cfg.p_back:
                L.append("    %s(%s);" % (names[c][r.randrange(d)],
                                         ", ".join(arg(c, d) for _ in range(P))))
            if r.random() < cfg.p_extern:
                L.append("    ext_touch(%s);" % arg(c, d))
            if r.random() < cfg.p_proto:
                L.append("    proto_rw(%s, %s);" % (arg(c, d), arg(c, d)))
            L.append("}")
    L.append("")
    L.append("int main(void) {")
    for c in range(n_chains):
        L.append("    %s(%s);" % (names[c][0], ", ".join("g%d" % r.randrange(cfg.n_globals)
                                                     for _ in range(P))))
    L.append("    return 0;")
    L.append("}")
    return "\n".join(L) + "\n"
