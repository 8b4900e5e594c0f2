"""Configuration C2: LULESH-2.0-shaped synthetic programs (C source).

Patterned on the corpus's `lulesh_mini.c` (a scaled-down LULESH proxy): a
time-step loop around ~40 offloaded kernels over ~200 global mesh arrays,
grouped into phases, some phases inside nested host loops (sub-cycling),
host-side reductions through functions that read globals (like
`courant_dt`), scalar time-step control, and host checks of a few fields.
Avoids constructs the reference front end rejects.
"""
from __future__ import annotations

import random


def generate_lulesh(seed: int = 0, n_arrays: int = 200, n_kernels: int = 40,
                    n_reducers: int = 4, steps: int = 12) -> str:
    r = random.Random(seed)
    L: list[str] = []
    L.append("/* LULESH-shaped synthetic program, seed %d */" % seed)
    L.append("#define NODES 1024")
    L.append("#define ELEMS 960")
    L.append("#define STEPS %d" % steps)
    arrays = ["f%d" % i for i in range(n_arrays)]
    size = {a: ("NODES" if r.random() < 0.5 else "ELEMS") for a in arrays}
    for a in arrays:
        L.append("double %s[%s];" % (a, size[a]))
    L.append("double sqrt(double v);")
    L.append("void init_mesh(void);")
    reducers = []
    for k in range(n_reducers):
        name = "reduce_%d" % k
        reducers.append(name)
        src = r.sample(arrays, 2)
        L.append("")
        L.append("double %s(double prev) {" % name)
        L.append("    double acc = prev;")
        L.append("    for (int i = 0; i < ELEMS; ++i) {")
        L.append("        acc = acc + %s[i] * %s[i];" % (src[0], src[1]))
        L.append("    }")
        L.append("    return acc;")
        L.append("}")
    L.append("")
    L.append("int main(void) {")
    L.append("    double dt = 1.0e-3;")
    L.append("    double total = 0.0;")
    L.append("    init_mesh();")
    L.append("    for (int step = 0; step < STEPS; ++step) {")
    ind = "        "
    kernels_left = n_kernels
    phase = 0
    while kernels_left > 0:
        n = min(kernels_left, r.randrange(2, 6))
        kernels_left -= n
        nested = r.random() < 0.3
        body_ind = ind
        if nested:
            L.append(ind + "for (int sub%d = 0; sub%d < 2; ++sub%d) {" % (phase, phase, phase))
            body_ind = ind + "    "
        for _ in range(n):
            outs = r.sample(arrays, r.randrange(1, 3))
            ins = r.sample(arrays, r.randrange(2, 5))
            lim = "NODES" if all(size[a] == "NODES" for a in outs + ins) else "ELEMS"
            L.append(body_ind + "#pragma omp target teams distribute parallel for")
            L.append(body_ind + "for (int k = 0; k < %s; ++k) {" % lim)
            expr = " + ".join("%s[k]" % a for a in ins)
            for o in outs:
                op = r.choice(["=", "+="])
                L.append(body_ind + "    %s[k] %s (%s) * dt;" % (o, op, expr))
            L.append(body_ind + "}")
        if nested:
            L.append(ind + "}")
        x = r.random()
        if x < 0.25:
            L.append(ind + "dt = %s(dt);" % r.choice(reducers))
        elif x < 0.45:
            a = r.choice(arrays)
            L.append(ind + "total = total + %s[%d];" % (a, r.randrange(8)))
        elif x < 0.55:
            a = r.choice(arrays)
            L.append(ind + "if (%s[0] > 1.0e6) {" % a)
            L.append(ind + "    dt = dt * 0.5;")
            L.append(ind + "}")
        phase += 1
    L.append(ind + "dt = %s(dt);" % r.choice(reducers))
    L.append("    }")
    chk = r.sample(arrays, 3)
    L.append("    total = total + %s[0] + %s[1] + %s[2];" % tuple(chk))
    L.append("    return (int) total;")
    L.append("}")
    return "\n".join(L) + "\n"
