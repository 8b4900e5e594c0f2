"""Configuration C4 as C source: the batch's functions emitted in the
reference's C subset, so the reference front end and its `analyze_function`
(`dartomp/dataflow.py:737-740`) can see them (SURVEY §8 d, C4: "both C source
(for oracle sampling) and direct lowering").

Function i of seed s is one translation unit: G global arrays and scalars,
one function `c4_<i>(double *p0, double *p1)` with local arrays and scalars,
and a structured body (`cprog.ProgramGen`: if/else, switch, for/while/do
nested <= 3 deep, kernels with firstprivate-eligible scalars) grown until the
function has N_f ~ U[n_min, n_max] host CFG nodes (`astcfg.py:201-253`
node kinds, counted as the generator emits them).  V_f is drawn from
`var_choices` and split over global arrays, global scalars, local arrays,
local scalars and the two pointer parameters.  Shapes come from a counter
hash of (seed, i), so any subset of the batch is generated independently.

The generated functions avoid every construct the reference rejects (no
braceless bodies, no late declarations, no jumps, no calls), like the
bytecode generator `csrc/c4gen.cpp`, whose shape parameters these are.
"""
from __future__ import annotations

from dataclasses import dataclass

from .cprog import GenConfig, ProgramGen, _Fn


@dataclass(frozen=True)
class C4SourceConfig:
    n_min: int = 64
    n_max: int = 2048
    var_choices: tuple = (32, 64, 128, 256, 512)
    seed: int = 0
    size: int = 64


def _mix(x: int) -> int:
    x &= (1 << 64) - 1
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & ((1 << 64) - 1)
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & ((1 << 64) - 1)
    return x ^ (x >> 31)


def c4_source_shape(cfg: C4SourceConfig, i: int) -> tuple[int, int]:
    """(N_f target host CFG nodes, V_f declared variables) of function i."""
    h = _mix(cfg.seed * 0x9E3779B97F4A7C15 + i * 0xD1B54A32D192ED03 + 1)
    n = cfg.n_min + h % (cfg.n_max - cfg.n_min + 1)
    v = cfg.var_choices[(h >> 32) % len(cfg.var_choices)]
    return int(n), int(v)


class _C4Gen(ProgramGen):
    """ProgramGen that counts host CFG nodes as it emits statements."""

    def __init__(self, seed, cfg, target):
        super().__init__(seed, cfg)
        self.nodes = 2                  # ENTRY, EXIT
        self.target = target
        self._seen = 0                  # lines already scanned for control heads

    def kernel(self, ctx):
        self.nodes += 1                 # one STMT node per target directive
        super().kernel(ctx)

    def simple(self, ctx, ivars):
        r = self.r
        if r.random() < self.cfg.p_kernel:
            self.kernel(ctx)
            return
        self.nodes += 1
        self.e.line(self.assign(ctx["arrays"], ctx["scalars"], ivars,
                                ctx["arrays"], ctx["scalars"]))

    def block(self, ctx, budget, depth, loop_depth, ivars):
        for _ in range(budget):
            if self.nodes >= self.target:
                return
            self.stmt(ctx, depth, loop_depth, ivars)

    def stmt(self, ctx, depth, loop_depth, ivars):
        super().stmt(ctx, depth, loop_depth, ivars)
        # control statements: count their extra nodes from the emitted heads
        # (nested statements were scanned by their own call)
        new = self.e.lines[self._seen:]
        self._seen = len(self.e.lines)
        for ln in new:
            s = ln.strip()
            if s.startswith("if ("):
                self.nodes += 1                         # PRED
            elif s.startswith("for (int i"):
                self.nodes += 3                         # init DECL, PRED, LOOP_BACK
            elif s.startswith("while ("):
                self.nodes += 2                         # PRED, LOOP_BACK
            elif s.startswith("} while ("):
                self.nodes += 2
            elif s.startswith("case ") or s == "default:":
                self.nodes += 1
            elif s.startswith("switch ("):
                self.nodes += 1
            elif s.startswith("break;"):
                self.nodes += 1
            elif s.endswith(" + 1;") and "=" in s and "[" not in s.split("=")[0]:
                self.nodes += 1                         # loop counter increments

    def c4_function(self, name: str, n_vars: int) -> str:
        cfg = self.cfg
        r = self.r
        e = self.e
        # V_f = 2 params + global arrays + global scalars + local arrays + local scalars + 1 counter
        n_free = max(4, n_vars - 3)
        n_ga = max(1, int(n_free * 0.55))
        n_gs = max(1, int(n_free * 0.15))
        n_la = max(1, int(n_free * 0.15))
        n_ls = max(1, n_free - n_ga - n_gs - n_la)
        e.line("#define N %d" % cfg.size)
        ga = ["g%d" % k for k in range(n_ga)]
        gs = ["gs%d" % k for k in range(n_gs)]
        for g in ga:
            e.line("double %s[%d];" % (g, cfg.size + 2))
        for s in gs:
            e.line("double %s;" % s)
        e.line("")
        e.line("void %s(double *p0, double *p1) {" % name)
        e.ind += 1
        la = ["la%d" % k for k in range(n_la)]
        ls = ["ls%d" % k for k in range(n_ls)]
        for a in la:
            e.line("double %s[%d];" % (a, cfg.size + 2))
            self.nodes += 1
        for s in ls:
            e.line("double %s = %d.0;" % (s, r.randrange(0, 5)))
            self.nodes += 1
        e.line("int it0 = 0;")
        self.nodes += 1
        self._seen = len(e.lines)
        ctx = {"arrays": ga + la + ["p0", "p1"], "scalars": gs + ls, "iscalars": ["it0"],
               "callees": [], "callees_dev": [], "kernels": 0}
        while self.nodes < self.target:
            self.stmt(ctx, 0, 0, [])
        e.ind -= 1
        e.line("}")
        return "\n".join(e.lines) + "\n"


def c4_source(cfg: C4SourceConfig, i: int) -> str:
    """C translation unit holding function `c4_<i>` of the batch."""
    n, v = c4_source_shape(cfg, i)
    gcfg = GenConfig(n_funcs=0, size=cfg.size, max_depth=4, max_loop_depth=3,
                     p_kernel=0.3, p_if=0.15, p_switch=0.04, p_loop=0.18, p_call=0.0,
                     p_jump=0.0, p_braceless=0.0, p_late_decl=0.0)
    g = _C4Gen(_mix(cfg.seed * 0x632BE59BD9B4E019 + i + 7), gcfg, n)
    return g.c4_function("c4_%d" % i, v)


def c4_function_name(i: int) -> str:
    return "c4_%d" % i


__all__ = ["C4SourceConfig", "c4_source", "c4_source_shape", "c4_function_name", "_Fn"]
