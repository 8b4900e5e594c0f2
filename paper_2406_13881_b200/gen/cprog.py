"""Seeded generator of structured C programs in the reference's C subset.

Used for (1) parity fixtures (random programs stressing every schedule quirk
of the reference analysis: nested if/switch (D1, D4), loops of every kind with
hoisting (D3, D7), firstprivate scalars (D2), jumps (D5), calls with global
effects (interproc)), (2) configuration C2 (LULESH-2.0-shaped program) and
(3) the C4 function batches.  Programs avoid constructs the reference
rejects at parse/classify time (pointer rebinding, `&` in kernels, `?:`,
`goto`); analysis-time errors (braces required, late declarations) are
generated on purpose with small probability, because error parity is part
of the contract.
"""
from __future__ import annotations

import random
from dataclasses import dataclass, field


@dataclass
class GenConfig:
    n_globals: int = 6            # global double arrays
    n_gscalars: int = 2           # global double scalars
    n_funcs: int = 1              # functions besides main
    n_locals: int = 3             # local arrays per function
    n_lscalars: int = 3           # local scalars per function
    n_stmts: int = 30             # top-level-ish statement budget per function
    max_depth: int = 3            # control nesting
    max_loop_depth: int = 3
    p_kernel: float = 0.25
    p_if: float = 0.15
    p_switch: float = 0.04
    p_loop: float = 0.18
    p_call: float = 0.05
    p_jump: float = 0.04
    p_braceless: float = 0.0      # braceless loop/if bodies (may trigger braces errors)
    p_late_decl: float = 0.0      # declare a local after the first kernel
    p_fp_clause: float = 0.15     # kernels with an explicit firstprivate(...) clause
    size: int = 64
    n_ptr_params: int = 2


@dataclass
class _Fn:
    name: str
    params: list = field(default_factory=list)      # (name, is_ptr)


class _Emitter:
    def __init__(self):
        self.lines: list[str] = []
        self.ind = 0

    def line(self, s: str) -> None:
        self.lines.append("    " * self.ind + s)


class ProgramGen:
    def __init__(self, seed: int, cfg: GenConfig | None = None):
        self.r = random.Random(seed)
        self.cfg = cfg or GenConfig()
        self.e = _Emitter()
        self.uid = 0

    def fresh(self, base: str) -> str:
        self.uid += 1
        return "%s%d" % (base, self.uid)

    # ---- expressions -----------------------------------------------------
    def idx(self, ivars: list[str]) -> str:
        r = self.r
        if ivars and r.random() < 0.8:
            v = r.choice(ivars)
            if r.random() < 0.2:
                return "%s + 1" % v
            return v
        return str(r.randrange(0, 4))

    def rvalue(self, arrays, scalars, ivars, depth=0) -> str:
        r = self.r
        x = r.random()
        if x < 0.45 and arrays:
            return "%s[%s]" % (r.choice(arrays), self.idx(ivars))
        if x < 0.7 and scalars:
            return r.choice(scalars)
        if x < 0.8 and depth < 2:
            return "(%s %s %s)" % (self.rvalue(arrays, scalars, ivars, depth + 1),
                                   r.choice("+-*"),
                                   self.rvalue(arrays, scalars, ivars, depth + 1))
        return "%d.0" % r.randrange(0, 9)

    def assign(self, arrays, scalars, ivars, targets_arrays, targets_scalars) -> str:
        r = self.r
        op = r.choice(["=", "=", "+="])
        if targets_arrays and (not targets_scalars or r.random() < 0.75):
            lhs = "%s[%s]" % (r.choice(targets_arrays), self.idx(ivars))
        else:
            lhs = r.choice(targets_scalars)
        return "%s %s %s;" % (lhs, op, self.rvalue(arrays, scalars, ivars))

    # ---- statements --------------------------------------------------------
    def kernel(self, ctx) -> None:
        r = self.r
        arrays, scalars = ctx["arrays"], ctx["scalars"]
        k = self.fresh("k")
        clauses = ""
        if r.random() < self.cfg.p_fp_clause and scalars:
            clauses = " firstprivate(%s)" % r.choice(scalars)
        kind = r.choice(["target teams distribute parallel for",
                         "target teams distribute parallel for",
                         "target parallel for", "target"])
        e = self.e
        e.line("#pragma omp %s%s" % (kind, clauses))
        e.line("for (int %s = 0; %s < %d; ++%s) {" % (k, k, self.cfg.size, k))
        e.ind += 1
        n = r.randrange(1, 4)
        kscal = [s for s in scalars if s not in ctx.get("no_dev_write", ())]
        for _ in range(n):
            e.line(self.assign(arrays, scalars, [k], arrays,
                               kscal if r.random() < 0.1 else []))
        if r.random() < 0.1 and ctx["callees_dev"]:
            e.line("%s;" % self.call_expr(ctx, [k], device=True))
        e.ind -= 1
        e.line("}")
        ctx["kernels"] += 1

    def call_expr(self, ctx, ivars, device=False) -> str:
        r = self.r
        fn = r.choice(ctx["callees_dev"] if device else ctx["callees"])
        args = []
        for pname, is_ptr in fn.params:
            if is_ptr:
                args.append(r.choice(ctx["arrays"]))
            else:
                args.append(r.choice(ctx["scalars"] + ["1.0"]))
        return "%s(%s)" % (fn.name, ", ".join(args))

    def block(self, ctx, budget: int, depth: int, loop_depth: int, ivars) -> None:
        for _ in range(budget):
            self.stmt(ctx, depth, loop_depth, ivars)

    def body(self, ctx, depth, loop_depth, ivars, braceless_ok=True) -> None:
        """A statement body; usually braced."""
        r = self.r
        e = self.e
        if braceless_ok and r.random() < self.cfg.p_braceless:
            e.ind += 1
            self.simple(ctx, ivars)
            e.ind -= 1
            return
        e.line("{")
        e.ind += 1
        self.block(ctx, r.randrange(1, 4), depth + 1, loop_depth, ivars)
        e.ind -= 1
        e.line("}")

    def simple(self, ctx, ivars) -> None:
        r = self.r
        if r.random() < self.cfg.p_kernel:
            self.kernel(ctx)
            return
        if ctx["callees"] and r.random() < self.cfg.p_call:
            self.e.line("%s;" % self.call_expr(ctx, ivars))
            return
        self.e.line(self.assign(ctx["arrays"], ctx["scalars"], ivars,
                                ctx["arrays"], ctx["scalars"]))

    def stmt(self, ctx, depth: int, loop_depth: int, ivars) -> None:
        r = self.r
        e = self.e
        cfg = self.cfg
        x = r.random()
        can_nest = depth < cfg.max_depth
        if can_nest and x < cfg.p_if:
            braceless = r.random() < cfg.p_braceless
            e.line("if (%s > %s)%s" % (self.rvalue(ctx["arrays"], ctx["scalars"], ivars),
                                      self.rvalue([], ctx["scalars"], ivars),
                                      "" if braceless else " {"))
            if braceless:
                e.ind += 1
                self.simple(ctx, ivars)
                e.ind -= 1
            else:
                e.ind += 1
                self.block(ctx, r.randrange(1, 4), depth + 1, loop_depth, ivars)
                e.ind -= 1
                e.line("}")
            if r.random() < 0.5:
                e.line("else {")
                e.ind += 1
                self.block(ctx, r.randrange(1, 3), depth + 1, loop_depth, ivars)
                e.ind -= 1
                e.line("}")
            return
        x -= cfg.p_if
        if can_nest and x < cfg.p_switch:
            e.line("switch (%s) {" % r.choice(ctx["iscalars"]))
            e.ind += 1
            ncase = r.randrange(1, 4)
            for ci in range(ncase):
                e.line("case %d:" % ci)
                e.ind += 1
                self.block(ctx, r.randrange(0, 3), depth + 1, loop_depth, ivars)
                if r.random() < 0.7:
                    e.line("break;")
                e.ind -= 1
            if r.random() < 0.5:
                e.line("default:")
                e.ind += 1
                self.block(ctx, r.randrange(0, 2), depth + 1, loop_depth, ivars)
                e.ind -= 1
            e.ind -= 1
            e.line("}")
            return
        x -= cfg.p_switch
        if can_nest and loop_depth < cfg.max_loop_depth and x < cfg.p_loop:
            kind = r.random()
            if kind < 0.7:
                iv = self.fresh("i")
                bound = r.choice([str(cfg.size), "%d" % r.randrange(2, 9)])
                e.line("for (int %s = 0; %s < %s; ++%s)" % (iv, iv, bound, iv))
                e.lines[-1] += " "
                if r.random() < cfg.p_braceless:
                    e.lines[-1] = e.lines[-1].rstrip()
                    e.ind += 1
                    self.simple(ctx, ivars + [iv])
                    e.ind -= 1
                else:
                    e.lines[-1] += "{"
                    e.ind += 1
                    self.block(ctx, r.randrange(1, 4), depth + 1, loop_depth + 1, ivars + [iv])
                    e.ind -= 1
                    e.line("}")
            elif kind < 0.85:
                c = r.choice(ctx["iscalars"])
                e.line("while (%s < %d) {" % (c, r.randrange(3, 9)))
                e.ind += 1
                self.block(ctx, r.randrange(1, 3), depth + 1, loop_depth + 1, ivars)
                e.line("%s = %s + 1;" % (c, c))
                e.ind -= 1
                e.line("}")
            else:
                c = r.choice(ctx["iscalars"])
                e.line("do {")
                e.ind += 1
                self.block(ctx, r.randrange(1, 3), depth + 1, loop_depth + 1, ivars)
                e.line("%s = %s + 1;" % (c, c))
                e.ind -= 1
                e.line("} while (%s < %s);" % (c, self.rvalue(ctx["arrays"], [], ivars)
                                                if r.random() < 0.4 else str(r.randrange(3, 9))))
            return
        if loop_depth > 0 and r.random() < cfg.p_jump:
            e.line("if (%s > 3.0) {" % self.rvalue(ctx["arrays"], ctx["scalars"], ivars))
            e.ind += 1
            e.line(r.choice(["break;", "continue;"]))
            e.ind -= 1
            e.line("}")
            return
        self.simple(ctx, ivars)

    # ---- functions / program ---------------------------------------------
    def function(self, fn: _Fn, ret: str, globals_, gscalars, callees, is_main=False) -> None:
        r = self.r
        cfg = self.cfg
        e = self.e
        params = []
        for pname, is_ptr in fn.params:
            params.append(("double *%s" % pname) if is_ptr else ("double %s" % pname))
        if is_main:
            params = ["int argc"]
        e.line("%s %s(%s) {" % (ret, fn.name, ", ".join(params) if params else "void"))
        e.ind += 1
        larrays = [self.fresh("la") for _ in range(cfg.n_locals)]
        lscal = [self.fresh("ls") for _ in range(cfg.n_lscalars)]
        iscal = [self.fresh("it")]
        for a in larrays:
            e.line("double %s[%d];" % (a, cfg.size + 2))
        for s in lscal:
            e.line("double %s = %d.0;" % (s, r.randrange(0, 5)))
        for s in iscal:
            e.line("int %s = 0;" % s)
        arrays = list(globals_) + larrays + [p for p, isp in fn.params if isp]
        scalars = list(gscalars) + lscal + [p for p, isp in fn.params if not isp]
        ctx = {"arrays": arrays, "scalars": scalars, "iscalars": iscal,
               "callees": callees, "callees_dev": [c for c in callees if c.name.startswith("dev")],
               "kernels": 0}
        n = max(1, cfg.n_stmts)
        late = cfg.p_late_decl and r.random() < cfg.p_late_decl
        for i in range(n):
            if late and ctx["kernels"] > 0:
                late = False
                nm = self.fresh("late")
                e.line("double %s[%d];" % (nm, cfg.size + 2))
                ctx["arrays"].append(nm)
            self.stmt(ctx, 0, 0, [])
        if ret == "int":
            e.line("return (int) %s;" % self.rvalue(arrays, scalars, []))
        elif ret == "double":
            e.line("return %s;" % self.rvalue(arrays, scalars, []))
        e.ind -= 1
        e.line("}")
        e.line("")

    def program(self) -> str:
        cfg = self.cfg
        r = self.r
        e = self.e
        e.line("#define N %d" % cfg.size)
        globals_ = ["g%d" % i for i in range(cfg.n_globals)]
        gscalars = ["gs%d" % i for i in range(cfg.n_gscalars)]
        for g in globals_:
            e.line("double %s[%d];" % (g, cfg.size + 2))
        for s in gscalars:
            e.line("double %s;" % s)
        e.line("double ext_reduce(const double *v, int n);")
        e.line("")
        fns: list[_Fn] = []
        for i in range(cfg.n_funcs):
            name = ("dev_f%d" if r.random() < 0.3 else "f%d") % i
            f = _Fn(name, [("p%d" % j, True) for j in range(cfg.n_ptr_params)]
                    + [("x%d" % i, False)])
            fns.append(f)
        # callees come earlier in the file: define in reverse so f_i may call f_j (j>i)
        for i in reversed(range(len(fns))):
            self.function(fns[i], "void", globals_, gscalars, fns[i + 1:])
        self.function(_Fn("main"), "int", globals_, gscalars, fns, is_main=True)
        return "\n".join(e.lines) + "\n"


def generate(seed: int, cfg: GenConfig | None = None) -> str:
    return ProgramGen(seed, cfg).program()
