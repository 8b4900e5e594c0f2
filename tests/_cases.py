"""Shared parity-case helpers: seeded program configs and canonical plan forms."""
from __future__ import annotations

import random

from paper_2406_13881_b200.gen.cprog import GenConfig, generate


def random_cfg(seed: int) -> GenConfig:
    r = random.Random(seed)
    return GenConfig(n_funcs=r.randrange(0, 3), n_stmts=r.randrange(3, 14),
                     max_depth=r.randrange(2, 5), max_loop_depth=r.randrange(1, 4),
                     p_braceless=r.choice([0, 0, 0.1]), p_late_decl=r.choice([0, 0, 0.3]),
                     p_jump=0.06)


def random_program(seed: int) -> str:
    return generate(seed, random_cfg(seed))


def _sp(node):
    return [node.span.start, node.span.end]


def canon_plan(plan) -> dict:
    """FunctionPlan -> JSON-able form keyed by source spans (object identity of
    anchors is checked separately by the in-process comparisons)."""
    r = plan.region
    reg = None
    if r is not None:
        reg = {"block": _sp(r.block), "begin": _sp(r.begin), "end": _sp(r.end),
               "to": list(r.map_to), "from": list(r.map_from),
               "tofrom": list(r.map_tofrom), "alloc": list(r.map_alloc)}
    dp = lambda c: [c.kind.value, list(c.names), _sp(c.anchor), c.position]  # noqa: E731
    return {"function": plan.function.name, "region": reg,
            "kernel_clauses": [dp(c) for c in plan.kernel_clauses],
            "updates": [dp(c) for c in plan.updates],
            "suppressed": list(plan.suppressed)}


def canon_result(fn):
    """Run `fn()` -> ("ok", canon plan) or ("err", type name, rendered text)."""
    try:
        return ["ok", canon_plan(fn())]
    except Exception as e:  # reference ToolError subclasses
        msg = e.render() if hasattr(e, "render") else str(e)
        return ["err", type(e).__name__, msg]


def identity_equal(a, b) -> bool:
    """Anchor identity check between two FunctionPlans on the same AST."""
    if (a.region is None) != (b.region is None):
        return False
    if a.region is not None:
        ra, rb = a.region, b.region
        if not (ra.block is rb.block and ra.begin is rb.begin and ra.end is rb.end):
            return False
    for xa, xb in ((a.kernel_clauses, b.kernel_clauses), (a.updates, b.updates)):
        if len(xa) != len(xb):
            return False
        for pa, pb in zip(xa, xb):
            if pa.anchor is not pb.anchor or pa != pb:
                return False
    return True
