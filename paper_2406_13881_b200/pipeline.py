"""Drop-in driver: the reference's `load` / `plan_transform` / `transform`
(`dartomp/pipeline.py:38-105`) with the hot path swapped for the engine.

The lexer, AST-CFG and access classification are the host package's own; the
parser is `frontend.py`'s (the reference's tree, checked node for node in
`tests/test_frontend.py`); `summarize_all` runs on kernel (c), every
function's data-flow analysis runs in ONE batched launch of the E1 replay
kernel, and the emitter is native (`emit.py`).

`install()` patches a live `dartomp` in place (its `pipeline` and `cli`
modules pick the engine up), which is how an existing user -- including
`python -m dartomp ...` -- switches over.
"""
from __future__ import annotations

from ._host import import_dartomp

import_dartomp()
from dartomp.access import VariableTable, classify_accesses  # noqa: E402
from dartomp.astcfg import build_astcfg  # noqa: E402
from dartomp.lexer import expand_defines  # noqa: E402
from dartomp.nodes import defined_functions  # noqa: E402
from dartomp.diagnostics import PreconditionError  # noqa: E402
from dartomp.omp import DATA_MAPPING_KINDS  # noqa: E402
from dartomp.pipeline import Analysis, check_transform_preconditions  # noqa: E402
from dartomp.source import SourceFile  # noqa: E402

from .dataflow import analyze_function, analyze_functions  # noqa: E402
from .emit import apply_plans, plan_lines  # noqa: E402
from .frontend import parse, paused_gc  # noqa: E402
from .lower import premapped_directive  # noqa: E402
from .interproc import apply_call_effects, summarize_all  # noqa: E402


def load(path: str | None = None, text: str | None = None,
         sizes: dict[str, int] | None = None, pointer_default: int = 1024,
         summary_runner=None) -> Analysis:
    """`dartomp.pipeline.load` (`pipeline.py:38-62`) with kernel (c), the
    drop-in parser (`frontend.py`: the reference's tree by precedence
    climbing) and the cyclic collector paused for the call."""
    with paused_gc():
        if text is not None:
            src = SourceFile.from_text(text, path=path or "<string>")
        else:
            src = SourceFile.from_path(path)
        pre = expand_defines(src)
        tu, pwarnings = parse(src, pre)
        table = VariableTable(src, tu, sizes=sizes, pointer_default=pointer_default)
        warnings = list(pre.warnings) + list(pwarnings)
        cfgs, raw = {}, {}
        for name, fn in defined_functions(tu).items():
            cfg = build_astcfg(src, fn)
            cfgs[name] = cfg
            warnings.extend(cfg.warnings)
            raw[name] = classify_accesses(src, cfg, table)
        summaries = summarize_all(src, tu, cfgs, raw, table, runner=summary_runner)
        expanded = {name: apply_call_effects(src, cfgs[name], raw[name], summaries, table)
                    for name in cfgs}
        return Analysis(src=src, tu=tu, table=table, cfgs=cfgs, raw_accesses=raw,
                        accesses=expanded, summaries=summaries,
                        defines=dict(pre.defines), warnings=warnings)


def _precheck(analysis: Analysis, names: list):
    """`check_transform_preconditions` (`pipeline.py:65-82`) over the unit in
    the same pre-order: each function's first refused directive comes from
    its lowering (`FnProgram.premapped`, found in the lowering workers); only
    the nodes outside function definitions are walked here.  Raises the same
    `PreconditionError` for the same first directive."""
    def check(progs):
        by_root = {id(analysis.cfgs[n].function): p for n, p in zip(names, progs)}
        for top in analysis.tu.children:
            p = by_root.get(id(top))
            node = p.premapped if p is not None else premapped_directive(top)
            if node is None:
                continue
            src, info = analysis.src, node.omp
            line = src.line_of(node.span.start)
            if info.kind in DATA_MAPPING_KINDS:
                raise PreconditionError(
                    "input already contains a '%s' directive; the transform "
                    "expects offload regions without data-mapping constructs"
                    % info.kind.value, path=src.path, line=line)
            raise PreconditionError(
                "input already contains a 'map' clause on an offload "
                "directive; the transform expects unannotated kernels",
                path=src.path, line=line)
    return check


def plan_transform(analysis: Analysis, allow_stale: frozenset[str] = frozenset(),
                   replay_runner=None) -> list:
    """`dartomp.pipeline.plan_transform` (`pipeline.py:85-96`), one launch."""
    names = list(analysis.cfgs)
    items = [(analysis.src, analysis.cfgs[n], analysis.accesses[n], analysis.table)
             for n in names]
    try:
        results = analyze_functions(items, allow_stale, runner=replay_runner,
                                    precheck=_precheck(analysis, names))
    except PreconditionError:
        raise
    except Exception:
        check_transform_preconditions(analysis)   # the reference checks first
        raise
    plans = []
    for res in results:
        plan = res.get()            # raises the reference's error for that function
        if plan.region is not None or plan.all_plans:
            plans.append(plan)
    return plans


def transform(analysis: Analysis, allow_stale: frozenset[str] = frozenset(),
              indent_unit: str | None = None, replay_runner=None):
    """`dartomp.pipeline.transform` (`pipeline.py:99-105`): plans from one E1
    launch, text from the native emitter (`emit.py`, byte-identical to
    `rewriter.apply_plans`)."""
    plans = plan_transform(analysis, allow_stale, replay_runner=replay_runner)
    result = apply_plans(analysis.src, plans, indent_unit=indent_unit)
    return result, plans


def install() -> None:
    """Route an imported `dartomp` through the engine (plugin drop-in): the
    analysis (E1), the summaries (kernel c), `load` (its parser and paused
    collector, `frontend.py`), the emitter (native), and the CLI's `compare`
    (the CUDA transfer simulator; its comparison lines are the reference's
    byte for byte).  `simulate_analysis` (the CLI's `simulate`
    mode, whose verbose log lists the reference's per-round records) stays the
    reference's."""
    import dartomp.cli as cli
    import dartomp.dataflow as df
    import dartomp.interproc as ip
    import dartomp.pipeline as pl
    import dartomp.report as rp
    import dartomp.rewriter as rw
    from .simulator import compare
    df.analyze_function = analyze_function
    ip.summarize_all = summarize_all
    pl.analyze_function = analyze_function
    pl.summarize_all = summarize_all
    pl.plan_transform = plan_transform
    pl.load = load
    pl.transform = transform
    pl.apply_plans = apply_plans
    pl.compare = compare
    rw.apply_plans = apply_plans
    rp.plan_lines = plan_lines
    cli.load = load
    cli.transform = transform
    cli.plan_lines = plan_lines
    cli.compare = compare
