"""Generate tests/golden/c5_reference_summaries.json.gz from the REFERENCE.

Run here (where /root/reference exists):  python tests/golden/make_c5_golden.py

Configuration C5 at full size: the 10,000-function call graph (833 chains of
depth 12, 10% back edges, externals, prototypes, kernel call sites) emitted
as C by paper_2406_13881_b200/gen/callgraph.py (seed 7), parsed by the
reference front end, and summarised by the reference `summarize_all`
(`dartomp/interproc.py:90-144`) in-process.  The fixture holds, per defined
function, both summary dicts IN INSERTION ORDER (the order is part of the
output: apply_call_effects turns it into access order), plus the timing of
the reference's own summarize_all (front end excluded).  TEST INFRASTRUCTURE.
"""
from __future__ import annotations

import gzip
import json
import pathlib
import sys
import time

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
REF_SRC = pathlib.Path("/root/reference/pkg/src")
if REF_SRC.exists():
    sys.path.insert(0, str(REF_SRC))

from paper_2406_13881_b200.gen.callgraph import CallGraphConfig, generate  # noqa: E402

OUT = HERE / "c5_reference_summaries.json.gz"
SEED, N_FUNCS = 7, 10_000


def canon_summaries(summ: dict) -> dict:
    def eff(e):
        return [e.kind.value, sorted(s.value for s in e.spaces)]
    return {name: [[[int(i), *eff(e)] for i, e in s.param_effects.items()],
                   [[g, *eff(e)] for g, e in s.global_effects.items()]]
            for name, s in summ.items()}


def main():
    from dartomp.access import VariableTable, classify_accesses
    from dartomp.astcfg import build_astcfg
    from dartomp.interproc import summarize_all
    from dartomp.nodes import defined_functions
    from dartomp.parser import parse
    from dartomp.lexer import expand_defines
    from dartomp.source import SourceFile
    text = generate(SEED, CallGraphConfig(n_funcs=N_FUNCS, depth=12))
    src = SourceFile.from_text(text, path="c5.c")
    pre = expand_defines(src)
    tu, _ = parse(src, pre)
    table = VariableTable(src, tu)
    cfgs, raw = {}, {}
    for name, fn in defined_functions(tu).items():
        cfgs[name] = build_astcfg(src, fn)
        raw[name] = classify_accesses(src, cfgs[name], table)
    t0 = time.perf_counter()
    summ = summarize_all(src, tu, cfgs, raw, table)
    dt = time.perf_counter() - t0
    data = {"seed": SEED, "n_funcs": N_FUNCS, "defined": len(cfgs),
            "reference_summarize_all_s": dt, "summaries": canon_summaries(summ)}
    OUT.write_bytes(gzip.compress(json.dumps(data, separators=(",", ":")).encode(), 9))
    print("wrote %s: %d summaries, reference summarize_all %.1f s, %d bytes"
          % (OUT, len(summ), dt, OUT.stat().st_size))


if __name__ == "__main__":
    main()
