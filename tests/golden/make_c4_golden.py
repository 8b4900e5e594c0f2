"""Generate tests/golden/c4_source_plans.json.gz from the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_c4_golden.py

Configuration C4 as C source (paper_2406_13881_b200/gen/c4src.py): a fixed
sample of the batch's functions (64-2048 host CFG nodes, V_f in
{32..512}), each parsed by the reference front end and analysed by the
reference `analyze_function` (`dartomp/dataflow.py:737-740`) in-process.  Per
function the fixture holds the span-canonical plan (tests/_cases.canon_plan),
the CFG node count and the number of variables touched, so the GPU test
(tests/test_c4_source.py) can compare the CUDA drop-in with the reference
without the reference on the box.  One process per core; test
infrastructure only.
"""
from __future__ import annotations

import gzip
import json
import multiprocessing as mp
import pathlib
import sys

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
REF_SRC = pathlib.Path("/root/reference/pkg/src")
if REF_SRC.exists():
    sys.path.insert(0, str(REF_SRC))

from paper_2406_13881_b200.gen.c4src import C4SourceConfig, c4_source  # noqa: E402

SAMPLE = list(range(0, 100_000, 389))[:256]      # 256 functions across the batch
OUT = HERE / "c4_source_plans.json.gz"


def one(i: int):
    import dartomp
    from dartomp.dataflow import analyze_function
    from dartomp.pipeline import load
    import _cases
    assert str(REF_SRC) in dartomp.__file__ or "baseline/_ref" in dartomp.__file__
    a = load(text=c4_source(C4SourceConfig(), i))
    name = "c4_%d" % i
    cfg, accs = a.cfgs[name], a.accesses[name]
    res = _cases.canon_result(lambda: analyze_function(a.src, cfg, accs, a.table))
    return {"i": i, "nodes": len(cfg.nodes), "vars": len({id(x.var) for x in accs}),
            "result": res}


def main():
    with mp.Pool() as pool:
        rows = pool.map(one, SAMPLE, chunksize=1)
    errs = [r["i"] for r in rows if r["result"][0] != "ok"]
    assert not errs, "C4 functions must analyse cleanly: %s" % errs[:5]
    data = {"config": {"seed": 0, "n_min": 64, "n_max": 2048,
                       "var_choices": [32, 64, 128, 256, 512]},
            "functions": rows}
    OUT.write_bytes(gzip.compress(json.dumps(data, separators=(",", ":")).encode(), 9))
    facts = sum(r["nodes"] * r["vars"] for r in rows)
    print("wrote %s: %d functions, %d facts, %d bytes" % (OUT, len(rows), facts, OUT.stat().st_size))


if __name__ == "__main__":
    main()
