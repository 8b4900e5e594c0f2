"""Worker side of the simulator bench (`bench.py` "sim" record): per C4
source function, the transformed program (host preparation, untimed), its
simulation lowering (`simlower.lower_program`, timed: the host half of the
verifier) and the reference `simulate` on the same program (timed: the CPU
baseline), with the reference's aggregate fields for the parity check.

Runs in spawned pool workers (no CUDA); the reference is the host package
`dartomp` (baseline/_ref on the GPU box)."""
from __future__ import annotations

import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent


def one(args):
    i, mode = args
    for p in (str(ROOT), str(ROOT / "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    from paper_2406_13881_b200._host import import_dartomp
    from paper_2406_13881_b200.gen.c4src import C4SourceConfig, c4_source
    from paper_2406_13881_b200.simlower import lower_program
    import_dartomp()
    import _sim
    from dartomp.pipeline import load, program_model, transform
    from dartomp.simulator import SimConfig, simulate
    a = load(text=c4_source(C4SourceConfig(), i), path="c4_%d.c" % i)
    if mode == "annotated":
        res, _ = transform(a)
        a = load(text=res.text, path="c4_%d.c (transformed)" % i)
    cfg = SimConfig(mode=mode)
    model = program_model(a)
    t0 = time.perf_counter()
    prog = lower_program(model, cfg)
    t1 = time.perf_counter()
    ref = simulate(program_model(a), cfg)
    t2 = time.perf_counter()
    return i, prog, _sim.aggregate_fields(ref), t1 - t0, t2 - t1
