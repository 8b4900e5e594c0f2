"""Generate the parity fixtures under tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py

For every case -- the reference's 27-file corpus (pkg/tests/corpus), the
SURVEY Appendix-D probe programs (tests/golden/probes/) and seeded random
structured programs (paper_2406_13881_b200/gen/cprog.py) -- it runs the
reference `dartomp` 0.1.0 in-process and records:

* reference_plans.json: per case, per function, the reference
  `analyze_function` result in span-canonical form (or the exception type and
  rendered message), plus `dart-omp report` lines and the sha256 of the
  `transform` output text;
* replay_batch.npz: the lowered E1 programs of all those functions packed as
  one `dfx_replay_in` batch, and the expected raw engine output (events sorted
  by (fn, key), per-variable bits) -- produced by the CPU oracle and accepted
  only after the oracle's decoded plans matched the reference's exactly
  (including anchor object identity).  GPU tests compare the CUDA engine's raw
  output against this, so they need neither the reference nor its front end.
"""
from __future__ import annotations

import hashlib
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
REF_SRC = pathlib.Path("/root/reference/pkg/src")
if REF_SRC.exists():
    sys.path.insert(0, str(REF_SRC))

import dartomp  # noqa: E402
from dartomp.dataflow import analyze_function as ref_analyze  # noqa: E402
from dartomp.pipeline import load, transform  # noqa: E402
from dartomp.report import plan_lines  # noqa: E402

import _cases  # noqa: E402
import _oracle  # noqa: E402
from paper_2406_13881_b200 import _abi  # noqa: E402
from paper_2406_13881_b200.dataflow import decode, pack, run_replay  # noqa: E402
from paper_2406_13881_b200.lower import lower_function  # noqa: E402
from paper_2406_13881_b200 import interproc as ip  # noqa: E402
from paper_2406_13881_b200.gen.callgraph import CallGraphConfig  # noqa: E402
from paper_2406_13881_b200.gen.callgraph import generate as gen_callgraph  # noqa: E402
from dartomp.interproc import summarize_all as ref_summarize  # noqa: E402

N_RANDOM = 120
N_CALLGRAPH = 6          # generated call-graph programs (configuration C5 shape)


def cases():
    corpus = pathlib.Path("/root/reference/pkg/tests/corpus")
    for p in sorted(corpus.glob("*/*.c")):
        yield "corpus/%s/%s" % (p.parent.name, p.name), p.read_text()
    for p in sorted((HERE / "probes").glob("*.c")):
        yield "probe/%s" % p.name, p.read_text()
    for s in range(N_RANDOM):
        yield "random/%d" % s, _cases.random_program(s)


def main() -> None:
    print("reference dartomp from", dartomp.__file__)
    plans_json = {}
    progs, metas = [], []
    for name, text in cases():
        try:
            a = load(path=name, text=text)
        except Exception as e:
            print("skip (front end rejects)", name, e)
            continue
        entry = {"functions": {}}
        try:
            result, plans = transform(a)
            entry["report"] = plan_lines(a.src, plans)
            entry["transform_sha256"] = hashlib.sha256(result.text.encode()).hexdigest()
        except KeyError as e:          # report.py:35 has no AFTER key
            entry["report"] = ["<KeyError %s>" % e]
            entry["transform_sha256"] = hashlib.sha256(
                transform(a)[0].text.encode()).hexdigest()
        except Exception as e:
            entry["report"] = ["<%s: %s>" % (type(e).__name__, e.render() if hasattr(e, "render") else e)]
        for fname in a.cfgs:
            ref = _cases.canon_result(
                lambda: ref_analyze(a.src, a.cfgs[fname], a.accesses[fname], a.table))
            entry["functions"][fname] = ref
            progs.append(lower_function(a.src, a.cfgs[fname], a.accesses[fname], a.table))
            metas.append((name, fname, a))
        plans_json[name] = entry
    batch = pack(progs)
    raw = run_replay(batch, runner=_oracle.replay_runner)
    order = np.lexsort((raw.events["key"], raw.events["fn"]))
    evs = raw.events[order]
    bounds = np.searchsorted(evs["fn"], np.arange(len(progs) + 1))
    n_bad = 0
    for i, (p, (name, fname, a)) in enumerate(zip(progs, metas)):
        d = batch.fns[i]
        vo = raw.var_out[int(d["var_off"]):int(d["var_off"]) + int(d["n_vars"])]
        ev = evs[bounds[i]:bounds[i + 1]]
        got = _cases.canon_result(lambda: decode(p, a.src, a.accesses[fname], ev, vo))
        ref = plans_json[name]["functions"][fname]
        if got != ref:
            n_bad += 1
            print("MISMATCH", name, fname, "\n ref", ref, "\n got", got)
            continue
        if ref[0] == "ok":
            mine = decode(p, a.src, a.accesses[fname], ev, vo)
            theirs = ref_analyze(a.src, a.cfgs[fname], a.accesses[fname], a.table)
            if not _cases.identity_equal(mine, theirs):
                n_bad += 1
                print("ANCHOR IDENTITY MISMATCH", name, fname)
    if n_bad:
        raise SystemExit("%d mismatches: fixtures NOT written" % n_bad)
    np.savez_compressed(
        HERE / "replay_batch.npz",
        fns=batch.fns, ops=batch.ops, var_flags=batch.var_flags,
        stmt_span=batch.stmt_span, sites=batch.sites, arms=batch.arms,
        events=evs, var_out=raw.var_out)
    with open(HERE / "reference_plans.json", "w") as fh:
        json.dump(plans_json, fh, indent=0, sort_keys=True)
    print("cases %d functions %d events %d ops %d -> fixtures written"
          % (len(plans_json), len(progs), evs.shape[0], batch.ops.shape[0]))


def summary_cases():
    corpus = pathlib.Path("/root/reference/pkg/tests/corpus")
    for p in sorted(corpus.glob("*/*.c")):
        yield "corpus/%s/%s" % (p.parent.name, p.name), p.read_text()
    for s in range(40):
        yield "random/%d" % s, _cases.random_program(s)
    for s in range(N_CALLGRAPH):
        n = 1200 if s == 0 else 240
        yield "callgraph/%d" % s, gen_callgraph(s, CallGraphConfig(n_funcs=n, depth=12))


def summaries_main() -> None:
    """Fixtures for kernel (c): lowered call graphs + the reference's
    summaries (sets and dict insertion orders), checked through the oracle."""
    arrays = {}
    expected = {}
    n = 0
    for name, text in summary_cases():
        a = load(path=name, text=text)
        ref = ref_summarize(a.src, a.tu, a.cfgs, a.raw_accesses, a.table)
        g = ip.lower_call_graph(a.src, a.tu, a.cfgs, a.raw_accesses, a.table)
        r = ip.solve_call_graph(g, runner=_oracle.summaries_runner)
        mine = ip.summaries_from_result(g, r)
        assert list(mine) == list(ref), name
        for k in ref:
            assert mine[k].snapshot() == ref[k].snapshot(), (name, k)
            assert list(mine[k].param_effects.items()) == list(ref[k].param_effects.items()), (name, k)
            assert list(mine[k].global_effects.items()) == list(ref[k].global_effects.items()), (name, k)
        key = "c%d" % n
        for fld in ("init_bits", "init_list", "init_len", "direct", "src_off", "src", "slist",
                    "bind", "wave_off", "wave_fns"):
            arrays["%s_%s" % (key, fld)] = getattr(g, fld)
        arrays["%s_meta" % key] = np.array([g.n_funcs, g.n_params, r.passes], dtype=np.int64)
        arrays["%s_exp_bits" % key] = r.bits
        arrays["%s_exp_list" % key] = r.list
        arrays["%s_exp_len" % key] = r.len
        expected[key] = {"case": name, "functions": g.n_funcs, "slots": int(g.init_bits.shape[1]),
                         "passes": int(r.passes),
                         "snapshots": {k: repr(v.snapshot()) for k, v in list(ref.items())[:3]}}
        n += 1
    np.savez_compressed(HERE / "summary_cases.npz", **arrays)
    with open(HERE / "summary_cases.json", "w") as fh:
        json.dump(expected, fh, indent=0, sort_keys=True)
    print("summary cases %d -> fixtures written" % n)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "summaries":
        summaries_main()
    else:
        main()
        summaries_main()
