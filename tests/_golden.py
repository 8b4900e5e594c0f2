"""Loader for the committed parity fixtures (tests/golden/)."""
from __future__ import annotations

import json
import pathlib

import numpy as np

from paper_2406_13881_b200 import _abi
from paper_2406_13881_b200.dataflow import PackedBatch

HERE = pathlib.Path(__file__).resolve().parent / "golden"


def replay_fixture():
    z = np.load(HERE / "replay_batch.npz")
    batch = PackedBatch(fns=z["fns"], ops=z["ops"], var_flags=z["var_flags"],
                        stmt_span=z["stmt_span"], sites=z["sites"], arms=z["arms"])
    return batch, z["events"], z["var_out"]


def reference_plans() -> dict:
    return json.loads((HERE / "reference_plans.json").read_text())


def sort_events(ev):
    return ev[np.lexsort((ev["key"], ev["fn"]))]


def assert_raw_equal(got_events, got_var_out, exp_events, exp_var_out):
    g = sort_events(got_events)
    e = sort_events(exp_events)
    assert g.shape == e.shape, "event count %d != %d" % (g.shape[0], e.shape[0])
    for f in ("key", "fn", "var", "node", "kind", "pos"):
        bad = np.nonzero(g[f] != e[f])[0]
        assert bad.size == 0, "field %s differs at %s: got %s exp %s" % (
            f, bad[:5], g[bad[:5]], e[bad[:5]])
    assert np.array_equal(got_var_out, exp_var_out), "var_out differs at %s" % (
        np.nonzero(got_var_out != exp_var_out)[0][:10])


def summary_fixtures():
    """[(case name, CallGraph, (exp_bits, exp_list, exp_len, exp_passes))]"""
    from paper_2406_13881_b200.interproc import CallGraph
    z = np.load(HERE / "summary_cases.npz")
    meta = json.loads((HERE / "summary_cases.json").read_text())
    out = []
    for key in sorted(meta, key=lambda k: int(k[1:])):
        nf, n_params, passes = (int(x) for x in z["%s_meta" % key])
        bits = z["%s_init_bits" % key]
        g = CallGraph(names=["f%d" % i for i in range(nf)], fns=[None] * nf, n_params=n_params,
                      globals=["g%d" % i for i in range(bits.shape[1] - n_params)],
                      **{f: z["%s_%s" % (key, f)] for f in (
                          "init_bits", "init_len", "init_list", "direct", "src_off", "src",
                          "slist", "bind", "wave_off", "wave_fns")})
        out.append((meta[key]["case"], g, (z["%s_exp_bits" % key], z["%s_exp_list" % key],
                                           z["%s_exp_len" % key], passes)))
    return out


def assert_summary_equal(r, exp):
    eb, el, en, ep = exp
    assert np.array_equal(r.bits, eb), "summary bits differ"
    assert np.array_equal(r.len, en), "summary lengths differ"
    for f in range(en.shape[0]):
        assert np.array_equal(r.list[f, :en[f]], el[f, :en[f]]), "insertion order differs (fn %d)" % f
    assert r.passes == ep, "pass count %d != %d" % (r.passes, ep)
