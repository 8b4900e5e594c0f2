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
