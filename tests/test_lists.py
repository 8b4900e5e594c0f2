"""CPU: host-side list forms of kernels (a)+(b) (include/dfx.h dfx_acc_in /
dfx_req_list) -- numpy converters between dense planes and per-node lists."""
import numpy as np

import _mfp_ref
from paper_2406_13881_b200.csr import REQ_FP_FLAG, lists_to_planes, planes_to_acc


def test_planes_to_acc_round_trip():
    rng = np.random.default_rng(7)
    for words in (4, 8, 132):
        _, _, _, R, W, _ = _mfp_ref.random_graph(rng, 300, words)
        off, acc = planes_to_acc(R, W)
        assert off[0] == 0 and off[-1] == acc.shape[0]
        kind = acc >> 14
        assert np.all((kind >= 1) & (kind <= 3))
        # reads = entries with the read bit, writes = entries with the write bit
        rd, _ = lists_to_planes(off, np.where(kind & 1, acc & 0x3FFF, 0x4000).astype(np.uint16),
                                words, 0x4000)
        wr, _ = lists_to_planes(off, np.where(kind & 2, acc & 0x3FFF, 0x4000).astype(np.uint16),
                                words, 0x4000)
        assert np.array_equal(rd, R) and np.array_equal(wr, W)
        # ascending variables inside each node
        for i in range(0, 300, 17):
            v = (acc[off[i]:off[i + 1]] & 0x3FFF).astype(np.int64)
            assert np.all(np.diff(v) > 0)


def test_requirement_lists_split_on_firstprivate_flag():
    off = np.array([0, 3, 3, 5], dtype=np.int64)
    ent = np.array([1, 40, 5 | REQ_FP_FLAG, 127, 0 | REQ_FP_FLAG], dtype=np.uint16)
    req, fp = lists_to_planes(off, ent, 4, REQ_FP_FLAG)
    assert req[0, 0] == 2 and req[0, 1] == 1 << 8 and fp[0, 0] == 1 << 5
    assert not req[1].any() and not fp[1].any()
    assert req[2, 3] == 1 << 31 and fp[2, 0] == 1


def test_event_order_is_function_then_key():
    """`dataflow._event_order`: the combined 64-bit sort and the lexsort
    fallback (a key too wide to share 64 bits with the function index)."""
    import numpy as np
    from paper_2406_13881_b200 import _abi
    from paper_2406_13881_b200.dataflow import _event_order
    rng = np.random.default_rng(9)
    for wide in (False, True):
        n = 5000
        ev = np.zeros(n, dtype=_abi.EVENT_DTYPE)
        ev["fn"] = rng.integers(0, 3000, n)
        ev["key"] = rng.permutation(n).astype(np.uint64) << np.uint64(24)
        if wide:
            ev["key"][0] |= np.uint64(1) << np.uint64(62)
        o = _event_order(ev)
        exp = np.lexsort((ev["key"], ev["fn"]))
        assert np.array_equal(ev["fn"][o], ev["fn"][exp]) and np.array_equal(ev["key"][o], ev["key"][exp])


def test_first_occurrences_matches_a_python_scan():
    """`dataflow._first_occurrences` (the event dedup before decode), both the
    packed-key path and the lexsort path (forced by an out-of-range node)."""
    import numpy as np
    from paper_2406_13881_b200 import _abi
    from paper_2406_13881_b200.dataflow import _first_occurrences
    rng = np.random.default_rng(5)
    for big in (False, True):
        n = 3000
        ev = np.zeros(n, dtype=_abi.EVENT_DTYPE)
        ev["fn"] = np.sort(rng.integers(0, 40, n))
        ev["key"] = np.arange(n)
        ev["var"] = rng.integers(-1, 6, n)
        ev["node"] = rng.integers(0, 5, n) + (70000 if big else 0)
        ev["kind"] = rng.integers(1, 5, n)
        ev["pos"] = rng.integers(0, 3, n)
        ev["kind"][::97] = _abi.EV_ERR_DATAMAP          # errors are always kept
        seen, exp = set(), np.zeros(n, dtype=bool)
        for i, e in enumerate(ev):
            k = (int(e["fn"]), int(e["var"]), int(e["node"]), int(e["kind"]), int(e["pos"]))
            exp[i] = k not in seen or int(e["kind"]) >= _abi.EV_ERR_DATAMAP
            seen.add(k)
        assert np.array_equal(_first_occurrences(ev["fn"], ev["var"], ev["node"], ev["kind"],
                                                 ev["pos"]), exp)
