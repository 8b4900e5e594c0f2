"""Replay ops in the 8-byte form (dfx_replay_batch_packed, include/dfx.h):
the packer round-trips every op of the corpus, generated and C4 programs and
refuses fields that do not fit; on the GPU the packed call returns exactly the
16-byte call's events and per-variable bits."""
import numpy as np
import pytest

from paper_2406_13881_b200.dataflow import pack_ops, unpack_ops


def _c4_batch(n=400, step=250):
    from paper_2406_13881_b200.batch import C4Config, c4_generate
    b, _ = c4_generate(C4Config(), np.arange(0, n * step, step, dtype=np.int32))
    return b


def test_pack_round_trip_c4():
    b = _c4_batch()
    pk = pack_ops(b.ops)
    assert pk is not None and pk.dtype == np.uint32 and pk.shape == (b.ops.shape[0], 2)
    assert np.array_equal(unpack_ops(pk), b.ops)


def test_pack_round_trip_lowered_programs():
    from paper_2406_13881_b200._host import have_dartomp
    if not have_dartomp():
        pytest.skip("host front end not importable")
    from dartomp.pipeline import load
    from paper_2406_13881_b200.dataflow import lower_functions, pack
    from paper_2406_13881_b200.gen.cprog import GenConfig, generate
    a = load(text=generate(5, GenConfig(n_funcs=20, n_globals=12, n_stmts=30, p_kernel=0.3)))
    items = [(a.src, a.cfgs[n], a.accesses[n], a.table) for n in a.cfgs]
    batch = pack(lower_functions(items))
    pk = pack_ops(batch.ops)
    assert pk is not None
    assert np.array_equal(unpack_ops(pk), batch.ops)


def test_pack_refuses_fields_that_do_not_fit():
    ops = np.zeros((3, 4), dtype=np.int32)
    ops[0] = (1, 70000, 3, 5)            # HR on variable 70000: more than 16 bits
    assert pack_ops(ops) is None
    ops[0] = (1, 7, 3, 1 << 23)          # site offset beyond 23 bits
    assert pack_ops(ops) is None
    ops[0] = (5, 0, 9, 0)                # BR_BEGIN with a non-zero reserved word
    assert pack_ops(ops) is None
    ops[0] = (1 | (1 << 9), 7, 3, 5)     # HR with a flag: fits
    assert np.array_equal(unpack_ops(pack_ops(ops)), ops)


@pytest.mark.gpu
def test_cuda_packed_equals_16_byte_form():
    """A C4 sub-batch large enough for the range pipeline (>= 256
    functions): identical events and per-variable bits."""
    from paper_2406_13881_b200.dataflow import ReplaySession
    b = _c4_batch(600, 160)
    pk = pack_ops(b.ops)
    sess = ReplaySession()
    ref = sess.run(b)
    ev_ref = np.sort(ref.events.copy(), order=["fn", "key", "var", "node", "kind", "pos"])
    vo_ref = ref.var_out.copy()
    got = ReplaySession().run(b, packed_ops=pk)
    ev = np.sort(got.events.copy(), order=["fn", "key", "var", "node", "kind", "pos"])
    assert ev.shape == ev_ref.shape and (ev == ev_ref).all()
    assert np.array_equal(got.var_out, vo_ref)


@pytest.mark.gpu
def test_cuda_packed_small_batch_single_range():
    """A batch below the range pipeline's threshold (one range) and a single
    function: packed == 16-byte form."""
    from paper_2406_13881_b200.dataflow import ReplaySession
    for n in (1, 30):
        b = _c4_batch(n, 997)
        ref = ReplaySession().run(b)
        got = ReplaySession().run(b, packed_ops=pack_ops(b.ops))
        key = ["fn", "key", "var", "node", "kind", "pos"]
        assert (np.sort(got.events.copy(), order=key) == np.sort(ref.events.copy(), order=key)).all()
        assert np.array_equal(got.var_out, ref.var_out)
