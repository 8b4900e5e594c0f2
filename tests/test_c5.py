"""Configuration C5 (10k-function call graph, depth-12 chains) pinned to the
reference, and the component-sharded multi-rank summaries protocol.

* Full size vs the reference: the 10,000-function program (gen/callgraph.py,
  seed 7) through the drop-in `summarize_all` == the reference's
  `summarize_all` (`dartomp/interproc.py:90-144`) summaries, dict insertion
  order included, from the committed fixture
  tests/golden/c5_reference_summaries.json.gz (tests/golden/make_c5_golden.py).
* Component sharding (distributed.ComponentSummaries): one all-reduce per
  pass + one final all-gather; gloo world size 2 on CPU == the single-rank
  oracle; on the GPU, `dfx_summaries_sharded` over an NCCL communicator."""
import gzip
import json
import os
import pathlib
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import _oracle
from paper_2406_13881_b200._abi import LIB_PATH
from paper_2406_13881_b200._host import have_dartomp

GOLD = pathlib.Path(__file__).resolve().parent / "golden" / "c5_reference_summaries.json.gz"


def _canon(summ: dict) -> dict:
    def eff(e):
        return [e.kind.value, sorted(s.value for s in e.spaces)]
    return {name: [[[int(i), *eff(e)] for i, e in s.param_effects.items()],
                   [[g, *eff(e)] for g, e in s.global_effects.items()]]
            for name, s in summ.items()}


def _front_end_10k():
    from paper_2406_13881_b200._host import import_dartomp
    import_dartomp()
    from dartomp.access import VariableTable, classify_accesses
    from dartomp.astcfg import build_astcfg
    from dartomp.lexer import expand_defines
    from dartomp.nodes import defined_functions
    from dartomp.parser import parse
    from dartomp.source import SourceFile
    from paper_2406_13881_b200.gen.callgraph import CallGraphConfig, generate
    gold = json.loads(gzip.decompress(GOLD.read_bytes()))
    text = generate(gold["seed"], CallGraphConfig(n_funcs=gold["n_funcs"], depth=12))
    src = SourceFile.from_text(text, path="c5.c")
    pre = expand_defines(src)
    tu, _ = parse(src, pre)
    table = VariableTable(src, tu)
    cfgs, raw = {}, {}
    for name, fn in defined_functions(tu).items():
        cfgs[name] = build_astcfg(src, fn)
        raw[name] = classify_accesses(src, cfgs[name], table)
    return gold, (src, tu, cfgs, raw, table)


@pytest.mark.skipif(not have_dartomp(), reason="host front end absent")
def test_c5_full_size_oracle_equals_reference():
    """The lowering + the CPU oracle at 10k functions == the reference."""
    from paper_2406_13881_b200 import interproc as ip
    gold, fe = _front_end_10k()
    assert _canon(ip.summarize_all(*fe, runner=_oracle.summaries_runner)) == gold["summaries"]


@pytest.mark.skipif(not have_dartomp(), reason="host front end absent")
@pytest.mark.gpu
@pytest.mark.skipif(not LIB_PATH.exists(), reason="libdfx.so not built")
def test_c5_full_size_cuda_equals_reference():
    """10k functions: drop-in summarize_all on CUDA == the reference's
    summaries and dict orders; the component-sharded path (NCCL, one rank)
    gives the same rows with passes + 0 collectives beyond the per-pass flag."""
    from paper_2406_13881_b200 import interproc as ip
    from paper_2406_13881_b200.distributed import ComponentSummaries
    gold, fe = _front_end_10k()
    got = ip.summarize_all(*fe)
    assert _canon(got) == gold["summaries"]
    g = ip.lower_call_graph(*fe)
    exp = ip.solve_call_graph(g)
    cs = ComponentSummaries(g, 0, 1)
    bits, lst, ln, passes = cs.solve()
    assert passes == exp.passes and np.array_equal(bits, exp.bits) and np.array_equal(ln, exp.len)
    for f in range(ln.shape[0]):
        assert np.array_equal(lst[f, :ln[f]], exp.list[f, :ln[f]])
    assert cs.collectives == passes            # one all-reduce per pass; no gather at 1 rank
    cs.close()


def test_call_components_are_the_chains():
    from paper_2406_13881_b200.distributed import call_components, component_owner
    from paper_2406_13881_b200.gen.c5 import generate_c5
    g = generate_c5(seed=1, n_funcs=1200, depth=12, n_globals=64)
    comp = call_components(g)
    assert np.unique(comp).shape[0] == 100                     # 100 independent chains
    assert all(np.unique(comp[c * 12:(c + 1) * 12]).shape[0] == 1 for c in range(100))
    for world in (2, 4, 8):
        own = component_owner(g, world)
        cnt = np.bincount(own, minlength=world)
        assert cnt.max() - cnt.min() <= 24
        for c in range(100):                                     # whole chains per rank
            assert np.unique(own[c * 12:(c + 1) * 12]).shape[0] == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _component_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import _cg_cpu
    from paper_2406_13881_b200.distributed import ComponentSummaries
    from paper_2406_13881_b200.gen.c5 import generate_c5
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = generate_c5(seed=3, n_funcs=480, depth=12, n_globals=64, p_back=0.25)
    cs = ComponentSummaries(g, rank, world, wave_impl=_cg_cpu.make_cpu_wave)
    bits, lst, ln, passes = cs.solve()
    q.put((rank, bits, lst, ln, passes, cs.collectives))
    dist.destroy_process_group()


def test_component_summaries_gloo_world2_equals_oracle():
    from paper_2406_13881_b200.gen.c5 import generate_c5
    from paper_2406_13881_b200.interproc import solve_call_graph
    g = generate_c5(seed=3, n_funcs=480, depth=12, n_globals=64, p_back=0.25)
    exp = solve_call_graph(g, runner=_oracle.summaries_runner)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_component_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, bits, lst, ln, passes, ncoll in res:
        assert passes == exp.passes
        assert np.array_equal(bits, exp.bits), rank
        assert np.array_equal(ln, exp.len)
        for f in range(ln.shape[0]):
            assert np.array_equal(lst[f, :ln[f]], exp.list[f, :ln[f]])
        assert ncoll == passes + 1              # per-pass flag + one final all-gather
