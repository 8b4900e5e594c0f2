"""Multi-GPU drivers: one process per GPU, `torch.distributed` for plumbing.

* Kernel (c) across GPUs, component-sharded (`ComponentSummaries`, the
  product path): functions are owned by ranks whole call-graph component at
  a time (LPT on component cost), so during the passes no rank reads a row
  another rank writes.  Per pass each rank runs its own functions' waves,
  then ONE all-reduce(MAX) of the changed flag (the reference's global
  termination test, `interproc.py:105-143`); after the last pass ONE
  all-gather of the owned rows.  On GPUs all of it runs inside
  `dfx_summaries_sharded` over the handle's NCCL communicator
  (`dfx_comm_init`); the same protocol runs on CPU tensors with gloo for the
  world-size-2 tests.
* Kernel (c) across GPUs, wave-sharded (`ShardedSummaries`, for a call graph
  that is one giant component): each wave of the reference's
  pass schedule is split round-robin over the ranks; a rank rebuilds its
  share of the wave's functions on its GPU (`dfx_cg_wave`), then the ranks
  all-gather the rebuilt summary rows (bits + insertion order + length) --
  the only data exchanged, over NCCL/NVLink on GPUs (north star: "only
  function summaries are exchanged, by NCCL allgather").  A pass ends with a
  MAX all-reduce of the changed flag (the reference's termination test).
* Kernels (a)+(b) and E1 shard without communication (variables and
  functions are independent, SURVEY F3 / SPEC.md:345): see `bench.py`
  (`C3Config.w0`, `batch.lpt_shards`).

`wave_impl` is pluggable so the exchange protocol is tested on CPU with the
gloo backend (tests/test_distributed.py) against a CPU wave restatement.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _abi


class CgTables(C.Structure):
    _fields_ = [("bits", C.c_void_p), ("list", C.c_void_p), ("len", C.c_void_p)]


def call_components(g) -> np.ndarray:
    """Connected components of the call graph (union-find over the calls to
    defined functions, SRC_CALL rows): component id per function."""
    from .interproc import SRC_CALL
    nf = g.init_bits.shape[0]
    parent = np.arange(nf, dtype=np.int64)

    def find(x):
        r = x
        while parent[r] != r:
            r = parent[r]
        while parent[x] != r:
            parent[x], x = r, parent[x]
        return r
    src = np.asarray(g.src).reshape(-1, 4)
    for f in range(nf):
        for k in range(int(g.src_off[f]), int(g.src_off[f + 1])):
            if (int(src[k, 0]) & 0xFF) == SRC_CALL:
                a, b = find(f), find(int(src[k, 1]))
                if a != b:
                    parent[max(a, b)] = min(a, b)
    return np.array([find(f) for f in range(nf)], dtype=np.int64)


def component_owner(g, world: int) -> np.ndarray:
    """Owner rank of every function: whole components, longest processing
    time first on cost = functions + call-graph sources of the component."""
    from .batch import lpt_shards
    comp = call_components(g)
    nf = comp.shape[0]
    ids, inv = np.unique(comp, return_inverse=True)
    srcs = np.diff(np.asarray(g.src_off, dtype=np.int64))
    cost = np.bincount(inv, weights=1.0 + srcs, minlength=ids.shape[0])
    owner = np.zeros(nf, dtype=np.int32)
    for r, cs in enumerate(lpt_shards(cost, world)):
        owner[np.isin(inv, cs)] = r
    return owner


class ComponentSummaries:
    """summarize_all across ranks, one collective per pass (see the module
    docstring).  GPU: `dfx_summaries_sharded` on a handle whose NCCL
    communicator this object initialises (rank 0's unique id is broadcast
    through `torch.distributed`).  `wave_impl` selects the same protocol on
    CPU tensors with `torch.distributed` collectives (gloo tests)."""

    def __init__(self, g, rank: int = 0, world: int = 1, eng: _abi.Engine | None = None,
                 max_passes: int | None = None, wave_impl=None, owner=None):
        self.g = g
        self.rank, self.world = rank, world
        self.owner = component_owner(g, world) if owner is None else np.asarray(owner, np.int32)
        self.max_passes = max_passes or max(16, g.init_bits.shape[0] + 1)
        self.collectives = 0
        self.wave_impl = wave_impl
        if wave_impl is not None:
            return
        from .interproc import cg_struct
        self.eng = eng or _abi.engine()
        lib = self.eng.lib
        for n in ("dfx_comm_unique_id", "dfx_comm_init", "dfx_comm_destroy",
                  "dfx_summaries_sharded"):
            getattr(lib, n).restype = C.c_int
        uid = (C.c_char * 128)()
        if rank == 0:
            self.eng.check(lib.dfx_comm_unique_id(uid), "dfx_comm_unique_id")
        if world > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0)
            uid = (C.c_char * 128).from_buffer_copy(obj[0])
        self.eng.check(lib.dfx_comm_init(self.eng.h, uid, C.c_int32(world), C.c_int32(rank)),
                       "dfx_comm_init")
        self._keep: list = []
        self.cin = cg_struct(g, self._keep, self.max_passes)

    def local_schedule(self):
        """This rank's waves: its own functions, in the reference order."""
        g = self.g
        woff, wfns = [0], []
        for w in range(g.wave_off.shape[0] - 1):
            seg = g.wave_fns[g.wave_off[w]:g.wave_off[w + 1]]
            wfns.extend(int(f) for f in seg if self.owner[f] == self.rank)
            if len(wfns) > woff[-1]:
                woff.append(len(wfns))
        return np.array(woff, dtype=np.int32), np.array(wfns, dtype=np.int32)

    def solve(self):
        """Returns (bits uint8 [nf, ns], list int16 [nf, ns], len int32, passes)."""
        if self.wave_impl is not None:
            return self._solve_protocol()
        from .interproc import CgOut
        bits = np.zeros(self.g.init_bits.shape, dtype=np.uint8)
        lst = np.zeros(self.g.init_list.shape, dtype=np.int16)
        ln = np.zeros(self.g.init_bits.shape[0], dtype=np.int32)
        out = CgOut(bits.ctypes.data, lst.ctypes.data, ln.ctypes.data, 0, 0, 0.0)
        ncol = C.c_int32(0)
        own = np.ascontiguousarray(self.owner, dtype=np.int32)
        self.eng.check(self.eng.lib.dfx_summaries_sharded(
            self.eng.h, C.byref(self.cin), C.c_void_p(own.ctypes.data), C.byref(out),
            C.byref(ncol)), "dfx_summaries_sharded")
        self.kernel_ms = float(out.kernel_ms)
        self.collectives = int(ncol.value)
        return bits, lst, ln, int(out.passes)

    def _solve_protocol(self):
        """The same protocol on CPU tensors (wave_impl(prev, cur, w) rebuilds
        the listed functions of local wave w)."""
        import dataclasses
        woff, wfns = self.local_schedule()
        g, nf = self.g, self.g.init_bits.shape[0]
        local = dataclasses.replace(g, wave_off=woff, wave_fns=wfns)
        st = ShardedSummaries(local, 0, 1, device="cpu", wave_impl=lambda *a: 0,
                              max_passes=self.max_passes)
        st.wave_impl = self.wave_impl(st)
        st._reset()
        prev, passes = 0, 0
        while passes < self.max_passes:
            passes += 1
            cur = prev ^ 1
            changed = 0
            for w in range(woff.shape[0] - 1):
                changed |= st.wave_impl(prev, cur, w)
            flag = torch.tensor([changed], dtype=torch.int32)
            if self.world > 1:
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            self.collectives += 1
            prev = cur
            if not int(flag.item()):
                break
        t = st.t[prev]
        if self.world > 1:
            mine = torch.from_numpy(np.nonzero(self.owner == self.rank)[0].astype(np.int64))
            per = int(np.bincount(self.owner, minlength=self.world).max())
            rowb = st.nsp + 2 * st.nsp + 4
            send = torch.zeros((per, rowb), dtype=torch.uint8)
            k = mine.numel()
            send[:k, :st.nsp] = t["bits"].index_select(0, mine)
            send[:k, st.nsp:3 * st.nsp] = t["list"].index_select(0, mine).view(torch.uint8)
            send[:k, 3 * st.nsp:] = t["len"].index_select(0, mine).view(torch.uint8).view(-1, 4)
            recv = [torch.empty_like(send) for _ in range(self.world)]
            dist.all_gather(recv, send)
            self.collectives += 1
            for r in range(self.world):
                if r == self.rank:
                    continue
                ids = torch.from_numpy(np.nonzero(self.owner == r)[0].astype(np.int64))
                rows = recv[r][:ids.numel()]
                t["bits"].index_copy_(0, ids, rows[:, :st.nsp].contiguous())
                t["list"].index_copy_(0, ids, rows[:, st.nsp:3 * st.nsp].contiguous().view(torch.int16))
                t["len"].index_copy_(0, ids, rows[:, 3 * st.nsp:].contiguous().view(torch.int32).view(-1))
        return (t["bits"][:, :st.ns].numpy().copy(), t["list"][:, :st.ns].numpy().copy(),
                t["len"].numpy().copy(), passes)

    def close(self):
        if self.wave_impl is None and getattr(self, "eng", None) is not None:
            self.eng.lib.dfx_comm_destroy(self.eng.h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedSummaries:
    def __init__(self, g, rank: int = 0, world: int = 1, device: str | torch.device = "cuda",
                 wave_impl=None, max_passes: int | None = None):
        self.g = g
        self.rank, self.world = rank, world
        self.device = torch.device(device)
        nf, ns = g.init_bits.shape
        self.nf, self.ns = nf, ns
        self.nsp = ((ns + 31) // 32) * 32
        self.max_passes = max_passes or max(16, nf + 1)
        self.t = []
        for k in range(2):
            bits = torch.zeros((nf, self.nsp), dtype=torch.uint8, device=self.device)
            lst = torch.zeros((nf, self.nsp), dtype=torch.int16, device=self.device)
            ln = torch.zeros(nf, dtype=torch.int32, device=self.device)
            self.t.append({"bits": bits, "list": lst, "len": ln})
        self.wave_impl = wave_impl or self._gpu_wave
        self.cg = None
        self.launches = 0
        if wave_impl is None:
            from .interproc import cg_struct
            self.eng = _abi.engine(self.device.index or 0)
            lib = self.eng.lib
            for n in ("dfx_cg_create", "dfx_cg_destroy", "dfx_cg_wave"):
                getattr(lib, n).restype = C.c_int
            lib.dfx_cg_nsp.restype = C.c_int32
            self._keep: list = []
            cin = cg_struct(g, self._keep, self.max_passes)
            h = C.c_void_p()
            self.eng.check(lib.dfx_cg_create(self.eng.h, C.byref(cin), C.byref(h)), "dfx_cg_create")
            self.cg = h
            assert lib.dfx_cg_nsp(h) == self.nsp

    def _tables(self, k) -> CgTables:
        t = self.t[k]
        return CgTables(t["bits"].data_ptr(), t["list"].data_ptr(), t["len"].data_ptr())

    def _gpu_wave(self, prev: int, cur: int, w: int) -> int:
        changed = C.c_int32(0)
        pt, ct = self._tables(prev), self._tables(cur)
        self.eng.check(self.eng.lib.dfx_cg_wave(self.eng.h, self.cg, C.byref(pt), C.byref(ct),
                                                C.c_int32(w), C.c_int32(self.rank),
                                                C.c_int32(self.world), C.byref(changed)),
                       "dfx_cg_wave")
        return int(changed.value)

    def _exchange(self, cur: int, w: int) -> None:
        """All-gather the rows each rank rebuilt in wave `w` into every rank's
        `cur` tables."""
        if self.world == 1:
            return
        lo, hi = int(self.g.wave_off[w]), int(self.g.wave_off[w + 1])
        fns = torch.from_numpy(self.g.wave_fns[lo:hi].astype(np.int64)).to(self.device)
        m = (hi - lo + self.world - 1) // self.world
        if m == 0:
            return
        t = self.t[cur]
        rowb = self.nsp + 2 * self.nsp + 4
        mine = fns[self.rank::self.world]
        send = torch.zeros((m, rowb), dtype=torch.uint8, device=self.device)
        if mine.numel():
            send[:mine.numel(), :self.nsp] = t["bits"].index_select(0, mine)
            send[:mine.numel(), self.nsp:3 * self.nsp] = \
                t["list"].index_select(0, mine).view(torch.uint8)
            send[:mine.numel(), 3 * self.nsp:] = \
                t["len"].index_select(0, mine).view(torch.uint8).view(-1, 4)
        recv = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(recv, send)
        for r in range(self.world):
            ids = fns[r::self.world]
            k = ids.numel()
            if k == 0 or r == self.rank:
                continue
            rows = recv[r][:k]
            t["bits"].index_copy_(0, ids, rows[:, :self.nsp].contiguous())
            t["list"].index_copy_(0, ids, rows[:, self.nsp:3 * self.nsp].contiguous().view(torch.int16))
            t["len"].index_copy_(0, ids, rows[:, 3 * self.nsp:].contiguous().view(torch.int32).view(-1))
        if self.device.type == "cuda":
            # the next wave runs on the engine's stream: the scattered rows
            # (written on torch's stream) must have landed
            torch.cuda.current_stream(self.device).synchronize()

    def _reset(self) -> None:
        """Pass-0 summaries into table 0 (every solve starts from them)."""
        ns = self.ns
        self.t[0]["bits"][:, :ns] = torch.from_numpy(self.g.init_bits)
        self.t[0]["list"][:, :ns] = torch.from_numpy(self.g.init_list)
        self.t[0]["len"][:] = torch.from_numpy(self.g.init_len)

    def solve(self):
        """Returns (bits uint8 [nf, ns], list int16 [nf, ns], len int32, passes)."""
        self._reset()
        prev, passes = 0, 0
        n_waves = self.g.wave_off.shape[0] - 1
        while passes < self.max_passes:
            passes += 1
            cur = prev ^ 1
            changed = 0
            for w in range(n_waves):
                changed |= self.wave_impl(prev, cur, w)
                self.launches += 1
                self._exchange(cur, w)
            if self.world > 1:
                flag = torch.tensor([changed], dtype=torch.int32, device=self.device)
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)
                changed = int(flag.item())
            prev = cur
            if not changed:
                break
        t = self.t[prev]
        return (t["bits"][:, :self.ns].cpu().numpy(), t["list"][:, :self.ns].cpu().numpy(),
                t["len"].cpu().numpy(), passes)

    def close(self):
        if self.cg is not None:
            self.eng.lib.dfx_cg_destroy(self.eng.h, self.cg)
            self.cg = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PeerSummaries:
    """Kernel (c) across GPUs with the exchange fused into the producing
    kernel (`dfx_cgp_*`, csrc/summ.cu `cg_wave_peer_kernel`): the kernel that
    rebuilds a function's summary row stores it into every rank's tables over
    peer memory (NVLink P2P through CUDA IPC), and a wave ends on
    system-scope arrival counters -- no all-gather.  The IPC handles of the
    ranks' exchange blocks are swapped once, through `torch.distributed`."""

    def __init__(self, g, rank: int = 0, world: int = 1, eng: _abi.Engine | None = None,
                 max_passes: int | None = None):
        from .interproc import cg_struct
        self.g = g
        self.rank, self.world = rank, world
        self.eng = eng or _abi.engine()
        lib = self.eng.lib
        for n in ("dfx_cgp_create", "dfx_cgp_handle", "dfx_cgp_connect", "dfx_cgp_solve",
                  "dfx_cgp_destroy"):
            getattr(lib, n).restype = C.c_int
        self._keep: list = []
        self.cin = cg_struct(g, self._keep, max_passes or max(16, g.n_funcs + 1))
        h = C.c_void_p()
        self.eng.check(lib.dfx_cgp_create(self.eng.h, C.byref(self.cin), C.c_int32(world),
                                          C.c_int32(rank), C.byref(h)), "dfx_cgp_create")
        self.h = h
        mine = (C.c_char * 64)()
        self.eng.check(lib.dfx_cgp_handle(h, mine), "dfx_cgp_handle")
        handles = [bytes(mine)]
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, bytes(mine))
        allh = (C.c_char * (64 * world)).from_buffer_copy(b"".join(handles))
        self.eng.check(lib.dfx_cgp_connect(self.eng.h, h, allh), "dfx_cgp_connect")

    def solve(self):
        """Returns (bits uint8 [nf, ns], list int16 [nf, ns], len int32, passes)."""
        from .interproc import CgOut
        bits = np.zeros(self.g.init_bits.shape, dtype=np.uint8)
        lst = np.zeros(self.g.init_list.shape, dtype=np.int16)
        ln = np.zeros(self.g.n_funcs, dtype=np.int32)
        out = CgOut(bits.ctypes.data, lst.ctypes.data, ln.ctypes.data, 0, 0, 0.0)
        # the peer protocol (include/dfx.h): no rank may start solve k+1 (and
        # write pass-1 rows into a peer's tables) before every rank has
        # returned from solve k
        if self.world > 1:
            dist.barrier()
        self.eng.check(self.eng.lib.dfx_cgp_solve(self.eng.h, self.h, C.byref(out)), "dfx_cgp_solve")
        if self.world > 1:
            dist.barrier()
        self.kernel_ms = float(out.kernel_ms)
        return bits, lst, ln, int(out.passes)

    def close(self):
        if getattr(self, "h", None):
            self.eng.lib.dfx_cgp_destroy(self.eng.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
