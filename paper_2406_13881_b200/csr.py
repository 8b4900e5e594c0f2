"""Host wrapper of kernels (a)+(b): the CSR data-flow fixpoint engine.

`CsrProblem` owns one device-resident problem (`dfx_csr`): predecessor CSR,
node kinds, read/write bitplanes, and the fixpoint / requirement planes the
kernels produce.  Build it from host arrays (`from_arrays`, an H2D copy
through the C ABI) or generate configuration C3 directly in HBM
(`generate_c3`).  No CPU fallback exists: a missing libdfx.so or CUDA device
raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi


class CsrIn(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("words", C.c_int32), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("node_kind", C.c_void_p),
                ("R", C.c_void_p), ("W", C.c_void_p), ("S", C.c_void_p)]


class C3Spec(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_nodes", C.c_int64), ("words", C.c_int32),
                ("w0", C.c_int32), ("n_scalar", C.c_int32)]


class CsrStats(C.Structure):
    _fields_ = [("rounds_h", C.c_int32), ("rounds_d", C.c_int32),
                ("evaluated", C.c_int64), ("rows_read", C.c_int64),
                ("rows_written", C.c_int64), ("solve_ms", C.c_float),
                ("kernel_ms", C.c_float), ("req_ms", C.c_float), ("n_masks", C.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class ReqOut(C.Structure):
    _fields_ = [("row_off", C.c_void_p), ("occ", C.c_void_p), ("masks", C.c_void_p),
                ("cap", C.c_int64), ("n_masks", C.c_int64), ("occ_words", C.c_int32)]


REQ_UPDATE_FROM, REQ_UPDATE_TO, REQ_FIRSTPRIVATE = 1, 2, 3

# list forms (include/dfx.h, csrc/acc.cu)
ACC_READ, ACC_WRITE = 1, 2
REQ_FP_FLAG = 0x8000


class AccIn(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("words", C.c_int32), ("nnz", C.c_int64),
                ("n_acc", C.c_int64), ("row_ptr", C.c_void_p), ("col", C.c_void_p),
                ("node_kind", C.c_void_p), ("acc_off", C.c_void_p), ("acc", C.c_void_p),
                ("S", C.c_void_p)]


class ReqListOut(C.Structure):
    _fields_ = [("row_off", C.c_void_p), ("vars", C.c_void_p), ("cap", C.c_int64),
                ("n_out", C.c_int64)]


@dataclass
class ReqList:
    """Kernel (b) output as per-node variable lists (include/dfx.h
    dfx_req_list): node n's entries are vars[row_off[n]:row_off[n+1]],
    transfer requirements ascending, then firstprivate captures (REQ_FP_FLAG)."""
    row_off: np.ndarray      # int64 [n+1]
    vars: np.ndarray         # uint16 [n_out]
    words: int

    @property
    def nbytes(self) -> int:
        return self.row_off.nbytes + self.vars.nbytes

    def to_planes(self):
        """Expand into dense (REQ, FP) planes [n, words]."""
        return lists_to_planes(self.row_off, self.vars, self.words, REQ_FP_FLAG)


def planes_to_acc(R: np.ndarray, W: np.ndarray):
    """Dense read/write planes [n, words] -> (acc_off int64 [n+1], acc uint16):
    per node, accessed variables ascending, entry = var | kind << 14."""
    n, words = R.shape
    rb = np.unpackbits(np.ascontiguousarray(R).view(np.uint8).reshape(n, words * 4), axis=1,
                       bitorder="little").astype(np.uint16)
    wb = np.unpackbits(np.ascontiguousarray(W).view(np.uint8).reshape(n, words * 4), axis=1,
                       bitorder="little").astype(np.uint16)
    k = rb * ACC_READ + wb * ACC_WRITE
    nodes, vars_ = np.nonzero(k)
    acc = (vars_.astype(np.uint16) | (k[nodes, vars_] << 14)).astype(np.uint16)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(nodes, minlength=n), out=off[1:])
    return off, acc


def lists_to_planes(off: np.ndarray, entries: np.ndarray, words: int, flag: int):
    """Per-node variable lists -> two dense planes [n, words]: entries without
    `flag` and entries with it (variable = low 14 bits)."""
    n = off.shape[0] - 1
    node = np.repeat(np.arange(n), np.diff(off))
    var = (entries & 0x3FFF).astype(np.int64)
    second = (entries & flag) != 0
    planes = []
    for sel in (~second, second):
        bits = np.zeros((n, words * 32), dtype=np.uint8)
        bits[node[sel], var[sel]] = 1
        planes.append(np.packbits(bits, axis=1, bitorder="little").view(np.uint32)
                      .reshape(n, words).copy())
    return planes[0], planes[1]


@dataclass
class ReqRows:
    """Kernel (b) output: sparse word-rows of insertion points (include/dfx.h)."""
    row_off: np.ndarray      # int64 [n+1]
    occ: np.ndarray          # uint32 [n, occ_words]
    masks: np.ndarray        # uint32 [n_masks]
    words: int

    @property
    def nbytes(self) -> int:
        return self.row_off.nbytes + self.occ.nbytes + self.masks.nbytes

    def to_planes(self):
        """Expand into dense (REQ, FP) planes [n, words]."""
        n = self.row_off.shape[0] - 1
        ow = self.occ.shape[1] // 2
        bits = np.unpackbits(self.occ.view(np.uint8).reshape(n, 2 * ow, 4), axis=2,
                             bitorder="little").reshape(n, 2, ow * 32)[:, :, : self.words]
        req = np.zeros((n, self.words), dtype=np.uint32)
        fp = np.zeros_like(req)
        # order inside a node: requirement words ascending, then firstprivate
        flat = np.concatenate([bits[:, 0, :], bits[:, 1, :]], axis=1).astype(bool)
        assert int(flat.sum()) == self.masks.shape[0]
        vals = np.zeros(flat.shape, dtype=np.uint32)
        vals[flat] = self.masks
        req[:] = vals[:, : self.words]
        fp[:] = vals[:, self.words:]
        return req, fp

    def records(self, kind: np.ndarray):
        """(node, word, kind, mask) records in stream order."""
        req, fp = self.to_planes()
        out = []
        for n in range(req.shape[0]):
            k = REQ_UPDATE_TO if kind[n] else REQ_UPDATE_FROM
            for w in np.nonzero(req[n])[0]:
                out.append((n, int(w), k, int(req[n, w])))
            for w in np.nonzero(fp[n])[0]:
                out.append((n, int(w), REQ_FIRSTPRIVATE, int(fp[n, w])))
        return out


def _setup(lib):
    for name in ("dfx_set_stream", "dfx_csr_create", "dfx_csr_generate_c3", "dfx_csr_destroy",
                 "dfx_csr_solve", "dfx_csr_requirements", "dfx_csr_download", "dfx_mfp_csr",
                 "dfx_csr_export", "dfx_csr_create_acc", "dfx_csr_requirements_list",
                 "dfx_csr_solve_async",
                 "dfx_csr_export_acc", "dfx_mfp_acc"):
        getattr(lib, name).restype = C.c_int
    lib.dfx_csr_nnz.restype = C.c_int64


@dataclass
class C3Config:
    """Configuration C3 (BASELINE.json configs[2]): 1M nodes x 4096 variables."""
    n_nodes: int = 1 << 20
    n_vars: int = 4096
    seed: int = 0
    w0: int = 0                   # first global word (V-sharding across GPUs)
    scalar_frac: float = 0.02     # 2% of variables are firstprivate-eligible scalars

    @property
    def words(self) -> int:
        return self.n_vars // 32

    @property
    def n_scalar(self) -> int:
        return int(round(self.scalar_frac * self.n_vars))


def c3_scalar_mask(cfg: C3Config) -> np.ndarray:
    """Scalar-variable mask of a C3 slab: variables [0, n_scalar) (global
    numbering) are the firstprivate-eligible scalars."""
    out = np.zeros(cfg.words, dtype=np.uint32)
    for w in range(cfg.words):
        lo = 32 * (cfg.w0 + w)
        if cfg.n_scalar >= lo + 32:
            out[w] = 0xFFFFFFFF
        elif cfg.n_scalar > lo:
            out[w] = (1 << (cfg.n_scalar - lo)) - 1
    return out


def _check_graph_shapes(n: int, words: int, row_ptr, col, kind, S, planes=()) -> None:
    """Host buffer shapes the C ABI trusts (it copies n+1 / nnz / n x words
    elements from these pointers); the graph's contents are validated on the
    device (acc.cu check_csr)."""
    if row_ptr.ndim != 1 or row_ptr.shape[0] != n + 1:
        raise ValueError("row_ptr must have n_nodes + 1 = %d entries" % (n + 1))
    nnz = int(row_ptr[-1]) if n >= 0 else 0
    if col.ndim != 1 or col.shape[0] < nnz:
        raise ValueError("col has %d entries, row_ptr[-1] = %d" % (col.shape[0], nnz))
    if kind.shape != (n,):
        raise ValueError("node_kind must have n_nodes = %d entries" % n)
    if S.shape != (words,):
        raise ValueError("S must have words = %d entries" % words)
    for P in planes:
        if P.shape != (n, words):
            raise ValueError("bitplanes must be (n_nodes, words) = (%d, %d)" % (n, words))


class CsrProblem:
    def __init__(self, eng: _abi.Engine, handle: C.c_void_p, n_nodes: int, words: int):
        self.eng = eng
        self.h = handle
        self.n_nodes = n_nodes
        self.words = words
        self.stats = CsrStats()

    # ---- construction -----------------------------------------------------
    @classmethod
    def generate_c3(cls, cfg: C3Config, eng: _abi.Engine | None = None) -> "CsrProblem":
        eng = eng or _abi.engine()
        _setup(eng.lib)
        spec = C3Spec(cfg.seed, cfg.n_nodes, cfg.words, cfg.w0, cfg.n_scalar)
        h = C.c_void_p()
        eng.check(eng.lib.dfx_csr_generate_c3(eng.h, C.byref(spec), C.byref(h)),
                  "dfx_csr_generate_c3")
        return cls(eng, h, cfg.n_nodes, cfg.words)

    @classmethod
    def from_arrays(cls, row_ptr, col, kind, R, W, S, eng: _abi.Engine | None = None) -> "CsrProblem":
        eng = eng or _abi.engine()
        _setup(eng.lib)
        n, words = R.shape
        arrs = [np.ascontiguousarray(a) for a in (row_ptr, col, kind, R, W, S)]
        row_ptr, col, kind, R, W, S = arrs
        assert row_ptr.dtype == np.int32 and col.dtype == np.int32 and kind.dtype == np.uint8
        assert R.dtype == np.uint32 and W.dtype == np.uint32 and S.dtype == np.uint32
        _check_graph_shapes(n, words, row_ptr, col, kind, S, (R, W))
        cin = CsrIn(n, words, int(row_ptr[-1]), *(a.ctypes.data for a in arrs))
        h = C.c_void_p()
        eng.check(eng.lib.dfx_csr_create(eng.h, C.byref(cin), C.byref(h)), "dfx_csr_create")
        return cls(eng, h, n, words)

    @classmethod
    def from_acc(cls, row_ptr, col, kind, acc_off, acc, S, words: int,
                 eng: _abi.Engine | None = None) -> "CsrProblem":
        """Build from access lists (dfx_csr_create_acc): H2D + expansion."""
        eng = eng or _abi.engine()
        _setup(eng.lib)
        cin, keep = _acc_in(row_ptr, col, kind, acc_off, acc, S, words)
        h = C.c_void_p()
        eng.check(eng.lib.dfx_csr_create_acc(eng.h, C.byref(cin), C.byref(h)),
                  "dfx_csr_create_acc")
        del keep
        return cls(eng, h, int(row_ptr.shape[0]) - 1, words)

    def close(self) -> None:
        if self.h:
            self.eng.lib.dfx_csr_destroy(self.eng.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- kernels -------------------------------------------------------------
    def solve(self, chunk_nodes: int = 0) -> CsrStats:
        self.eng.check(self.eng.lib.dfx_csr_solve(self.eng.h, self.h, C.c_int32(chunk_nodes),
                                                  C.byref(self.stats)), "dfx_csr_solve")
        return self.stats

    def requirements(self, capacity: int | None = None, alloc=np.empty) -> ReqRows:
        """Kernel (b): requirement planes + order-preserving compaction."""
        if capacity is None:
            self.eng.check(self.eng.lib.dfx_csr_requirements(self.eng.h, self.h, None,
                                                             C.byref(self.stats)),
                           "dfx_csr_requirements(count)")
            capacity = int(self.stats.n_masks)
        return _req_call(lambda o: self.eng.lib.dfx_csr_requirements(
            self.eng.h, self.h, C.byref(o), C.byref(self.stats)),
            self.eng, self.n_nodes, self.words, capacity, alloc, self.stats)

    def solve_async(self, chunk_nodes: int = 0) -> None:
        """Kernel (a) enqueued without host synchronisation (dfx_csr_solve_async)."""
        self.eng.check(self.eng.lib.dfx_csr_solve_async(self.eng.h, self.h, C.c_int32(chunk_nodes)),
                       "dfx_csr_solve_async")

    def requirements_list(self, capacity: int | None = None, alloc=np.empty) -> ReqList:
        """Kernel (b) as per-node variable lists (dfx_csr_requirements_list)."""
        if capacity is None:
            o = ReqListOut(None, None, 0, 0)
            self.eng.check(self.eng.lib.dfx_csr_requirements_list(
                self.eng.h, self.h, C.byref(o), C.byref(self.stats)), "requirements_list(count)")
            capacity = int(o.n_out)
        while True:
            row_off = alloc((self.n_nodes + 1,), np.int64)
            vars_ = alloc((max(1, capacity),), np.uint16)
            o = ReqListOut(row_off.ctypes.data, vars_.ctypes.data, vars_.shape[0], 0)
            rc = self.eng.lib.dfx_csr_requirements_list(self.eng.h, self.h, C.byref(o),
                                                        C.byref(self.stats))
            if rc == _abi.DFX_E_NOSPC:
                capacity = int(o.n_out)
                continue
            self.eng.check(rc, "dfx_csr_requirements_list")
            return ReqList(row_off, vars_[: o.n_out], self.words)

    def export_acc(self, alloc=np.empty):
        """D2H of the problem's accesses as lists (acc_off int64 [n+1], acc uint16)."""
        n_acc = C.c_int64()
        self.eng.check(self.eng.lib.dfx_csr_export_acc(self.eng.h, self.h, None, None, 0,
                                                       C.byref(n_acc)), "export_acc(count)")
        off = alloc((self.n_nodes + 1,), np.int64)
        acc = alloc((max(1, n_acc.value),), np.uint16)
        self.eng.check(self.eng.lib.dfx_csr_export_acc(
            self.eng.h, self.h, C.c_void_p(off.ctypes.data), C.c_void_p(acc.ctypes.data),
            C.c_int64(acc.shape[0]), C.byref(n_acc)), "dfx_csr_export_acc")
        return off, acc[: n_acc.value]

    def export_inputs(self, alloc=np.empty):
        """D2H of the inputs (row_ptr, col, kind, R, W); `alloc(shape, dtype)`
        lets callers supply pinned host memory."""
        nnz = int(self.eng.lib.dfx_csr_nnz(self.h))
        rp = alloc((self.n_nodes + 1,), np.int32)
        col = alloc((max(1, nnz),), np.int32)
        kind = alloc((self.n_nodes,), np.uint8)
        R = alloc((self.n_nodes, self.words), np.uint32)
        W = alloc((self.n_nodes, self.words), np.uint32)
        p = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
        self.eng.check(self.eng.lib.dfx_csr_export(self.eng.h, self.h, p(rp), p(col), p(kind),
                                                   p(R), p(W)), "dfx_csr_export")
        return rp, col[:nnz], kind, R, W

    def download(self, out_h=True, out_d=True, req=False):
        shape = (self.n_nodes, self.words)
        oh = np.empty(shape, dtype=np.uint32) if out_h else None
        od = np.empty(shape, dtype=np.uint32) if out_d else None
        rq = np.empty(shape, dtype=np.uint32) if req else None
        p = lambda a: C.c_void_p(a.ctypes.data) if a is not None else None  # noqa: E731
        self.eng.check(self.eng.lib.dfx_csr_download(self.eng.h, self.h, p(oh), p(od), p(rq)),
                       "dfx_csr_download")
        return oh, od, rq


def _req_call(call, eng, n_nodes, words, capacity, alloc, stats) -> ReqRows:
    ow = 2 * ((words + 31) // 32)
    while True:
        row_off = alloc((n_nodes + 1,), np.int64)
        occ = alloc((n_nodes, ow), np.uint32)
        masks = alloc((max(1, capacity),), np.uint32)
        o = ReqOut(row_off.ctypes.data, occ.ctypes.data, masks.ctypes.data,
                   masks.shape[0], 0, 0)
        rc = call(o)
        if rc == _abi.DFX_E_NOSPC:
            capacity = int(o.n_masks)
            continue
        eng.check(rc, "requirements")
        return ReqRows(row_off, occ, masks[: o.n_masks], words)


class MfpSession:
    """Reference-facing all-in-one host-buffer path (`dfx_mfp_csr`): H2D of
    the inputs, kernels (a)+(b), D2H of the compacted requirement rows.
    Output host buffers are reused across calls (optionally pinned)."""

    def __init__(self, eng: _abi.Engine | None = None, alloc=np.empty):
        self.eng = eng or _abi.engine()
        _setup(self.eng.lib)
        self.alloc = alloc
        self.capacity = 0
        self.stats = CsrStats()
        self._bufs = None

    def run(self, row_ptr, col, kind, R, W, S) -> ReqRows:
        n, words = R.shape
        arrs = [np.ascontiguousarray(a) for a in (row_ptr, col, kind, R, W, S)]
        _check_graph_shapes(n, words, arrs[0], arrs[1], arrs[2], arrs[5], (arrs[3], arrs[4]))
        cin = CsrIn(n, words, int(arrs[0][-1]), *(a.ctypes.data for a in arrs))
        if self.capacity == 0:
            self.capacity = max(1024, n * words // 2)
        ow = 2 * ((words + 31) // 32)
        while True:
            if self._bufs is None or self._bufs[2].shape[0] < self.capacity \
                    or self._bufs[0].shape[0] != n + 1:
                self._bufs = (self.alloc((n + 1,), np.int64), self.alloc((n, ow), np.uint32),
                              self.alloc((self.capacity,), np.uint32))
            row_off, occ, masks = self._bufs
            o = ReqOut(row_off.ctypes.data, occ.ctypes.data, masks.ctypes.data,
                       masks.shape[0], 0, 0)
            rc = self.eng.lib.dfx_mfp_csr(self.eng.h, C.byref(cin), C.byref(o),
                                          C.byref(self.stats))
            if rc == _abi.DFX_E_NOSPC:
                self.capacity = int(o.n_masks)
                continue
            self.eng.check(rc, "dfx_mfp_csr")
            return ReqRows(row_off, occ, masks[: o.n_masks], words)


def _acc_in(row_ptr, col, kind, acc_off, acc, S, words):
    arrs = [np.ascontiguousarray(a) for a in (row_ptr, col, kind, acc_off, acc, S)]
    row_ptr, col, kind, acc_off, acc, S = arrs
    assert row_ptr.dtype == np.int32 and col.dtype == np.int32 and kind.dtype == np.uint8
    assert acc_off.dtype == np.int64 and acc.dtype == np.uint16 and S.dtype == np.uint32
    n = int(row_ptr.shape[0]) - 1
    _check_graph_shapes(n, words, row_ptr, col, kind, S)
    if acc_off.shape != (n + 1,) or acc.shape[0] < int(acc_off[-1]):
        raise ValueError("acc_off must have n_nodes + 1 entries and acc at least acc_off[-1]")
    cin = AccIn(n, words, int(row_ptr[-1]), int(acc_off[-1]),
                *(a.ctypes.data for a in arrs))
    return cin, arrs


# ---- byte-coded lists (include/dfx.h "B8") ----------------------------------
B8_REQ, B8_FP = 1, 2


class Acc8In(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("words", C.c_int32), ("nnz", C.c_int64),
                ("n_bytes", C.c_int64), ("row_ptr", C.c_void_p), ("col", C.c_void_p),
                ("node_kind", C.c_void_p), ("byte_off", C.c_void_p), ("bytes", C.c_void_p),
                ("S", C.c_void_p)]


class Req8Out(C.Structure):
    _fields_ = [("row_off", C.c_void_p), ("bytes", C.c_void_p), ("cap", C.c_int64),
                ("n_out", C.c_int64)]


def _b8_encode(node, var, kind, n, restart=None):
    """Entries (node, var, kind) grouped by node in ascending var order
    (`restart`: True where a new ascending run starts inside a node) -> (byte
    offsets int32 [n+1], bytes uint8).  b = kind << 6 | d, d == 63 continues."""
    var = var.astype(np.int64)
    first = np.ones(var.shape[0], dtype=bool)
    first[1:] = node[1:] != node[:-1]
    if restart is not None:
        first |= restart
    prev = np.empty_like(var)
    prev[0:1] = -1
    prev[1:] = var[:-1]
    prev[first] = -1
    delta = var - prev - 1
    if (delta < 0).any():
        raise ValueError("entries must ascend by variable within a node")
    nb = delta // 63 + 1                                  # bytes per entry
    end = np.cumsum(nb)
    out = np.repeat((kind.astype(np.uint8) << 6) | 63, nb).astype(np.uint8)
    if end.shape[0]:
        out[end - 1] = ((kind.astype(np.int64) << 6) | (delta % 63)).astype(np.uint8)
    per_node = np.bincount(node, weights=nb, minlength=n).astype(np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(per_node, out=off[1:])
    if off[-1] > 0x7FFFFFFF:
        raise ValueError("byte-coded lists are limited to 2^31 - 1 bytes")
    return off.astype(np.int32), out


def acc_to_b8(acc_off, acc):
    """uint16 access lists (var | kind << 14, ascending per node) -> B8."""
    n = int(acc_off.shape[0]) - 1
    node = np.repeat(np.arange(n), np.diff(acc_off))
    a = acc.astype(np.int64)
    return _b8_encode(node, a & 0x3FFF, a >> 14, n)


def b8_decode(off, b, restart_on_kind: bool = False):
    """B8 lists -> (node int64, var int64, kind uint8) per entry, in order.
    `restart_on_kind`: requirement lists, whose firstprivate entries restart
    the ascending run (access lists mix kinds within one run)."""
    b = np.asarray(b, dtype=np.uint8)
    n = int(off.shape[0]) - 1
    node_b = np.repeat(np.arange(n), np.diff(off.astype(np.int64)))
    d = (b & 63).astype(np.int64)
    kind = (b >> 6).astype(np.uint8)
    term = d < 63
    # a run restarts at each node and where the kind changes inside a node
    start = np.ones(b.shape[0], dtype=bool)
    start[1:] = node_b[1:] != node_b[:-1]
    if restart_on_kind:
        start[1:] |= kind[1:] != kind[:-1]
    contrib = d + term
    cs = np.cumsum(contrib)
    base = np.maximum.accumulate(np.where(start, cs - contrib, 0))
    var = cs - base - 1
    return node_b[term], var[term], kind[term]


def req8_to_lists(off, b, words):
    """B8 requirement lists -> (row_off int64, vars uint16) in the uint16 list
    form (`REQ_FP_FLAG` on firstprivate entries)."""
    node, var, kind = b8_decode(off, b, restart_on_kind=True)
    n = int(off.shape[0]) - 1
    vals = (var | np.where(kind == B8_FP, REQ_FP_FLAG, 0)).astype(np.uint16)
    row = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(node, minlength=n), out=row[1:])
    return ReqList(row, vals, words)


@dataclass
class Req8List:
    row_off: np.ndarray      # int32 [n+1]
    bytes: np.ndarray        # uint8 [n_out]
    words: int

    @property
    def nbytes(self) -> int:
        return self.row_off.nbytes + self.bytes.nbytes

    def to_lists(self) -> ReqList:
        return req8_to_lists(self.row_off, self.bytes, self.words)


class Acc8Session:
    """`AccSession` on byte-coded lists (`dfx_mfp_acc8`): about 1.2 bytes per
    access in and per planned transfer out instead of 2, the host link being
    what bounds the call.  Output buffers are reused (optionally pinned)."""

    def __init__(self, eng: _abi.Engine | None = None, alloc=np.empty):
        self.eng = eng or _abi.engine()
        _setup(self.eng.lib)
        self.eng.lib.dfx_mfp_acc8.restype = C.c_int
        self.alloc = alloc
        self.capacity = 0
        self.stats = CsrStats()
        self._bufs = None

    def run(self, row_ptr, col, kind, byte_off, b, S, words: int) -> Req8List:
        arrs = [np.ascontiguousarray(a) for a in (row_ptr, col, kind, byte_off, b, S)]
        row_ptr, col, kind, byte_off, b, S = arrs
        assert row_ptr.dtype == np.int32 and col.dtype == np.int32 and kind.dtype == np.uint8
        assert byte_off.dtype == np.int32 and b.dtype == np.uint8 and S.dtype == np.uint32
        n = int(row_ptr.shape[0]) - 1
        _check_graph_shapes(n, words, row_ptr, col, kind, S)
        if byte_off.shape != (n + 1,) or b.shape[0] < int(byte_off[-1]):
            raise ValueError("byte_off must have n_nodes + 1 entries and bytes at least byte_off[-1]")
        cin = Acc8In(n, words, int(row_ptr[-1]), int(byte_off[-1]), *(a.ctypes.data for a in arrs))
        if self.capacity == 0:
            self.capacity = max(4096, int(byte_off[-1]))
        while True:
            if self._bufs is None or self._bufs[1].shape[0] < self.capacity \
                    or self._bufs[0].shape[0] != n + 1:
                self._bufs = (self.alloc((n + 1,), np.int32), self.alloc((self.capacity,), np.uint8))
            row_off, out = self._bufs
            o = Req8Out(row_off.ctypes.data, out.ctypes.data, out.shape[0], 0)
            rc = self.eng.lib.dfx_mfp_acc8(self.eng.h, C.byref(cin), C.byref(o), C.byref(self.stats))
            if rc == _abi.DFX_E_NOSPC:
                self.capacity = int(o.n_out)
                continue
            self.eng.check(rc, "dfx_mfp_acc8")
            return Req8List(row_off, out[: o.n_out], words)


class AccSession:
    """Reference-facing all-in-one host-buffer path on lists (`dfx_mfp_acc`):
    H2D of the CSR and the per-node access lists, expansion, kernels (a)+(b),
    D2H of the per-node requirement lists.  Output buffers are reused across
    calls (optionally pinned)."""

    def __init__(self, eng: _abi.Engine | None = None, alloc=np.empty):
        self.eng = eng or _abi.engine()
        _setup(self.eng.lib)
        self.alloc = alloc
        self.capacity = 0
        self.stats = CsrStats()
        self._bufs = None

    def run(self, row_ptr, col, kind, acc_off, acc, S, words: int) -> ReqList:
        cin, keep = _acc_in(row_ptr, col, kind, acc_off, acc, S, words)
        n = int(cin.n_nodes)
        if self.capacity == 0:
            self.capacity = max(1024, int(cin.n_acc))
        while True:
            if self._bufs is None or self._bufs[1].shape[0] < self.capacity \
                    or self._bufs[0].shape[0] != n + 1:
                self._bufs = (self.alloc((n + 1,), np.int64),
                              self.alloc((self.capacity,), np.uint16))
            row_off, vars_ = self._bufs
            o = ReqListOut(row_off.ctypes.data, vars_.ctypes.data, vars_.shape[0], 0)
            rc = self.eng.lib.dfx_mfp_acc(self.eng.h, C.byref(cin), C.byref(o),
                                          C.byref(self.stats))
            if rc == _abi.DFX_E_NOSPC:
                self.capacity = int(o.n_out)
                continue
            self.eng.check(rc, "dfx_mfp_acc")
            del keep
            return ReqList(row_off, vars_[: o.n_out], words)


def mfp_csr(row_ptr, col, kind, R, W, S, eng: _abi.Engine | None = None):
    """One-shot all-in-one call; returns (ReqRows, stats)."""
    sess = MfpSession(eng)
    rows = sess.run(row_ptr, col, kind, R, W, S)
    return rows, sess.stats
