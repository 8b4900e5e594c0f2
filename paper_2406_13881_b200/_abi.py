"""ctypes mirror of include/dfx.h and the loader for libdfx.so.

The product path loads only `libdfx.so` (built in-tree by `make -C
paper_2406_13881_b200/csrc`); there is no CPU fallback: if the library or a
CUDA device is missing, `engine()` raises.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import threading

import numpy as np

PKG_DIR = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libdfx.so"

ABI_VERSION = 1


class FnDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "op_off", "n_ops", "var_off", "n_vars", "stmt_off", "n_stmts",
        "site_off", "arm_off", "region_begin_start", "n_slots",
        "max_loop_depth", "max_br_depth", "max_arms", "flags")] + [("reserved", C.c_int32 * 2)]


FN_DESC_DTYPE = np.dtype([(n, np.int32) for n in (
    "op_off", "n_ops", "var_off", "n_vars", "stmt_off", "n_stmts",
    "site_off", "arm_off", "region_begin_start", "n_slots",
    "max_loop_depth", "max_br_depth", "max_arms", "flags", "r1", "r2")])
assert FN_DESC_DTYPE.itemsize == C.sizeof(FnDesc) == 64


class ReplayIn(C.Structure):
    _fields_ = [
        ("n_funcs", C.c_int32),
        ("fns", C.c_void_p),
        ("ops", C.c_void_p),
        ("var_flags", C.c_void_p),
        ("stmt_span", C.c_void_p),
        ("sites", C.c_void_p),
        ("arms", C.c_void_p),
        ("n_ops", C.c_int64), ("n_vars", C.c_int64), ("n_stmts", C.c_int64),
        ("n_sites", C.c_int64), ("n_arms", C.c_int64),
    ]


EVENT_DTYPE = np.dtype([("key", np.uint64), ("fn", np.int32), ("var", np.int32),
                        ("node", np.int32), ("kind", np.uint8), ("pos", np.uint8),
                        ("pad", np.uint16)])
assert EVENT_DTYPE.itemsize == 24


class ReplayOut(C.Structure):
    _fields_ = [
        ("events", C.c_void_p),
        ("event_cap", C.c_int64),
        ("n_events", C.c_int64),
        ("var_out", C.c_void_p),
        ("kernel_ms", C.c_float),
    ]


# event kinds / positions / output bits (include/dfx.h)
EV_UPDATE_FROM, EV_UPDATE_TO, EV_FIRSTPRIVATE, EV_SUPPRESS = 1, 2, 3, 4
EV_ERR_DATAMAP, EV_ERR_BRACES_LOOP, EV_ERR_BRACES_ARM, EV_ERR_DECL, EV_ERR_ENGINE = \
    16, 17, 18, 19, 20
POS_BEFORE, POS_AFTER, POS_BODY_END, POS_KERNEL = 0, 1, 2, 3
OUT_PRESENCE, OUT_TO, OUT_FROM, OUT_H, OUT_D = 1, 2, 4, 8, 16
FN_NO_ERR_SITES = 1          # dfx_fn_desc.flags (include/dfx.h)
# opcodes (include/dfx.h; lower.py emits them)
(OP_END, OP_HR, OP_HW, OP_DR, OP_DW, OP_BR_BEGIN, OP_ARM_FORK, OP_ARM_CLOSE, OP_ARM_PASSIVE,
 OP_BR_END, OP_LOOP_BEGIN, OP_LOOP_END, OP_ERR) = range(13)

DFX_OK, DFX_E_ARG, DFX_E_CUDA, DFX_E_NOSPC, DFX_E_LIMIT = 0, -1, -2, -3, -4


def ptr(a: np.ndarray | None) -> int | None:
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class EngineError(RuntimeError):
    pass


class Engine:
    """One `dfx_handle` on one CUDA device."""

    def __init__(self, lib: C.CDLL, device: int = 0):
        self.lib = lib
        self.device = device
        h = C.c_void_p()
        rc = lib.dfx_open(device, C.byref(h))
        if rc != 0:
            raise EngineError("dfx_open(%d) failed: %s" % (device, self.last_error()))
        self.h = h

    def last_error(self) -> str:
        s = self.lib.dfx_last_error()
        return s.decode() if s else ""

    def check(self, rc: int, what: str) -> int:
        if rc not in (DFX_OK, DFX_E_NOSPC):
            raise EngineError("%s failed (%d): %s" % (what, rc, self.last_error()))
        return rc

    def close(self):
        if self.h:
            self.lib.dfx_close(self.h)
            self.h = None


_lock = threading.Lock()
_engines: dict[int, Engine] = {}
_lib: C.CDLL | None = None


def load_lib(path: str | os.PathLike | None = None) -> C.CDLL:
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = pathlib.Path(path) if path else LIB_PATH
    if not p.exists():
        raise EngineError(
            "libdfx.so not built (%s); run `python -c 'import __graft_entry__ as g; "
            "g.build()'` or `make -C paper_2406_13881_b200/csrc`" % p)
    lib = C.CDLL(str(p))
    lib.dfx_last_error.restype = C.c_char_p
    lib.dfx_abi_version.restype = C.c_int
    for name in ("dfx_open", "dfx_close", "dfx_replay_batch", "dfx_replay_batch_packed"):
        getattr(lib, name).restype = C.c_int
    if lib.dfx_abi_version() != ABI_VERSION:
        raise EngineError("libdfx ABI %d != %d" % (lib.dfx_abi_version(), ABI_VERSION))
    if path is None:
        _lib = lib
    return lib


def engine(device: int | None = None) -> Engine:
    """The process-wide engine for `device` (default: $DFX_DEVICE or 0)."""
    if device is None:
        device = int(os.environ.get("DFX_DEVICE", "0"))
    with _lock:
        e = _engines.get(device)
        if e is None:
            e = Engine(load_lib(), device)
            _engines[device] = e
        return e
