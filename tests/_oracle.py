"""Test-side loader for the CPU oracle library (oracle/liboracle.so).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg use this module.
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

ROOT = pathlib.Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "liboracle.so"

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_LIB.exists():
            subprocess.run(["make", "-C", str(ORACLE_DIR)], check=True,
                           stdout=subprocess.DEVNULL)
        _lib = C.CDLL(str(ORACLE_LIB))
        _lib.oracle_replay_batch.restype = C.c_int
    return _lib


def replay_runner(rin, rout) -> int:
    return lib().oracle_replay_batch(C.byref(rin), C.byref(rout))
