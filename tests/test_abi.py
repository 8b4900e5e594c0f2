"""CPU: the C-ABI library loads and exports every symbol include/dfx.h declares."""
import ctypes
import pathlib
import re

import pytest

from paper_2406_13881_b200 import _abi

ROOT = pathlib.Path(__file__).resolve().parent.parent


def declared_symbols():
    syms = set()
    for h in (ROOT / "include").glob("*.h"):
        for m in re.finditer(r"^\s*(?:int|const char \*|void)\s*\**\s*(dfx_\w+)\s*\(",
                             h.read_text(), re.M):
            syms.add(m.group(1))
    return sorted(syms)


def test_header_declares_entry_points():
    syms = declared_symbols()
    for need in ("dfx_open", "dfx_close", "dfx_last_error", "dfx_abi_version",
                 "dfx_replay_batch"):
        assert need in syms


@pytest.mark.skipif(not _abi.LIB_PATH.exists(), reason="libdfx.so not built")
def test_library_exports_all_declared_symbols():
    lib = ctypes.CDLL(str(_abi.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    lib.dfx_abi_version.restype = ctypes.c_int
    assert lib.dfx_abi_version() == _abi.ABI_VERSION


def test_graph_shape_checks_on_host():
    """Short host arrays are rejected before the C ABI copies from them."""
    import numpy as np
    import pytest
    from paper_2406_13881_b200.csr import _check_graph_shapes
    rp = np.array([0, 1, 2], dtype=np.int32)
    col = np.array([0, 1], dtype=np.int32)
    kind = np.zeros(2, dtype=np.uint8)
    S = np.zeros(4, dtype=np.uint32)
    R = np.zeros((2, 4), dtype=np.uint32)
    _check_graph_shapes(2, 4, rp, col, kind, S, (R, R))
    with pytest.raises(ValueError):
        _check_graph_shapes(2, 4, rp, col[:1], kind, S)
    with pytest.raises(ValueError):
        _check_graph_shapes(3, 4, rp, col, kind, S)
    with pytest.raises(ValueError):
        _check_graph_shapes(2, 4, rp, col, kind, S, (R[:1],))
    with pytest.raises(ValueError):
        _check_graph_shapes(2, 4, rp, col, kind, S[:2])
