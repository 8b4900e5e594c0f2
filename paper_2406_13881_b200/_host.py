"""Locate the host application (`dartomp`) whose analysis this engine replaces.

The engine is a drop-in for `dartomp.dataflow.analyze_function` and
`dartomp.interproc.summarize_all`; the front end (lexer, parser, AST-CFG,
access classification) and the directive emitter stay the host package's own.
`dartomp` is resolved from the normal import path first, then from
`$DFX_DARTOMP_PATH`, then from the repo-local install under `baseline/_ref`
(the offline `pip install --target` of the reference package).
"""
from __future__ import annotations

import importlib
import os
import pathlib
import sys

REPO_ROOT = pathlib.Path(__file__).resolve().parent.parent


def import_dartomp():
    try:
        return importlib.import_module("dartomp")
    except ImportError:
        pass
    cands = []
    if os.environ.get("DFX_DARTOMP_PATH"):
        cands.append(pathlib.Path(os.environ["DFX_DARTOMP_PATH"]))
    cands.append(REPO_ROOT / "baseline" / "_ref")
    for c in cands:
        if (c / "dartomp" / "__init__.py").exists():
            if str(c) not in sys.path:
                sys.path.append(str(c))
            return importlib.import_module("dartomp")
    raise ImportError(
        "dartomp (the host front end) is not importable; install it or set "
        "DFX_DARTOMP_PATH to a directory containing the dartomp package")


def have_dartomp() -> bool:
    try:
        import_dartomp()
        return True
    except ImportError:
        return False
