"""ORACLE -- test infrastructure only: import the UNMODIFIED reference package
(deftsim) from the copy oracle/copy_ref.py put in oracle/_ref/.  Callers: the
tests, bench.py's reference arm / solver block and the golden generators."""
from __future__ import annotations

import importlib
import sys
from pathlib import Path

REF = Path(__file__).resolve().parent / "_ref"


def available() -> bool:
    return (REF / "deftsim" / "__init__.py").exists()


def deftsim():
    """The reference package, imported from oracle/_ref (raises if absent)."""
    if not available():
        raise ImportError(f"{REF}/deftsim is missing: run oracle/copy_ref.py (build())")
    mod = sys.modules.get("deftsim")
    if mod is not None and Path(mod.__file__).resolve().parent == (REF / "deftsim").resolve():
        return mod
    if mod is not None:
        raise ImportError("another module named deftsim is already imported")
    sys.path.insert(0, str(REF))
    try:
        return importlib.import_module("deftsim")
    finally:
        sys.path.remove(str(REF))
