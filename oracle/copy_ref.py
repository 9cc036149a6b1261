"""ORACLE recipe (test infrastructure only): copy the reference package into
oracle/_ref/ so that it travels to the GPU box with the gpurun snapshot.

The reference (deftsim) is pure Python (click + numpy), so "building" it is a
copy of its sources -- never into the repository's history: oracle/_ref/ is
git-ignored (but not gpurun-ignored).  Copied:

  /root/reference/pkg/src/deftsim  -> oracle/_ref/deftsim    (the reference itself)
  /root/reference/pkg/tests        -> oracle/_ref/tests      (its own test suite)
  /root/reference/pkg/fixtures     -> oracle/_ref/fixtures   (its fixture profiles)

Used by: bench.py's reference arm and solver block (the reference's CPU path
timed on the GPU host), tests/test_reference_suite.py (the reference's own
tests run against paper_2503_16815_b200 aliased as ``deftsim``) and the golden
generators.  Nothing in the product package imports it.
"""
from __future__ import annotations

import shutil
import sys
from pathlib import Path

SRC = Path("/root/reference/pkg")
DST = Path(__file__).resolve().parent / "_ref"


def copy(src: Path = SRC, dst: Path = DST) -> bool:
    if not (src / "src" / "deftsim").is_dir():
        return False          # on the GPU box: use the copy that travelled
    ign = shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache", ".hypothesis")
    for a, b in (("src/deftsim", "deftsim"), ("tests", "tests"), ("fixtures", "fixtures")):
        if (dst / b).exists():
            shutil.rmtree(dst / b)
        shutil.copytree(src / a, dst / b, ignore=ign)
    (dst / "SOURCE").write_text(f"copied from {src} by oracle/copy_ref.py\n")
    return True


if __name__ == "__main__":
    print("copied" if copy() else "reference not present; kept", DST)
    sys.exit(0)
