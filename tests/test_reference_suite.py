"""Drop-in proof: the reference's OWN test suite (pkg/tests, 145 tests; copied
unmodified into oracle/_ref/tests by oracle/copy_ref.py) run with ``deftsim``
bound to this package (tests/ref_shim).  Everything on the hot path -- the
knapsack solver, partitioning, profiles, the DeFT state machine and baselines,
the preserver and its feedback loop, acceptance criteria C1-C4, C6, C9-C11 --
must pass; only the simulator engine, trace reconstruction and the CLI
(test_simulator.py, test_trace.py, test_cli.py and the acceptance criteria
that call them) are out of scope, and every skip must say so."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = ROOT / "oracle" / "_ref" / "tests"
IN_SCOPE = ["test_knapsack.py", "test_partition.py", "test_profiles.py", "test_scheduler.py",
            "test_preserver.py", "test_acceptance.py"]
OUT_OF_SCOPE = ["test_simulator.py", "test_trace.py", "test_cli.py"]

pytestmark = pytest.mark.gpu      # the solver runs on the GPU (no CPU fallback)


def test_reference_suite_against_this_package(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not REF_TESTS.is_dir():
        pytest.skip("oracle/_ref/tests missing (build() copies the reference)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "ref_shim"), str(ROOT)])
    cmd = [sys.executable, "-m", "pytest", "-q", "-rs", "-p", "no:cacheprovider",
           "--rootdir", str(REF_TESTS), "-o", "addopts="] + \
          [str(REF_TESTS / f) for f in IN_SCOPE]
    r = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True,
                       timeout=1500)
    out = r.stdout + r.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "reference_suite.log").write_text(out)
    m = re.search(r"(\d+) passed", out)
    passed = int(m.group(1)) if m else 0
    failed = re.search(r"(\d+) failed", out)
    assert r.returncode == 0 and not failed, out[-4000:]
    # every skip names the out-of-scope subsystem
    for line in out.splitlines():
        if line.startswith("SKIPPED"):
            assert "outside the B200 hot path" in line, line
    skipped = re.search(r"(\d+) skipped", out)
    skipped = int(skipped.group(1)) if skipped else 0
    # 91 in-scope tests: C5 (trace), C7/C8 (simulator), C12 (CLI) skip, the rest pass
    assert passed + skipped == 91 and skipped <= 4, out[-2000:]
