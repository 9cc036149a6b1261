"""Golden report files for the report-harness parity.

Runs the UNMODIFIED reference's experiment pipeline (cli.py:205-391:
run_experiment -> emit_reports) on its own fixture experiment
(pkg/fixtures/experiment_vgg.json) and keeps what the B200 report writer must
reproduce: summary.json, comparison.csv and plotdata/*.csv.  The timeline /
Chrome-trace files are not kept (simulator output, out of scope).

Usage (only in the build container; never on the GPU box):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_report_golden.py
"""
from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_FIX = Path("/root/reference/pkg/fixtures")
OUT = Path(__file__).resolve().parent / "reports"

sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from deftsim.cli import emit_reports, load_experiment_config, run_experiment  # noqa: E402


def main():
    OUT.mkdir(exist_ok=True)
    cfg = load_experiment_config(REF_FIX / "experiment_vgg.json")
    bundle = run_experiment(cfg, seed=0)
    with tempfile.TemporaryDirectory() as tmp:
        emit_reports(bundle, tmp)
        tmp = Path(tmp)
        shutil.copy(tmp / "summary.json", OUT / "summary.json")
        shutil.copy(tmp / "comparison.csv", OUT / "comparison.csv")
        for p in sorted((tmp / "plotdata").glob("*.csv")):
            shutil.copy(p, OUT / p.name)
    exp = json.loads((REF_FIX / "experiment_vgg.json").read_text())
    (OUT / "experiment_vgg.json").write_text(json.dumps(exp, indent=2, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
