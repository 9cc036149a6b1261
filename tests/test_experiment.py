"""Report-harness parity: the hardware experiment runner
reads the reference's experiment JSON and writes its summary.json /
comparison.csv / plotdata schema.  Pinned on files the reference itself wrote
for its fixture experiment (tests/golden/make_report_golden.py)."""
import json
from pathlib import Path

import pytest

from conftest import GOLDEN
import paper_2503_16815_b200 as D
from paper_2503_16815_b200 import experiment as X
from paper_2503_16815_b200 import knapsack as K
from oracle import deft_oracle as O

REP = GOLDEN / "reports"


@pytest.fixture(scope="module")
def golden_summary():
    return json.loads((REP / "summary.json").read_text())


@pytest.fixture(scope="module")
def cfg():
    return X.load_experiment_config(REP / "experiment_vgg.json")


def test_config_and_hash_match_reference(cfg, golden_summary):
    assert cfg.schemes == ("wfbp", "priority", "nonsequential", "deft", "deft_single_link")
    assert cfg.iterations == 60 and cfg.partition.comm_startup_us == 150
    assert X.config_hash(cfg, 0) == golden_summary["config_hash"]
    labels = [p.label() for p in X.sweep_points(cfg)]
    assert sorted(labels) == sorted({r["run_id"].split("__")[1] for r in golden_summary["runs"]})


def test_schema_errors(tmp_path):
    with pytest.raises(D.SchemaError, match="schemes"):
        X.experiment_config_from_dict({"profile": "x.json", "iterations": 5}, tmp_path)
    with pytest.raises(D.SchemaError, match="unknown schemes"):
        X.experiment_config_from_dict({"profile": "x.json", "schemes": ["teleport"],
                                       "iterations": 5}, tmp_path)
    with pytest.raises(D.SchemaError, match="non-empty"):
        X.experiment_config_from_dict({"profile": "x.json", "schemes": ["wfbp"],
                                       "iterations": 5, "sweeps": {"bandwidth_scale": []}},
                                      tmp_path)
    bad = tmp_path / "bad.json"
    bad.write_text("{")
    with pytest.raises(D.SchemaError, match="invalid JSON"):
        X.load_experiment_config(bad)


def _bundle_from(summary):
    runs = []
    for r in summary["runs"]:
        sp = r["sweep_point"]
        rep = r["report"]
        report = X.RunReport(rep["scheme"], rep["profile"], rep["iterations"],
                             rep["total_time_us"], rep["mean_iteration_time_us"],
                             rep["bubble_time_us"], rep["bubble_ratio"],
                             rep["updates_performed"], rep["throughput_samples_per_s"])
        point = X.SweepPoint(sp["bandwidth_scale"], sp["partition_size"], sp["gpu_count"])
        runs.append(X.RunRecord(r["scheme"], point, report, r["scheme"], r["preserver"]))
    return X.ReportBundle(summary["config_hash"], runs, summary["iterations"])


def test_report_files_byte_identical(tmp_path, golden_summary):
    """Given the same per-run numbers, the writer reproduces the reference's
    files byte for byte (comparison table, speedups, plot data)."""
    files = X.emit_reports(_bundle_from(golden_summary), tmp_path)
    assert {f.name for f in files} == {"summary.json", "comparison.csv",
                                       "speedup_vs_bandwidth.csv",
                                       "speedup_vs_partition_size.csv"}
    assert (tmp_path / "summary.json").read_text() == (REP / "summary.json").read_text()
    assert (tmp_path / "comparison.csv").read_text() == (REP / "comparison.csv").read_text()
    for name in ("speedup_vs_bandwidth.csv", "speedup_vs_partition_size.csv"):
        assert (tmp_path / "plotdata" / name).read_text() == (REP / name).read_text()


def test_compare_errors():
    r = X.RunReport("deft", "m", 10, 100, 10.0, 0, 0.0, 9, 1.0)
    with pytest.raises(D.ComparisonError):
        X.compare({})
    with pytest.raises(D.ComparisonError, match="baseline"):
        X.compare({"deft": r})
    with pytest.raises(D.ComparisonError, match="iteration counts"):
        X.compare({"deft": r, "wfbp": X.RunReport("wfbp", "m", 5, 1, 1.0, 0, 0.0, 5, 1.0)})


def test_from_measurement():
    r = X.RunReport.from_measurement("deft", "vgg19", 60, total_ms=900.0,
                                     compute_only_ms_per_step=14.0, batch_size=64,
                                     updates_performed=58)
    assert r.total_time_us == 900_000 and r.bubble_time_us == 60_000
    assert r.mean_iteration_time_us == 15_000.0
    assert abs(r.bubble_ratio - 60_000 / 900_000) < 1e-15
    assert abs(r.throughput_samples_per_s - 60 * 64 / 0.9) < 1e-9
    s = X.RunReport.from_measurement("wfbp", "vgg19", 10, 100.0, 11.0, 64, 10)
    assert s.bubble_time_us == 0          # never negative


def test_preserver_verdicts_match_reference(cfg, golden_summary, golden_inputs):
    """The verdict block the hardware runner attaches to delayed schemes equals
    the reference's for the same schedule (fixture profile, every sweep point)."""
    prof = D.profile_from_dict(golden_inputs["profiles"]["vgg19"])
    cluster = D.cluster_from_dict(golden_inputs["clusters"]["dual"])
    by_id = {r["run_id"]: r for r in golden_summary["runs"]}
    checked = 0
    with K.subset_sum_backend(O.subset_sum_c_batch):
        for point in X.sweep_points(cfg):
            p_prof = X.point_profile(prof, point, None)
            part_cfg = cfg.partition
            if point.partition_size is not None:
                from dataclasses import replace
                part_cfg = replace(part_cfg, partition_size=point.partition_size)
            for scheme, single in (("deft", False), ("deft_single_link", True)):
                sched = D.deft_schedule(p_prof, cluster, part_cfg, cfg.iterations,
                                        single_link=single, engine="host")
                got = X.preserver_verdict(sched, cfg.walk)
                assert got == by_id[f"{scheme}__{point.label()}"]["preserver"], \
                    (scheme, point.label())
                checked += 1
    assert checked == 8
