"""The hardware report runner end to end on one GPU: the
reference's experiment-file schema (cli.py:100-143) run through
DeftDataParallel on a small MLP -- profile measured on the device, every
scheme the executor runs (nonsequential with its hardware-timed candidate
probe), every sweep point -- written in the reference's report schema
(cli.py:294-391, pinned on the reference-written files in tests/golden/reports)."""
import csv
import json

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import GOLDEN  # noqa: E402
from paper_2503_16815_b200 import experiment as X  # noqa: E402

REP = GOLDEN / "reports"


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _mlp():
    torch.manual_seed(0)
    return torch.nn.Sequential(
        torch.nn.Linear(256, 512), torch.nn.ReLU(), torch.nn.Linear(512, 512), torch.nn.ReLU(),
        torch.nn.Linear(512, 512), torch.nn.ReLU(), torch.nn.Linear(512, 64)).cuda()


def _loss(module, batch):
    return torch.nn.functional.mse_loss(module(batch[0]), batch[1])


def test_hw_experiment_reports(tmp_path):
    data = json.loads((REP / "experiment_vgg.json").read_text())
    data.update(iterations=8, partition={"partition_size": 120_000, "mu": 1.65,
                                         "comm_startup_us": 150})
    data["sweeps"] = {"bandwidth_scale": [1.0, 0.5]}
    cfg = X.experiment_config_from_dict(data, REP)
    g = torch.Generator(device="cuda").manual_seed(1)
    batch = (torch.randn(32, 256, device="cuda", generator=g),
             torch.randn(32, 64, device="cuda", generator=g))
    seen = []
    bundle = X.run_hw_experiment(cfg, _mlp, batch, _loss, warmup=3,
                                 executor_kwargs={"autocast_dtype": None, "lr": 0.01,
                                                  "momentum": 0.9},
                                 log=seen.append)
    assert not bundle.skipped, bundle.skipped
    assert len(bundle.runs) == 2 * 5 == len(seen)             # 2 sweep points x 5 schemes
    assert {r.scheme for r in bundle.runs} == set(cfg.schemes)
    files = X.emit_reports(bundle, tmp_path)
    names = {f.name for f in files}
    assert {"summary.json", "comparison.csv"} <= names
    got = json.loads((tmp_path / "summary.json").read_text())
    want = json.loads((REP / "summary.json").read_text())
    assert set(got) == set(want)
    assert got["config_hash"] == X.config_hash(cfg, 0)
    # every run: exactly the reference's keys, plus this runner's "hardware" block
    # (world, buckets, links, compute-only step, placement) that only a run on GPUs has
    assert {set(r) - {"hardware"} == set(want["runs"][0]) for r in got["runs"]} == {True}
    assert all({"world", "buckets", "compute_only_ms_per_step"} <= set(r["hardware"])
               for r in got["runs"])
    for r in got["runs"]:
        assert r["report"]["total_time_us"] > 0
        if r["scheme"].startswith("deft"):
            assert r["preserver"] is not None                  # the walk is configured
    with open(tmp_path / "comparison.csv") as f, open(REP / "comparison.csv") as g2:
        assert next(csv.reader(f)) == next(csv.reader(g2))     # the reference's header
