import gzip
import json
import os
import sys
from pathlib import Path

import pytest

# loopback worlds (tests/test_gpu_loopback.py) want one hardware queue per
# stream; only read when the CUDA context is created
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# ... and no lazily loaded kernel (its first launch waits for the whole device)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")
    config.addinivalue_line("markers", "slow: long-running")


def read_jsonl_gz(name):
    with gzip.open(GOLDEN / name, "rt") as f:
        return [json.loads(line) for line in f]


def golden_schedule_text(entry):
    with gzip.open(GOLDEN / entry["file"], "rt") as f:
        return f.read()


@pytest.fixture(scope="session")
def golden_inputs():
    return json.loads((GOLDEN / "inputs.json").read_text())


@pytest.fixture(scope="session")
def golden_index():
    return json.loads((GOLDEN / "schedules.json").read_text())


def uniform_buckets(n, comm_us=900, fwd_total=3600, bwd_total=7200):
    """tests/conftest.py:65-87 of the reference, as dict buckets."""
    fwd = [fwd_total // n] * n
    bwd = [bwd_total // n] * n
    for i in range(fwd_total - sum(fwd)):
        fwd[i] += 1
    for i in range(bwd_total - sum(bwd)):
        bwd[i] += 1
    return [{"id": i + 1, "param_count": 1000, "forward_us": fwd[i], "backward_us": bwd[i],
             "comm_fast_us": comm_us} for i in range(n)]


def spec_inputs(entry, inputs):
    """(raw profile dict, cluster dict, partition cfg or None, comm factor, mult, iterations)."""
    spec = entry["spec"]
    if "uniform" in spec:
        prof = {"name": f"uniform{spec['uniform']}", "batch_size": 256, "learning_rate": 0.01,
                "buckets": uniform_buckets(spec["uniform"]), "notes": {}}
    else:
        prof = inputs["profiles"][spec["profile"]]
    cluster = inputs["clusters"][spec["cluster"]]
    mult = 1.0
    for _ in range(spec.get("mult_steps", 0)):
        mult *= 1.1
    # comm factor applied with ModelProfile.scaled_comm (profiles.py:134-152):
    # 1/bw_scale for the reference's bandwidth sweep points, or an explicit comm_scale
    factor = spec["comm_scale"] if "comm_scale" in spec else 1.0 / spec.get("bw_scale", 1.0)
    return prof, cluster, spec.get("partition"), factor, mult, entry["iterations"]
