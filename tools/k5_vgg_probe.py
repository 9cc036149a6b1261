"""Where the persistent scheduler kernel's wall time goes for one deft_schedule
(the VGG-19 outlier of the solver block): kernel ms vs host decode ms, per fixture.

python tools/k5_vgg_probe.py
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2503_16815_b200 as D  # noqa: E402
from paper_2503_16815_b200 import _native, gpu_scheduler  # noqa: E402
from paper_2503_16815_b200.scheduler import DeftScheduler, _prepare  # noqa: E402


def main():
    inputs = json.loads((ROOT / "tests" / "golden" / "inputs.json").read_text())
    cl = D.cluster_from_dict(inputs["clusters"]["dual"])
    cfg = D.PartitionConfig(6_500_000, mu=1.65)
    solver = _native.subset_sum_solver()
    for rep in range(2):
        for name in ("resnet101", "vgg19", "gpt2"):
            part = _prepare(D.profile_from_dict(inputs["profiles"][name]), cfg)
            sched = DeftScheduler(part, cl, 1.0)
            k0 = solver.kernel_ms
            t0 = time.perf_counter()
            lazy = gpu_scheduler.run_schedules_lazy(part, cl, [1.0], 200, [sched])
            t1 = time.perf_counter()
            dec = lazy[0].decisions() if lazy[0] is not None else None
            t2 = time.perf_counter()
            print(json.dumps({"rep": rep, "profile": name, "buckets": part.n_buckets,
                              "kernel_ms": round(solver.kernel_ms - k0, 3),
                              "launch_wall_ms": round((t1 - t0) * 1e3, 3),
                              "decode_ms": round((t2 - t1) * 1e3, 3),
                              "supported": lazy[0] is not None,
                              "decisions": len(dec) if dec else 0}), flush=True)


if __name__ == "__main__":
    main()
