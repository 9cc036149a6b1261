"""Solver benchmark: the DeFT scheduler's knapsack path on the B200 vs the CPU.

python tools/solver_bench.py [--quick]

Per fixture configuration (reference pkg/fixtures profiles, dual-link cluster):
  * feedback_loop (200 iterations, up to 10 retries) through the product path
    (GPU subset-sum kernel, speculative lock-step retries), wall time;
  * the same decision streams from the CPU oracle port (oracle/, C DP), wall time,
    1 core -- the reference itself (pure Python) is not on the GPU box; its
    times measured in the build container are in BASELINE.md (8.4-31.6 s);
  * DP kernel time (CUDA events inside deft_solver_solve) and its algorithmic
    bytes (sum over placeable items of 2*ceil((cap'+1)/8)).
Also the SURVEY 8d grid (n in {10, 25, 48, 551} x cap in {2.5e5, 1e6, 1e7}, w ~ U[1, cap/n],
seed 0) single-problem and 256-per-launch, and 1024 random problems (n=48, cap 1e6) per launch.
"""
import argparse
import json
import math
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2503_16815_b200 as D  # noqa: E402
from paper_2503_16815_b200 import _native  # noqa: E402
from oracle import deft_oracle as O  # noqa: E402


def alg_bytes(problems):
    tot = 0
    for ws, cap in problems:
        q = 1
        if cap > 10_000_000:
            q = math.ceil(cap / 10_000_000)
            cap //= q
        row = 2 * ((cap + 1 + 7) // 8)
        tot += sum(row for w in ws if math.ceil(w / q) <= cap)
    return tot


class Counting:
    def __init__(self, solver):
        self.solver = solver
        self.bytes = 0

    def __call__(self, problems):
        self.bytes += alg_bytes(problems)
        return self.solver.solve(problems)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    inputs = json.loads((ROOT / "tests" / "golden" / "inputs.json").read_text())
    walk = D.WalkParams.from_dict(inputs["walk"])
    cl_d = inputs["clusters"]["dual"]
    cluster = D.cluster_from_dict(cl_d)
    solver = _native.subset_sum_solver()
    solver.solve([([3, 5, 7], 9)])  # warm the context
    configs = [("resnet101", 1.0), ("vgg19", 1.0), ("gpt2", 1.0), ("resnet101", 0.25),
               ("vgg19", 0.25), ("gpt2", 0.25)]
    if args.quick:
        configs = configs[:2]
    rows = []
    for name, bw in configs:
        prof = D.profile_from_dict(inputs["profiles"][name])
        if bw != 1.0:
            prof = prof.scaled_comm(1.0 / bw)
        cfg = D.PartitionConfig(6_500_000, mu=1.65)
        # K5: every attempt in one persistent scheduler kernel
        from paper_2503_16815_b200 import gpu_scheduler
        gpu_scheduler.run_schedules_lazy(D.partition_buckets(prof, cfg), cluster, [1.0], 4)
        k0 = solver.kernel_ms
        t0 = time.perf_counter()
        sched_k, verdict_k = D.feedback_loop(prof, cluster, cfg, walk, iterations=200,
                                             engine="kernel")
        t_k5 = time.perf_counter() - t0
        k5_ms = solver.kernel_ms - k0
        # host state machine, knapsacks batched on the GPU
        counting = Counting(solver)
        k0, ms0, calls0 = solver.kernel_ms, solver.kernel_ms, solver.calls
        with D.knapsack.subset_sum_backend(counting):
            t0 = time.perf_counter()
            sched, verdict = D.feedback_loop(prof, cluster, cfg, walk, iterations=200,
                                             engine="host")
            t_gpu = time.perf_counter() - t0
        kms = solver.kernel_ms - k0
        calls = solver.calls - calls0
        assert sched_k.jsonl_lines() == sched.jsonl_lines()
        # CPU oracle port: the same attempts, sequentially, C DP on 1 core
        b = O.scaled_comm(inputs["profiles"][name]["buckets"], 1.0 / bw) if bw != 1.0 else \
            inputs["profiles"][name]["buckets"]
        part = O.partition(b, sum(x["forward_us"] for x in b), 6_500_000, 1.65)
        ratios = [l["speed_ratio_to_fast"] for l in cl_d["links"]]
        names = [l["name"] for l in cl_d["links"]]
        t0 = time.perf_counter()
        m = 1.0
        for a in range(verdict.retries + 1):
            dec = O.schedule(part, ratios, names, 200, m)
            m *= 1.1
        t_cpu = time.perf_counter() - t0
        assert O.jsonl(dec) == "".join(l + "\n" for l in sched.jsonl_lines())
        rows.append({"config": f"{name} dual bw x{bw}", "buckets": len(part),
                     "retries": verdict.retries, "preserved": verdict.preserved,
                     "feedback_loop_k5_s": round(t_k5, 4), "k5_kernel_ms": round(k5_ms, 3),
                     "feedback_loop_host_engine_s": round(t_gpu, 4),
                     "oracle_cpu_s": round(t_cpu, 4),
                     "dp_launch_calls": calls, "dp_kernel_ms_total": round(kms, 3),
                     "dp_alg_bytes": counting.bytes,
                     "dp_achieved_gbs": round(counting.bytes / (kms / 1e3) / 1e9, 1) if kms else None})
        print(json.dumps(rows[-1]), flush=True)
    # SURVEY 8d solver microbench grid: w ~ U[1, cap/n], n x cap, seed 0; one problem
    # per call (latency) and 256 per launch (throughput), vs the C oracle on 1 core
    rng = random.Random(0)
    for n in (10, 25, 48, 551):
        for cap in (250_000, 1_000_000, 10_000_000):
            probs = [([rng.randint(1, max(1, cap // n)) for _ in range(n)], cap)
                     for _ in range(256)]
            assert solver.solve(probs[:4]) == O.subset_sum_c_batch(probs[:4])
            k0 = solver.kernel_ms
            t0 = time.perf_counter()
            for pr in probs[:16]:
                solver.solve([pr])
            t_single = (time.perf_counter() - t0) / 16
            k_single = (solver.kernel_ms - k0) / 16
            k0 = solver.kernel_ms
            solver.solve(probs)
            k_batch = solver.kernel_ms - k0
            t0 = time.perf_counter()
            O.subset_sum_c_batch(probs[:8])
            t_cpu = (time.perf_counter() - t0) / 8
            nb = alg_bytes(probs)
            print(json.dumps({"config": f"grid n={n} cap={cap}", "single_wall_ms":
                              round(t_single * 1e3, 3), "single_kernel_ms": round(k_single, 4),
                              "batch256_kernel_ms": round(k_batch, 3),
                              "batch256_alg_gbs": round(nb / (k_batch / 1e3) / 1e9, 1),
                              "oracle_cpu_ms_per_problem": round(t_cpu * 1e3, 3)}), flush=True)
    # batched throughput: many independent problems per launch
    rng = random.Random(0)
    probs = [([rng.randint(1, 40_000) for _ in range(48)], 1_000_000) for _ in range(1024)]
    solver.solve(probs[:8])
    k0 = solver.kernel_ms
    t0 = time.perf_counter()
    solver.solve(probs)
    t = time.perf_counter() - t0
    kms = solver.kernel_ms - k0
    nb = alg_bytes(probs)
    t0 = time.perf_counter()
    O.subset_sum_c_batch(probs[:64])
    t_cpu = (time.perf_counter() - t0) * 16
    out = {"config": "batched 1024 x (n=48, cap=1e6)", "dp_kernel_ms": round(kms, 3),
           "wall_ms": round(t * 1e3, 2), "dp_alg_bytes": nb,
           "dp_achieved_gbs": round(nb / (kms / 1e3) / 1e9, 1),
           "oracle_cpu_ms_1core_est": round(t_cpu * 1e3, 1)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
