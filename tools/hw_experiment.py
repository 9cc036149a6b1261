"""Run a reference experiment file on the B200s; write the reference's report files.

torchrun --nproc-per-node N tools/hw_experiment.py \
    [--config tests/golden/reports/experiment_vgg.json] [--out reports_hw/] \
    [--model vgg19] [--batch 64] [--iterations 60]

Reads the same experiment JSON as the reference's `deftsim run` (cli.py:100-143),
runs every (scheme, sweep point) through DeftDataParallel on real GPUs
(paper_2503_16815_b200/experiment.py explains what each field means on
hardware) and writes summary.json / comparison.csv / plotdata/*.csv in the
reference's schema (cli.py:294-391).  The model defaults to the profile's name
(vgg19.json -> VGG-19, random init, synthetic batch of 64 per GPU).
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_16815_b200 import experiment as X  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=str(ROOT / "tests/golden/reports/experiment_vgg.json"))
    ap.add_argument("--out", default=str(ROOT / "gpurun_out/hw_reports"))
    ap.add_argument("--model", default=None, choices=[None, "resnet101", "vgg19", "gpt2"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--iterations", type=int, default=None)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    cfg = X.load_experiment_config(args.config)
    if args.iterations:
        from dataclasses import replace
        cfg = replace(cfg, iterations=args.iterations)
    model_name = args.model or Path(cfg.profile_path).stem
    batch_size = args.batch or (16 if model_name == "gpt2" else 64)
    local = int(os.environ.get("LOCAL_RANK", 0))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    world = int(os.environ.get("WORLD_SIZE", 1))
    dist = torch.distributed
    if world > 1:
        bench.init_quiet(dist, device)
    rank = dist.get_rank() if world > 1 else 0
    batch = bench.make_batch(model_name, batch_size, device, seed=1234 + rank)
    loss_fn = bench.loss_fn_for(model_name)

    def compute_only(model):
        ms, _ = bench.compute_only_step_ms(model, batch, loss_fn, 20, 5, world, dist, device)
        return ms

    def log(rec):
        if rank == 0:
            print(json.dumps({"run_id": rec.run_id, **rec.report.summary_dict(),
                              **rec.hardware}), file=sys.stderr, flush=True)

    bundle = X.run_hw_experiment(
        cfg, lambda: bench.build_model(model_name, device), batch, loss_fn, seed=args.seed,
        executor_kwargs={"autocast_dtype": None if model_name == "gpt2" else torch.bfloat16,
                         "lr": 0.1, "momentum": 0.9},
        log=log, compute_only_ms=compute_only)
    if rank == 0:
        files = X.emit_reports(bundle, args.out)
        print(json.dumps({"written": [str(f) for f in files], "runs": len(bundle.runs),
                          "skipped": bundle.skipped}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
