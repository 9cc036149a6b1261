"""GPU timeline of steady-state training steps (CUPTI via torch.profiler).

torchrun --nproc-per-node N tools/trace_step.py [--model vgg19] [--batch 8]
    [--scheme deft|wfbp|priority] [--partition-mb 26] [--steps 4] [--out DIR]

Writes DIR/trace_rank{r}.json (Chrome trace; kernels inside replayed CUDA
graphs included) and prints, per rank, a summary of the last steps: step time,
compute-stream busy time, and for every native DeFT kernel its stream, start
offset in the step and duration.  Diagnostic only (timings under a profiler
are never bench values).
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
import paper_2503_16815_b200 as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="vgg19")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--scheme", default="deft")
    ap.add_argument("--partition-mb", type=float, default=None)
    ap.add_argument("--placement", default="auto")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out/trace"))
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    world = int(os.environ.get("WORLD_SIZE", 1))
    dist = torch.distributed
    if world > 1:
        bench.init_quiet(dist, device)
    rank = dist.get_rank() if world > 1 else 0
    model = bench.build_model(args.model, device)
    batch = bench.make_batch(args.model, args.batch, device, seed=1234 + rank)
    loss_fn = bench.loss_fn_for(args.model)
    psize = 6_500_000 if args.partition_mb is None else int(args.partition_mb * 2**20 / 4)
    cfg = D.DeftConfig(lr=0.1, momentum=0.9, scheme=args.scheme,
                       update_placement=args.placement,
                       autocast_dtype=None if args.model == "gpt2" else torch.bfloat16,
                       partition=D.PartitionConfig(partition_size=psize, mu=1.0))
    ddp = D.DeftDataParallel(model, cfg)
    prof = ddp.measure_profile(batch, loss_fn, iters=3, name=args.model, batch_size=args.batch)
    part = ddp.plan(prof, ddp.cluster)
    ddp.warm_up(batch, loss_fn, min_steps=4)
    if ddp.static_batch is not None:
        batch = ddp.static_batch
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    marks = []
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                            torch.profiler.ProfilerActivity.CUDA]) as p:
        for _ in range(args.steps):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append(ev)
            ddp.train_step(batch, loss_fn)
        torch.cuda.synchronize()
    path = out / f"trace_rank{rank}.json"
    p.export_chrome_trace(str(path))
    meta = {"rank": rank, "world": world, "buckets": part.n_buckets,
            "bucket_ranges": [(b.lo, b.hi) for b in ddp.buckets],
            "graph_choice": ddp.graph_choice, "placement": ddp.placement,
            "decisions": [[d.to_dict() for d in pair] for pair in ddp.decision_log[-8:]]}
    (out / f"meta_rank{rank}.json").write_text(json.dumps(meta))
    ddp.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
