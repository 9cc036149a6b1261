"""One DeFT training step bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (launch list / full-set captures).

python tools/profile_step.py [--model resnet101] [--steps 1] [--eager]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2503_16815_b200 as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet101")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--eager", action="store_true")
    args = ap.parse_args()
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda", 0)
    model = bench.build_model(args.model, dev)
    loss_fn = bench.loss_fn_for(args.model)
    batch = bench.make_batch(args.model, 64, dev)
    walk = D.WalkParams.from_dict(bench.DEFAULT_WALK)
    cfg = D.DeftConfig(lr=0.1, momentum=0.9, walk=walk, cuda_graphs=not args.eager,
                       partition=D.PartitionConfig(partition_size=6_500_000, mu=1.0))
    ddp = D.DeftDataParallel(model, cfg)
    ddp.measure_profile(batch, loss_fn, iters=2, name=args.model, batch_size=64)
    ddp.plan()
    ddp.warm_up(batch, loss_fn)
    if ddp.static_batch is not None:
        batch = ddp.static_batch
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.steps):
        ddp.train_step(batch, loss_fn)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(json.dumps({"ok": True, "buckets": len(ddp.buckets),
                      "graphs": len(ddp._graphs) if ddp._graphs is not None else 0}))
    ddp.close()


if __name__ == "__main__":
    main()
