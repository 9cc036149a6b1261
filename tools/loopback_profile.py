"""ncu target for the comm kernels on ONE GPU: a loopback world (W ranks in one
process, peers' buffers local) running the collective reduce-scatter / update
launches (one launch for all ranks, gridDim.y = W), which complete under a
kernel profiler's replay.  The "peer" traffic is local HBM here, so this shows
the kernels' pipeline, stall and shared-memory behaviour, not NVLink.

ncu --set full -k regex:update_allgather_tma -s 2 -c 1 python tools/loopback_profile.py --mb 64
"""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2503_16815_b200 import _native  # noqa: E402
from paper_2503_16815_b200.loopback import LoopbackWorld  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--mb", type=float, default=64)
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lw = LoopbackWorld(args.world, dev)
    n = int(args.mb * 2**20) // 4
    comms = lw.make_comms(1, n, torch.float32)
    for c in comms:
        c.grads.normal_()
        c.params.normal_()
    moms = [torch.zeros(n, device=dev) for _ in comms]
    s = torch.cuda.Stream(dev)
    for _ in range(args.reps):
        lw.collective_reduce_scatter(comms, _native.CHANNEL_SM, 0, [(0, n)], s)
        lw.collective_update(comms, 0, [(0, n)], 1e-9, 1e-3, 0.9, moms, s)
    s.synchronize()
    for c in comms:
        c.close(barrier=False)
    print(f"loopback W={args.world} {args.mb} MB x{args.reps}: rs + update collectives done")


if __name__ == "__main__":
    main()
