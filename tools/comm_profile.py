"""ncu --set full of ONE multi-GPU comm kernel on the real NVLink.

torchrun --nproc-per-node 2 --no-python tools/gpu/ncu_full_rank0.sh OUT KERNEL \
    python tools/comm_profile.py --kernel update --mb 64

No NCCL anywhere in the process (a kernel profiler attached to a process that
initialises NCCL hangs in the communicator set-up): the IPC handles and the
rank barriers go over a gloo process group, and DEFT_PROFILE_NO_PEER_BARRIER=1
(set by ncu_full_rank0.sh) turns the kernels' cross-GPU barriers off, so the
profiler can replay rank 0's launch while rank 1 is elsewhere.  The timings
and results of such a run are meaningless; its counters (DRAM bytes, NVLink
bytes, stall reasons, shared-memory / TMA activity) are what it is for.

  --kernel rs       reduce_scatter_tma_kernel   (SM channel, bucket of --mb MB)
  --kernel update   update_allgather_tma_kernel
  --kernel oneshot  oneshot_update_kernel
"""
import argparse
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2503_16815_b200 import _native  # noqa: E402
from paper_2503_16815_b200.comm import BucketComm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", choices=["rs", "update", "oneshot"], default="update")
    ap.add_argument("--mb", type=float, default=64)
    ap.add_argument("--launches", type=int, default=6)
    ap.add_argument("--bf16", action="store_true")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    W, rank = dist.get_world_size(), dist.get_rank()
    dt = torch.bfloat16 if args.bf16 else torch.float32
    esz = 2 if args.bf16 else 4
    n = int(args.mb * 2**20) // esz
    comm = BucketComm(rank, W, 1, n, dt, dev)
    comm.grads.normal_()
    comm.params.normal_()
    mom = torch.zeros(n, device=dev)
    s = torch.cuda.Stream(dev)
    fn = {"rs": lambda: comm.reduce_scatter(_native.CHANNEL_SM, 0, 0, n, s),
          "update": lambda: comm.update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s),
          "oneshot": lambda: comm.sync_update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s)
          }[args.kernel]
    for _ in range(args.launches):
        fn()
        s.synchronize()
        dist.barrier()
    comm.close(barrier=False)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(f"profiled {args.kernel} {args.mb} MB x{args.launches} at W={W}")


if __name__ == "__main__":
    main()
