"""NVLink bytes per launch of the comm kernels from the driver's per-link
throughput counters (`nvidia-smi nvlink -gt d`), read on rank 0 before and after
K launches of each kernel -- no profiler attached (ncu stalls on processes with
CUDA-IPC peer mappings).

torchrun --nproc-per-node 2 tools/nvlink_smi.py [--mb 64] [--launches 50]
"""
import argparse
import json
import os
import re
import subprocess
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2503_16815_b200 import _native  # noqa: E402
from paper_2503_16815_b200.comm import BucketComm  # noqa: E402

UNIT = {"B": 1, "KIB": 1024, "MIB": 1024**2, "GIB": 1024**3, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def counters(gpu: int):
    """(tx_bytes, rx_bytes, raw text) summed over the GPU's links, or None."""
    for cmd in (["nvidia-smi", "nvlink", "-gt", "d", "-i", str(gpu)],
                ["nvidia-smi", "nvlink", "--getthroughput", "d", "-i", str(gpu)]):
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=30).stdout
        except Exception as e:  # noqa: BLE001
            out = repr(e)
        tx = rx = 0.0
        seen = False
        for line in out.splitlines():
            m = re.search(r"(Tx|Rx)\w*\s*:?\s*([\d.]+)\s*([KMG]i?B)?", line, re.I)
            if m:
                seen = True
                v = float(m.group(2)) * UNIT.get((m.group(3) or "KiB").upper(), 1024)
                if m.group(1).lower() == "tx":
                    tx += v
                else:
                    rx += v
        if seen:
            return tx, rx, out[:600]
    return None, None, out[:600]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=float, default=64)
    ap.add_argument("--launches", type=int, default=50)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    W, rank = dist.get_world_size(), dist.get_rank()
    n = int(args.mb * 2**20) // 4
    comm = BucketComm(rank, W, 1, n, torch.float32, dev)
    comm.grads.normal_()
    mom = torch.zeros(n, device=dev)
    x = torch.randn(n, device=dev)
    s = torch.cuda.Stream(dev)
    kinds = {
        "reduce_scatter_tma": lambda: comm.reduce_scatter(_native.CHANNEL_SM, 0, 0, n, s),
        "update_allgather_tma": lambda: comm.update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s),
        "nccl_all_reduce": lambda: dist.all_reduce(x),
    }
    out = {"world": W, "bucket_mb": args.mb, "launches": args.launches,
           "algorithmic_bytes_per_launch": {"reduce_scatter_tma (rx)": (W - 1) * n * 4 // W,
                                            "update_allgather_tma (tx)": (W - 1) * n * 4 // W,
                                            "nccl_all_reduce (tx = rx)": 2 * (W - 1) * n * 4 // W}}
    for name, fn in kinds.items():
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        dist.barrier()
        before = counters(local) if rank == 0 else None
        dist.barrier()
        with torch.cuda.stream(s):
            for _ in range(args.launches):
                fn()
        torch.cuda.synchronize()
        dist.barrier()
        after = counters(local) if rank == 0 else None
        if rank == 0:
            if before[0] is None or after[0] is None:
                out[name] = {"error": "no counters", "raw": after[2]}
            else:
                out[name] = {"tx_bytes_per_launch": round((after[0] - before[0]) / args.launches),
                             "rx_bytes_per_launch": round((after[1] - before[1]) / args.launches)}
    if rank == 0:
        out["raw_sample"] = after[2] if after else None
        print(json.dumps(out), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
