"""Bucket communication microbenchmark (BASELINE configs[4]: 1-256 MB buckets at
2/4/8 GPUs vs the NCCL baseline).

torchrun --nproc-per-node N tools/comm_bench.py [--sizes-mb 1,4,16,64,256]

For each bucket size, timed with CUDA events on the launching stream after a
barrier, max over ranks:
  rs_sm     reduce-scatter, SM P2P channel        (deft_bucket_reduce_scatter ch 0)
  rs_ce     reduce-scatter, copy-engine channel   (ch 1)
  upd_ag    fused SGD/momentum + parameter all-gather (deft_bucket_update)
  deft      rs_sm + upd_ag back to back = a full DeFT bucket sync incl. the update
  oneshot   fused all-reduce + update in one launch (deft_bucket_sync_update_multi)
  nccl_ar   NCCL all_reduce (fp32 sum) of the bucket
  nccl_ar_sgd  NCCL all_reduce + torch SGD/momentum on the bucket (the DDP baseline)
Bus bandwidth: RS and AG move (W-1)/W of the bucket per rank each; AR 2(W-1)/W.
--nvml: NVLink TX/RX bytes per launch of every kernel, from the NVML
throughput counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, summed over
links) read around the timed loop -- isolated launches, so no profiler replay
of cross-GPU barriers is needed; compare with the algorithmic bytes.
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2503_16815_b200 import _native  # noqa: E402
from paper_2503_16815_b200.comm import BucketComm  # noqa: E402


NVML = {}


def nvlink_bytes():
    """{family: (tx, rx)} NVLink bytes of this GPU so far, from every NVML counter
    family this driver offers (summed over links): COUNT_XMIT/RCV_BYTES (the
    per-link byte counters) and THROUGHPUT_DATA_TX/RX (KiB units)."""
    h = NVML.get("h")
    if h is None:
        return None
    import pynvml as N
    fams = {"count_bytes": (N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
                            N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, 1),
            "throughput_data": (N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024)}
    out = {}
    for fam, (ftx, frx, unit) in fams.items():
        fields = []
        for link in range(NVML["links"]):
            fields += [(ftx, link), (frx, link)]
        try:
            vals = N.nvmlDeviceGetFieldValues(h, fields)
        except Exception as e:  # noqa: BLE001
            out[fam] = repr(e)
            continue
        ok = [v for v in vals if v.nvmlReturn == 0]
        if not ok:
            out[fam] = f"nvmlReturn {vals[0].nvmlReturn}"
            continue
        tx = sum(v.value.ullVal for v in vals[0::2] if v.nvmlReturn == 0)
        rx = sum(v.value.ullVal for v in vals[1::2] if v.nvmlReturn == 0)
        out[fam] = (tx * unit, rx * unit)
    return out


def nvml_init(device):
    try:
        import pynvml as N
        N.nvmlInit()
        idx = torch.cuda._get_nvml_device_index(device.index)
        NVML["h"] = N.nvmlDeviceGetHandleByIndex(idx)
        NVML["links"] = 18
    except Exception as e:  # reported in the output
        NVML["error"] = repr(e)


def timeit(fn, reps, warm, stream, device):
    """ms per call, CUDA events on `stream`, after a barrier, max over ranks."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def nvml_count(fn, reps, nv, key):
    """NVLink bytes per call of `fn` (NVML counters read before and after `reps`
    barrier-aligned calls; never inside a timed region -- reading NVML takes
    milliseconds and would skew the ranks)."""
    import time
    torch.cuda.synchronize()
    dist.barrier()
    time.sleep(0.2)
    before = nvlink_bytes()
    dist.barrier()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    time.sleep(0.2)          # counters are sampled by the driver
    after = nvlink_bytes()
    res = {}
    for fam, v in after.items():
        if isinstance(v, tuple) and isinstance(before.get(fam), tuple):
            res[fam] = {"tx": (v[0] - before[fam][0]) / reps, "rx": (v[1] - before[fam][1]) / reps}
        else:
            res[fam] = v
    nv[key] = res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,256")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--update-blocks", type=int, default=0,
                    help="CTA budget of the update kernels (0 = default)")
    ap.add_argument("--check", action="store_true",
                    help="verify every reduce-scatter result before timing")
    ap.add_argument("--nvml", action="store_true", help="NVLink bytes per launch (NVML)")
    ap.add_argument("--no-nccl", action="store_true")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    W, rank = dist.get_world_size(), dist.get_rank()
    if args.nvml:
        nvml_init(dev)
    sizes = [float(x) for x in args.sizes_mb.split(",")]
    max_elems = int(max(sizes) * 2**20) // 4
    comm = BucketComm(rank, W, 1, max_elems, torch.float32, dev)
    comm.grads.normal_()
    comm.set_update_blocks(args.update_blocks)
    mom = torch.zeros(max_elems, device=dev)
    s = torch.cuda.Stream(dev)
    rows = []
    for mb in sizes:
        n = int(mb * 2**20) // 4
        nbytes = n * 4
        res = {"bucket_mb": mb, "world": W}
        if args.check:
            for ch in (_native.CHANNEL_SM, _native.CHANNEL_CE):
                idx = torch.arange(n, device=dev, dtype=torch.float32)
                comm.grads[0, :n].copy_(torch.sin(idx * 0.001 + rank))
                torch.cuda.synchronize()
                dist.barrier()
                comm.reduce_scatter(ch, 0, 0, n, s)
                torch.cuda.synchronize()
                want = sum(torch.sin(idx * 0.001 + r) for r in range(W))
                per = (n + W - 1) // W
                lo = 0 if rank == 0 else -(-(rank * per) // 4) * 4
                hi = n if rank == W - 1 else -(-((rank + 1) * per) // 4) * 4
                err = float((comm.grads[0, lo:hi] - want[lo:hi]).abs().max())
                res[f"check_err_ch{ch}"] = err
                assert err < 1e-4, (ch, err)
                dist.barrier()
        nv = {} if args.nvml else None
        with torch.cuda.stream(s):
            kernels = {
                "rs_sm": lambda: comm.reduce_scatter(_native.CHANNEL_SM, 0, 0, n, s),
                "rs_ce": lambda: comm.reduce_scatter(_native.CHANNEL_CE, 0, 0, n, s),
                # the multi-bucket entry point: the TMA-pipelined update kernel
                "upd_ag": lambda: comm.update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s),
                "oneshot": lambda: comm.sync_update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s),
            }
            for key, fn in kernels.items():
                res[f"{key}_ms"] = timeit(fn, args.reps, 3, s, dev)
            if nv is not None:
                for key, fn in kernels.items():
                    nvml_count(fn, args.reps, nv, key)

            def deft():
                comm.reduce_scatter(_native.CHANNEL_SM, 0, 0, n, s)
                comm.update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s)
            res["deft_ms"] = timeit(deft, args.reps, 3, s, dev)
            if not args.no_nccl:
                x = torch.randn(n, device=dev)
                p = torch.randn(n, device=dev)
                v = torch.zeros(n, device=dev)
                res["nccl_ar_ms"] = timeit(lambda: dist.all_reduce(x), args.reps, 3, s, dev)
                if nv is not None:
                    nvml_count(lambda: dist.all_reduce(x), args.reps, nv, "nccl_ar")

                def nccl_sgd():
                    dist.all_reduce(x)
                    v.mul_(0.9).add_(x, alpha=1e-3)
                    p.add_(v, alpha=-1e-9)
                res["nccl_ar_sgd_ms"] = timeit(nccl_sgd, args.reps, 3, s, dev)
        frac = (W - 1) / W
        res["rs_sm_busbw_gbs"] = round(frac * nbytes / res["rs_sm_ms"] / 1e6, 1)
        res["rs_ce_busbw_gbs"] = round(frac * nbytes / res["rs_ce_ms"] / 1e6, 1)
        res["upd_ag_busbw_gbs"] = round(frac * nbytes / res["upd_ag_ms"] / 1e6, 1)
        res["deft_busbw_gbs"] = round(2 * frac * nbytes / res["deft_ms"] / 1e6, 1)
        res["oneshot_busbw_gbs"] = round(2 * frac * nbytes / res["oneshot_ms"] / 1e6, 1)
        res["best_sync_ms"] = min(res["deft_ms"], res["oneshot_ms"])
        if "nccl_ar_ms" in res:
            res["nccl_ar_busbw_gbs"] = round(2 * frac * nbytes / res["nccl_ar_ms"] / 1e6, 1)
            res["deft_vs_nccl_ar_sgd"] = round(res["nccl_ar_sgd_ms"] / res["deft_ms"], 3)
            res["best_vs_nccl_ar"] = round(res["nccl_ar_ms"] / res["best_sync_ms"], 3)
        if nv is not None:
            # algorithmic NVLink bytes per rank: RS rx (W-1)/W, AG tx (W-1)/W,
            # one-shot rx (W-1) x bucket; the measured counters beside them
            res["nvlink"] = nv
            res["nvlink_algorithmic"] = {"rs_rx": int(frac * nbytes), "upd_ag_tx":
                                         int(frac * nbytes), "oneshot_rx": (W - 1) * nbytes}
        if NVML.get("error"):
            res["nvml_error"] = NVML["error"]
        for k in list(res):
            if k.endswith("_ms"):
                res[k] = round(res[k], 4)
        rows.append(res)
        if rank == 0:
            print(json.dumps(res), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
