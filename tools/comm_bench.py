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
NVLink bytes per launch: run it under tools/gpu/ncu_rank0.sh (ncu on rank 0
only, single-pass nvltx__bytes / nvlrx__bytes counters: no kernel replay, so
the cross-GPU barriers still meet their peers); tools/nvlink_bytes.py turns
that launch list into bytes per kernel next to the algorithmic figures.  (The
NVML NVLink counters report NOT_SUPPORTED on these B200s, and querying them
through pynvml corrupted the heap: not used.)
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


def timeit(fn, reps, warm, stream, device, graph=False):
    """ms per call, CUDA events on `stream`, after a barrier, max over ranks.
    graph: the reps calls are captured into one CUDA graph and replayed (no host
    launch cost between calls -- the way the training step issues them)."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    run = None
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(reps):
                fn()
        g.replay()                      # warm replay
        torch.cuda.synchronize()
        run = g.replay
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    if run is not None:
        run()
    else:
        for _ in range(reps):
            fn()
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


PHASE_NAMES = ["start", "epoch", "entry_barrier", "first_stage", "body", "drain", "end"]


def phases(comm, fn, stream, device):
    """Two back-to-back launches of fn with phase stamps (ns) -> per phase the
    median / max over blocks of (stamp - the launch's earliest start), us, plus
    the gap from the first launch's last block end to the second's first start."""
    bufs = [torch.zeros(256 * 8, dtype=torch.int64, device=device) for _ in range(2)]
    torch.cuda.synchronize()
    dist.barrier()
    for b in bufs:
        comm.set_phase_trace(b)
        fn()
    comm.set_phase_trace(None)
    torch.cuda.synchronize()
    out = {}
    ends = []
    for i, b in enumerate(bufs):
        st = b.view(256, 8).cpu().tolist()
        rows = [r for r in st if r[0] > 0]
        t0 = min(r[0] for r in rows)
        ph = {}
        for k, name in enumerate(PHASE_NAMES):
            d = sorted((r[k] - t0) / 1e3 for r in rows if r[k] > 0)
            if d:
                ph[name] = [round(d[len(d) // 2], 2), round(d[-1], 2)]
        ph["blocks"] = len(rows)
        out[f"launch{i}"] = ph
        ends.append((t0, max(r[6] for r in rows if r[6] > 0)))
    out["gap_us"] = round((ends[1][0] - ends[0][1]) / 1e3, 2)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,256")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--update-blocks", type=int, default=0,
                    help="CTA budget of the update kernels (0 = default)")
    ap.add_argument("--check", action="store_true",
                    help="verify every reduce-scatter result before timing")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="time every variant as a CUDA graph of --reps calls (device time "
                         "without host launch cost); keys *_ms then are graph times")
    ap.add_argument("--phases", action="store_true",
                    help="per-phase globaltimer stamps of every block (deft_comm_set_phase_trace): "
                         "start -> epoch -> entry barrier -> first stage -> body -> drain -> end, "
                         "and the gap between two back-to-back launches")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    W, rank = dist.get_world_size(), dist.get_rank()
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
        res = {"bucket_mb": mb, "world": W, "timing": "cuda graph" if args.graph else "eager"}
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
        with torch.cuda.stream(s):
            kernels = {
                "rs_sm": lambda: comm.reduce_scatter(_native.CHANNEL_SM, 0, 0, n, s),
                "rs_ce": lambda: comm.reduce_scatter(_native.CHANNEL_CE, 0, 0, n, s),
                # the multi-bucket entry point: the TMA-pipelined update kernel
                "upd_ag": lambda: comm.update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s),
                "oneshot": lambda: comm.sync_update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s),
            }
            for key, fn in kernels.items():
                res[f"{key}_ms"] = timeit(fn, args.reps, 3, s, dev, args.graph)
                if args.phases and key != "rs_ce":
                    res.setdefault("phases_us", {})[key] = phases(comm, fn, s, dev)

            def deft():
                comm.reduce_scatter(_native.CHANNEL_SM, 0, 0, n, s)
                comm.update_multi(0, [(0, n)], 1e-3, 1e-9, 0.9, mom, s)
            res["deft_ms"] = timeit(deft, args.reps, 3, s, dev, args.graph)
            if not args.no_nccl:
                x = torch.randn(n, device=dev)
                p = torch.randn(n, device=dev)
                v = torch.zeros(n, device=dev)
                res["nccl_ar_ms"] = timeit(lambda: dist.all_reduce(x), args.reps, 3, s, dev, args.graph)

                def nccl_sgd():
                    dist.all_reduce(x)
                    v.mul_(0.9).add_(x, alpha=1e-3)
                    p.add_(v, alpha=-1e-9)
                res["nccl_ar_sgd_ms"] = timeit(nccl_sgd, args.reps, 3, s, dev, args.graph)
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
        # algorithmic NVLink bytes per rank and launch: RS rx (W-1)/W, AG tx
        # (W-1)/W, one-shot rx (W-1) x bucket (the ncu counters: nvlink_bytes.py)
        res["nvlink_algorithmic"] = {"rs_rx": int(frac * nbytes), "upd_ag_tx":
                                     int(frac * nbytes), "oneshot_rx": (W - 1) * nbytes}
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
