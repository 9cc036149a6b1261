"""W = 1 fused delayed update (sgd_local_kernel) variants, one GPU:
units per thread (DEFT_SGD_UNROLL) x grid cap (DEFT_SGD_CTAS_PER_SM), each in
a fresh process (the launcher reads its env once), timed with CUDA events over
back-to-back launches on the ResNet-101 parameter count (44,549,160 fp32, 8
buckets, 20 B/param of algorithmic HBM traffic) -> JSON lines.

python tools/update_bench.py [--params 44549160 --buckets 8 --reps 20]
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child(params, nb, reps, dtype_name):
    sys.path.insert(0, str(ROOT))
    import torch
    from paper_2503_16815_b200.comm import BucketComm
    dtype = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    dev = torch.device("cuda", 0)
    c = BucketComm(0, 1, 1, params, dtype, dev)
    c.grads[0].normal_()
    c.params.normal_()
    mom = torch.zeros(params, dtype=torch.float32, device=dev)
    cuts = [params * i // nb for i in range(nb + 1)]
    ranges = list(zip(cuts, cuts[1:]))
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            c.update_multi(0, ranges, 1.0, 1e-3, 0.9, mom, s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            c.update_multi(0, ranges, 1.0, 1e-3, 0.9, mom, s)
        b.record(s)
        torch.cuda.synchronize()
    us = a.elapsed_time(b) / reps * 1e3
    nbytes = params * (20 if dtype == torch.float32 else 4 + 2 + 2 + 12)
    print(json.dumps({"us_per_launch": round(us, 2), "bytes": nbytes,
                      "gbs": round(nbytes / us / 1e3, 1)}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--params", type=int, default=44_549_160)
    ap.add_argument("--buckets", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--grid", default="1:8,2:8,4:8,2:4,4:4,2:16,1:16")
    a = ap.parse_args()
    if a.child:
        return child(a.params, a.buckets, a.reps, a.dtype)
    peak = None
    try:
        peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        pass
    for spec in a.grid.split(","):
        u, k = spec.split(":")
        env = dict(os.environ, DEFT_SGD_UNROLL=u, DEFT_SGD_CTAS_PER_SM=k)
        r = subprocess.run([sys.executable, __file__, "--child", "--params", str(a.params),
                            "--buckets", str(a.buckets), "--reps", str(a.reps),
                            "--dtype", a.dtype], env=env, capture_output=True, text=True)
        line = {"unroll": int(u), "ctas_per_sm": int(k), "dtype": a.dtype}
        try:
            line.update(json.loads(r.stdout.strip().splitlines()[-1]))
            if peak:
                line["frac_of_hbm_peak"] = round(line["gbs"] / peak, 4)
        except Exception:
            line["error"] = r.stderr[-400:]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
