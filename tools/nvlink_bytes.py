"""NVLink bytes per launch from an ncu rank-0 launch list (tools/gpu/ncu_rank0.sh):
per kernel, the mean nvltx / nvlrx bytes (all and user data) and duration over
its launches, beside the algorithmic bytes crossing NVLink per rank.

python tools/nvlink_bytes.py LAUNCHES.csv --bucket-mb 64 --world 4 [--dtype-bytes 4]
"""
import argparse
import collections
import csv
import json
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--bucket-mb", type=float, required=True)
    ap.add_argument("--world", type=int, required=True)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    h = rows[hdr]
    ki, ii, mi, vi = (h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"),
                      h.index("Metric Value"))
    per = collections.defaultdict(lambda: collections.defaultdict(dict))
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"^void |[<(].*$", "", r[ki]).replace("deft::", "")
        try:
            per[name][r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    nbytes = int(a.bucket_mb * 2**20)
    frac = (a.world - 1) / a.world
    algo = {"reduce_scatter_tma_kernel": ("rx", frac * nbytes),
            "reduce_scatter_kernel": ("rx", frac * nbytes),
            "update_allgather_tma_kernel": ("tx", frac * nbytes),
            "oneshot_update_kernel": ("rx", (a.world - 1) * nbytes)}
    out = {"bucket_mb": a.bucket_mb, "world": a.world, "kernels": {}}
    for name, launches in per.items():
        ms = list(launches.values())
        avg = {k: sum(m.get(k, 0.0) for m in ms) / len(ms) for k in ms[0]}
        rec = {"launches": len(ms),
               "duration_us": round(avg.get("gpu__time_duration.sum", 0) / 1e3, 2),
               "nvl_tx_bytes": int(avg.get("nvltx__bytes.sum", 0)),
               "nvl_rx_bytes": int(avg.get("nvlrx__bytes.sum", 0)),
               "nvl_tx_user_bytes": int(avg.get("nvltx__bytes_data_user.sum", 0)),
               "nvl_rx_user_bytes": int(avg.get("nvlrx__bytes_data_user.sum", 0))}
        if name in algo:
            d, b = algo[name]
            rec["algorithmic_bytes"] = int(b)
            rec["algorithmic_direction"] = d
            rec["user_over_algorithmic"] = round(rec[f"nvl_{d}_user_bytes"] / b, 3) if b else None
        out["kernels"][name] = rec
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
