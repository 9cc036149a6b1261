"""Key counters of one `ncu --page raw --csv` export (one profiled launch).

python tools/ncu_summary.py gpurun_out/X.raw.csv [--alg-bytes N] [--json]

Prints duration, DRAM / L2 / NVLink bytes, achieved bandwidths, SM and memory
throughput percentages and the top warp-stall reasons -- the numbers
profiles/*_ncu_*.json keep for the comm and update kernels.
"""
import argparse
import csv
import json
import sys

KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "l2_read_bytes": "lts__t_bytes_srcunit_tex_op_read.sum",
    "nvlink_tx_bytes": "nvltx__bytes.sum",
    "nvlink_rx_bytes": "nvlrx__bytes.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "mem_throughput_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "smem_per_block_bytes": "launch__shared_mem_per_block",
}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def load(path):
    with open(path, newline="") as f:
        rows = [r for r in csv.reader(f)]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    names, units = rows[hdr], rows[hdr + 1]
    data = [r for r in rows[hdr + 2:] if len(r) == len(names)]
    return names, units, data


def summary(path, alg_bytes=None):
    names, units, data = load(path)
    col = {n: i for i, n in enumerate(names)}
    r = data[0]
    out = {"kernel": r[col["Kernel Name"]][:120]}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6,
             "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for k, m in KEYS.items():
        if m in col:
            v = num(r[col[m]])
            if v is not None:
                out[k] = v * scale.get(units[col[m]], 1)
    d = out.get("duration_ns")
    if d:
        dram = out.get("dram_read_bytes", 0) + out.get("dram_write_bytes", 0)
        out["dram_gbs"] = round(dram / d, 1)
        for k in ("nvlink_tx_bytes", "nvlink_rx_bytes"):
            if k in out:
                out[k.replace("_bytes", "_gbs")] = round(out[k] / d, 1)
        if alg_bytes:
            out["alg_bytes"] = alg_bytes
            out["alg_gbs"] = round(alg_bytes / d, 1)
    stalls = {}
    pre = "smsp__average_warp_latency_issue_stalled_"
    pre2 = "smsp__average_warps_issue_stalled_"
    for n, i in col.items():
        for p in (pre, pre2):
            if n.startswith(p) and n.endswith("_per_issue_active.ratio"):
                v = num(r[i])
                if v:
                    stalls[n[len(p):-len("_per_issue_active.ratio")]] = v
    out["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--alg-bytes", type=float, default=None)
    args = ap.parse_args()
    json.dump(summary(args.csv, args.alg_bytes), sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
