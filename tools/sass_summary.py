"""SASS evidence for the hot kernels: dump the sm_100a SASS of
the comm / update / solver kernels from the built libdeft_b200.so and count the
instructions that show how they move data (bulk copies, mbarrier syncs, 128-bit
loads/stores, system-scope fences).

python tools/sass_summary.py [--out profiles/r02_sass]  -> <out>/<kernel>.sass + summary.json
"""
import argparse
import collections
import json
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "paper_2503_16815_b200" / "libdeft_b200.so"
# the instantiations the W = 4 fp32 step runs (and W = 8 / bf16 where they differ)
WANT = [
    "reduce_scatter_tma_kernel<float, 2, 4, false>",
    "reduce_scatter_tma_kernel<float, 4, 4, false>",
    "update_allgather_tma_kernel<float, 2, 4, 1, false, 4096>",
    "update_allgather_tma_kernel<float, 4, 4, 1, false, 2048>",
    "update_allgather_tma_kernel<__nv_bfloat16, 8, 4, 1, false, 2048>",
    "oneshot_update_kernel<float, 4>",
    "sgd_local_kernel<float, 2>",
    "gather_kernel",
    "ce_reduce_kernel<float>",
    "barrier_kernel",
    "subset_sum_kernel<false>",
    "subset_sum_kernel<true>",
    "deft_scheduler_kernel",
]
OPS = ["UBLKCP", "UTMALDG", "UTMASTG", "UBLKRED", "SYNCS", "LDG.E.128", "LDG.E.ENL2.128",
       "STG.E.128", "LDS.128", "STS.128", "LDG", "STG", "ATOMG", "RED", "MEMBAR", "FENCE",
       "NANOSLEEP", "FFMA", "LOP3", "SHF", "POPC", "FLO", "BAR", "WARPSYNC", "VOTE", "SHFL"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_sass"))
    a = ap.parse_args()
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    text = subprocess.run(["cuobjdump", "-sass", str(SO)], check=True, capture_output=True,
                          text=True).stdout
    funcs = re.split(r"\n\s*Function : ", text)[1:]
    summary = {}
    for f in funcs:
        mangled = f.split("\n", 1)[0].strip()
        name = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
        short = re.sub(r"^void |^deft::|\(.*$", "", name).replace("deft::", "")
        if short not in WANT:
            continue
        ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", f)
        c = collections.Counter(ins)
        counts = {op: sum(v for k, v in c.items() if k == op or k.startswith(op + "."))
                  for op in OPS}
        summary[short] = {"instructions": len(ins),
                          "counts": {k: v for k, v in counts.items() if v}}
        fn = re.sub(r"[^A-Za-z0-9_]+", "_", short).strip("_")
        (out / f"{fn}.sass").write_text(f)
    (out / "summary.json").write_text(json.dumps(summary, indent=1, sort_keys=True) + "\n")
    for k, v in summary.items():
        print(k, v["instructions"], v["counts"])


if __name__ == "__main__":
    main()
