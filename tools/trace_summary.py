"""Summarise tools/trace_step.py's Chrome traces (run here, not on the box).

python tools/trace_summary.py gpurun_out/trace_dir [--rank 0] [--steps 2]
"""
import argparse
import json
from collections import defaultdict
from pathlib import Path

NATIVE = ("reduce_scatter", "update_allgather", "gather_kernel", "sgd_local", "ce_reduce",
          "barrier_kernel", "deft_")


def short(name):
    for k in NATIVE:
        if k in name:
            return name.split("<")[0].split("(")[0]
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dir")
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    d = Path(args.dir)
    tr = json.loads((d / f"trace_rank{args.rank}.json").read_text())
    evs = [e for e in tr["traceEvents"] if e.get("ph") == "X" and
           e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    evs.sort(key=lambda e: e["ts"])
    streams = defaultdict(list)
    for e in evs:
        streams[e["args"].get("stream", e.get("tid"))].append(e)
    # compute stream = the stream with the most MODEL (non-DeFT, non-copy) kernel
    # time -- under graph replay CUPTI spreads a graph's branches over several
    # streams, and a busy link stream (copy-engine pulls, spinning barrier
    # kernels) can out-total the compute stream
    busy = {s: sum(e["dur"] for e in v) for s, v in streams.items()}
    model = {s: sum(e["dur"] for e in v if not short(e["name"]) and e["cat"] == "kernel")
             for s, v in streams.items()}
    comp = max(model, key=model.get)
    t0, t1 = evs[0]["ts"], max(e["ts"] + e["dur"] for e in evs)
    print(f"span {t1 - t0:.0f} us over the traced steps; streams:")
    for s, v in sorted(streams.items(), key=lambda kv: -busy[kv[0]]):
        names = defaultdict(lambda: [0, 0.0])
        for e in v:
            k = short(e["name"]) or ("memcpy" if e["cat"] == "gpu_memcpy" else "model")
            names[k][0] += 1
            names[k][1] += e["dur"]
        tag = " (compute)" if s == comp else ""
        print(f"  stream {s}{tag}: busy {busy[s]:.0f} us, " +
              ", ".join(f"{k} x{n} {t:.0f}us" for k, (n, t) in sorted(names.items())))
    # idle gaps on the compute stream > 5 us
    cv = streams[comp]
    gaps = []
    for a, b in zip(cv, cv[1:]):
        g = b["ts"] - (a["ts"] + a["dur"])
        if g > 5:
            gaps.append((g, a["ts"] - t0, a["name"][:60], b["name"][:60]))
    gaps.sort(reverse=True)
    # union of all model-kernel activity (any stream): idle = no model kernel runs
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in evs
                if e["cat"] == "kernel" and not short(e["name"]))
    union, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                union += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        union += cur[1] - cur[0]
    print(f"model kernels active {union:.0f} us of {t1 - t0:.0f} us "
          f"({100 * union / (t1 - t0):.1f} %)")
    print(f"compute-stream idle total {sum(g for g, *_ in gaps):.0f} us in {len(gaps)} gaps > 5 us;"
          " largest:")
    for g, at, a, b in gaps[:15]:
        print(f"  {g:8.1f} us at +{at:9.1f}: after {a!r} before {b!r}")
    print("native kernels (first 80):")
    for e in [e for e in evs if short(e["name"])][:80]:
        print(f"  +{e['ts'] - t0:9.1f} us  {e['dur']:7.1f} us  stream {e['args'].get('stream')}"
              f"  {short(e['name'])}")


if __name__ == "__main__":
    main()
