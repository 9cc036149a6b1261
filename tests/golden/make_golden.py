"""Generate the golden vectors the parity tests are pinned on.

Runs the UNMODIFIED reference (`deftsim`, imported read-only from
/root/reference/pkg/src) in this container and records its outputs:

* ``inputs.json``            -- the reference fixture profiles / clusters / walk
                                parameters, re-serialised (the GPU box has no
                                /root/reference, so the tests read them from here)
* ``naive.jsonl.gz``         -- naive_knapsack  (knapsack.py:55-94)
* ``recursive.jsonl.gz``     -- recursive_knapsack (knapsack.py:97-127)
* ``greedy.jsonl.gz``        -- greedy_multi_knapsack (knapsack.py:130-159)
* ``partition.json``         -- partition_buckets (partition.py:67-120)
* ``schedules/*.jsonl.gz``   -- Schedule.dump_jsonl byte streams (scheduler.py:142-145)
* ``schedules.json``         -- index: config -> file, sha256, feedback_loop verdict
* ``preserver.json``         -- expected_next_state / check_sequence values

Usage (only in the build container; never on the GPU box):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
"""
from __future__ import annotations

import gzip
import hashlib
import json
import random
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
REF_FIX = Path("/root/reference/pkg/fixtures")
OUT = Path(__file__).resolve().parent

sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

import deftsim as ds  # noqa: E402
from deftsim.knapsack import MAX_EXACT_CAPACITY  # noqa: E402

NEAR_ONE = 1.0000001  # reference tests/conftest.py:19


def uniform_profile(n, comm_us=900, fwd_total=3600, bwd_total=7200, batch=256):
    """Same construction as the reference's tests/conftest.py:65-87."""
    fwd = [fwd_total // n] * n
    bwd = [bwd_total // n] * n
    for i in range(fwd_total - sum(fwd)):
        fwd[i] += 1
    for i in range(bwd_total - sum(bwd)):
        bwd[i] += 1
    return ds.ModelProfile(
        name=f"uniform{n}",
        buckets=tuple(ds.BucketProfile(i + 1, 1000, fwd[i], bwd[i], comm_us) for i in range(n)),
        batch_size=batch,
    )


def clusters():
    dual = ds.load_cluster(REF_FIX / "cluster_dual.json")
    fast = ds.ClusterSpec(links=(ds.LinkSpec(name="fast"),))
    equal = ds.ClusterSpec(links=(ds.LinkSpec(name="fast"),
                                  ds.LinkSpec(name="twin", speed_ratio_to_fast=NEAR_ONE)))
    return {"dual": dual, "fast": fast, "equal_dual": equal}


def cluster_dict(c):
    return {"links": [{"name": l.name, "speed_ratio_to_fast": l.speed_ratio_to_fast,
                       "bandwidth_bps": l.bandwidth_bps, "startup_us": l.startup_us}
                      for l in c.links]}


def write_jsonl_gz(path: Path, rows):
    path.parent.mkdir(parents=True, exist_ok=True)
    blob = "".join(json.dumps(r, sort_keys=True) + "\n" for r in rows).encode()
    with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as f:
        f.write(blob)


def items_of(ws, ids=None):
    ids = ids or list(range(1, len(ws) + 1))
    return [ds.Item(bucket_id=i, weight=w) for i, w in zip(ids, ws)]


def gen_naive():
    rng = random.Random(20261018)
    rows = []

    def rec(ws, cap, ids=None):
        ids = ids or list(range(1, len(ws) + 1))
        asn = ds.naive_knapsack(items_of(ws, ids), cap)
        rows.append({"ids": ids, "weights": ws, "cap": cap,
                     "selection": list(asn.selections[0]), "value": asn.total_value,
                     "leftovers": list(asn.leftovers)})

    # edge cases (reference tests/test_knapsack.py:34-51)
    rec([], 100)
    rec([5, 3], 0)
    rec([4, 6, 3], 10)
    rec([5, 5], 5)
    rec([1], 1)
    rec([7], 6)
    rec([3, 3, 3, 3], 6)
    rec([10, 20, 30], 1000)          # everything fits
    rec([2, 3, 5, 7, 11, 13], 20)
    # non-contiguous, shuffled ids: solver sorts by id internally
    rec([9, 4, 4, 1], 8, [40, 3, 17, 8])
    # small random (acceptance C2 style)
    for _ in range(400):
        n = rng.randint(1, 15)
        ws = [rng.randint(1, 600) for _ in range(n)]
        rec(ws, rng.randint(0, sum(ws) + 50))
    # many ties
    for _ in range(200):
        n = rng.randint(2, 20)
        ws = [rng.choice([3, 5, 6, 9, 10, 15]) for _ in range(n)]
        rec(ws, rng.randint(0, sum(ws)))
    # scheduler-sized exact mode: n 10..60, capacities up to ~1.5e6 us
    for _ in range(150):
        n = rng.randint(10, 60)
        cap = rng.randint(50_000, 1_500_000)
        ws = [rng.randint(1, max(2, cap // max(1, n // 3))) for _ in range(n)]
        rec(ws, cap)
    # word-boundary stress: weights / caps near multiples of 32 and 64
    for _ in range(100):
        n = rng.randint(1, 24)
        ws = [rng.choice([31, 32, 33, 63, 64, 65, 95, 96, 97, 127, 128, 129]) * rng.randint(1, 9)
              for _ in range(n)]
        cap = rng.choice([31, 32, 33, 63, 64, 65, 1023, 1024, 1025]) * rng.randint(1, 12)
        rec(ws, cap)
    # scaled mode: capacity above MAX_EXACT_CAPACITY (knapsack.py:47-52)
    for _ in range(12):
        n = rng.randint(2, 14)
        cap = rng.randint(MAX_EXACT_CAPACITY + 1, 4 * MAX_EXACT_CAPACITY)
        ws = [rng.randint(10**5, cap // 2) for _ in range(n)]
        rec(ws, cap)
    rec([10**7 + 5, 3, 10**7 - 3], 10**7 + 1)
    return rows


def gen_recursive():
    rng = random.Random(404_2026)
    rows = []

    def rec(ws_desc, ids_desc, remain, bwd):
        order = ds.recursive_knapsack(items_of(ws_desc, ids_desc), remain, bwd)
        rows.append({"ids": ids_desc, "weights": ws_desc, "remain": remain,
                     "backward": bwd, "order": order})

    # SURVEY §7 counterexample: deeper level wins in scaled mode
    rec([10**7 + 5, 3, 10**7 - 3], [3, 2, 1], 10**7 + 1, [0, 1, 0])
    rec([], [], 5, [])
    rec([5], [1], -3, [0])
    for _ in range(300):
        n = rng.randint(1, 9)
        ws = [rng.randint(1, 150) for _ in range(n)]
        bwd = [rng.randint(0, 80) for _ in range(n)]
        ids = list(range(n, 0, -1))
        rec(ws, ids, rng.randint(-50, 400), bwd)
    for _ in range(40):
        n = rng.randint(5, 40)
        ws = [rng.randint(1000, 60000) for _ in range(n)]
        bwd = [rng.randint(0, 20000) for _ in range(n)]
        ids = list(range(n, 0, -1))
        rec(ws, ids, rng.randint(0, sum(ws)), bwd)
    # scaled mode at the top level, exact at deeper levels
    for _ in range(8):
        n = rng.randint(2, 6)
        ws = [rng.randint(10**6, 9 * 10**6) for _ in range(n)]
        bwd = [rng.randint(0, 4 * 10**6) for _ in range(n)]
        ids = list(range(n, 0, -1))
        rec(ws, ids, rng.randint(MAX_EXACT_CAPACITY + 1, 2 * MAX_EXACT_CAPACITY), bwd)
    return rows


def gen_greedy():
    rng = random.Random(77_2026)
    rows = []
    for _ in range(400):
        n = rng.randint(0, 18)
        m = rng.randint(1, 4)
        ws = [rng.randint(1, 500) for _ in range(n)]
        caps = [rng.randint(0, 1000) for _ in range(m)]
        asn = ds.greedy_multi_knapsack(items_of(ws), caps)
        rows.append({"weights": ws, "caps": caps,
                     "selections": [list(s) for s in asn.selections],
                     "value": asn.total_value, "leftovers": list(asn.leftovers)})
    return rows


def main():
    cl = clusters()
    profiles = {name: ds.load_profile(REF_FIX / f"{name}.json")
                for name in ("resnet101", "vgg19", "gpt2")}
    walk_raw = json.loads((REF_FIX / "walk_merged_updates.json").read_text())
    walk = ds.WalkParams.from_dict(walk_raw)
    inputs = {
        "profiles": {k: ds.profile_to_dict(v) for k, v in profiles.items()},
        "clusters": {k: cluster_dict(v) for k, v in cl.items()},
        "walk": walk_raw,
        "near_one": NEAR_ONE,
    }
    (OUT / "inputs.json").write_text(json.dumps(inputs, indent=1, sort_keys=True))

    write_jsonl_gz(OUT / "naive.jsonl.gz", gen_naive())
    write_jsonl_gz(OUT / "recursive.jsonl.gz", gen_recursive())
    write_jsonl_gz(OUT / "greedy.jsonl.gz", gen_greedy())

    mu_of = {"dual": 1.65, "fast": 1.0, "equal_dual": 1.0}
    part_rows = []
    index = []

    def add_schedule(key, sched, verdict=None, extra=None):
        lines = [json.dumps(d.to_dict(), sort_keys=True) for d in sched.decisions]
        blob = ("\n".join(lines) + "\n").encode()
        path = OUT / "schedules" / f"{key}.jsonl.gz"
        path.parent.mkdir(parents=True, exist_ok=True)
        with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as f:
            f.write(blob)
        ent = {"key": key, "file": f"schedules/{key}.jsonl.gz",
               "sha256": hashlib.sha256(blob).hexdigest(), "iterations": sched.iterations,
               "scheme": sched.scheme,
               "partitioned": ds.profile_to_dict(sched.profile)["buckets"]}
        if verdict is not None:
            ent["verdict"] = verdict
        if extra:
            ent.update(extra)
        index.append(ent)
        print(key, len(lines), ent["sha256"][:12], flush=True)

    for pname, prof in profiles.items():
        for cname, cluster in cl.items():
            for bw in (1.0, 0.5, 0.25):
                p = prof if bw == 1.0 else prof.scaled_comm(1.0 / bw)
                cfg = ds.PartitionConfig(partition_size=6_500_000, mu=mu_of[cname])
                key = f"{pname}__{cname}__bw{bw}"
                spec = {"profile": pname, "cluster": cname, "bw_scale": bw,
                        "partition": {"partition_size": 6_500_000, "mu": mu_of[cname]}}
                try:
                    part = ds.partition_buckets(p, cfg)
                    part_rows.append({"key": key, "buckets": ds.profile_to_dict(part)["buckets"]})
                except ds.InfeasiblePartitionError as e:
                    part_rows.append({"key": key, "infeasible": True, "bucket_id": e.bucket_id})
                    continue
                s = ds.deft_schedule(p, cluster, cfg, 200)
                final, v = ds.feedback_loop(p, cluster, cfg, walk, iterations=200)
                verdict = {"preserved": v.preserved, "ratio": v.ratio,
                           "expected_state": v.expected_state, "baseline_state": v.baseline_state,
                           "k_values": list(v.sequence.k_values), "retries": v.retries,
                           "capacity_multiplier": v.capacity_multiplier}
                final_lines = [json.dumps(d.to_dict(), sort_keys=True) for d in final.decisions]
                verdict["final_sha256"] = hashlib.sha256(
                    ("\n".join(final_lines) + "\n").encode()).hexdigest()
                add_schedule(key, s, verdict, {"spec": spec})
                if cname == "dual":
                    s1 = ds.deft_schedule(p, cluster, cfg, 200, single_link=True)
                    add_schedule(key + "__single", s1, None,
                                 {"spec": dict(spec, single_link=True)})

    # uniform profiles straight into the state machine (tests/test_scheduler.py)
    for n in (12, 24, 36, 48):
        p = uniform_profile(n)
        sched = ds.DeftScheduler(p, cl["equal_dual"]).run(200)
        s = ds.Schedule("deft", p, cl["equal_dual"], sched, True, 200)
        add_schedule(f"uniform{n}__equal_dual__raw", s, None,
                     {"spec": {"uniform": n, "cluster": "equal_dual", "raw": True}})
        for mult_steps in (1, 3):
            m = 1.0
            for _ in range(mult_steps):
                m *= 1.1
            sched = ds.DeftScheduler(p, cl["equal_dual"], m).run(200)
            s = ds.Schedule("deft", p, cl["equal_dual"], sched, True, 200)
            add_schedule(f"uniform{n}__equal_dual__raw__m{mult_steps}", s, None,
                         {"spec": {"uniform": n, "cluster": "equal_dual", "raw": True,
                                   "mult_steps": mult_steps}})

    # bucket-size sweep: VGG-19 at 16 / 4 / 1 MB fp32 buckets
    for mb, iters in ((16, 100), (4, 30), (1, 8)):
        ps = mb * 2**20 // 4
        cfg = ds.PartitionConfig(partition_size=ps, mu=1.65)
        s = ds.deft_schedule(profiles["vgg19"], cl["dual"], cfg, iters)
        add_schedule(f"vgg19__dual__ps{mb}MB", s, None,
                     {"spec": {"profile": "vgg19", "cluster": "dual", "bw_scale": 1.0,
                               "partition": {"partition_size": ps, "mu": 1.65},
                               "iterations": iters}})

    # scaled-mode schedule: capacities above 1e7 us, every recursion level live
    big = ds.ModelProfile(
        name="bigwindow",
        buckets=tuple(ds.BucketProfile(i + 1, 10**6, 400_000 + 7919 * i, 700_000 + 104_729 * i,
                                       900_000 + 31_337 * (i * i % 11))
                      for i in range(10)),
        batch_size=32,
    )
    inputs["profiles"]["bigwindow"] = ds.profile_to_dict(big)
    (OUT / "inputs.json").write_text(json.dumps(inputs, indent=1, sort_keys=True))
    for cname in ("dual", "fast"):
        cfg = ds.PartitionConfig(partition_size=6_500_000, mu=mu_of[cname])
        s = ds.deft_schedule(big, cl[cname], cfg, 12)
        add_schedule(f"bigwindow__{cname}", s, None,
                     {"spec": {"profile": "bigwindow", "cluster": cname, "bw_scale": 1.0,
                               "partition": {"partition_size": 6_500_000, "mu": mu_of[cname]},
                               "iterations": 12}})

    # profiles MEASURED on B200s by bench.py --dump-profile (the
    # profiler's JSON is also the input to reference parity).  NVLink comm is tiny
    # next to compute, so comm is also scaled up to drive the merge regimes.
    prof_dir = OUT.parent.parent / "profiles"
    for path in sorted(prof_dir.glob("r01_measured_profile_*.json")):
        doc = json.loads(path.read_text())
        mprof = ds.profile_from_dict(doc["profile"])
        mcl = ds.cluster_from_dict(doc["cluster"])
        tag = path.stem.replace("r01_measured_profile_", "measured_")
        inputs["profiles"][tag] = doc["profile"]
        inputs["clusters"][tag] = doc["cluster"]
        mu = max(l.speed_ratio_to_fast for l in mcl.links)
        for scale in (1.0, 60.0, 200.0):
            p = mprof if scale == 1.0 else mprof.scaled_comm(scale)
            cfg = ds.PartitionConfig(partition_size=6_500_000, mu=mu)
            key = f"{tag}__x{int(scale)}"
            s = ds.deft_schedule(p, mcl, cfg, 100)
            final, v = ds.feedback_loop(p, mcl, cfg, walk, iterations=100)
            final_lines = [json.dumps(d.to_dict(), sort_keys=True) for d in final.decisions]
            verdict = {"preserved": v.preserved, "ratio": v.ratio,
                       "expected_state": v.expected_state, "baseline_state": v.baseline_state,
                       "k_values": list(v.sequence.k_values), "retries": v.retries,
                       "capacity_multiplier": v.capacity_multiplier,
                       "final_sha256": hashlib.sha256(
                           ("\n".join(final_lines) + "\n").encode()).hexdigest()}
            add_schedule(key, s, verdict,
                         {"spec": {"profile": tag, "cluster": tag, "comm_scale": scale,
                                   "partition": {"partition_size": 6_500_000, "mu": mu},
                                   "iterations": 100}})
    (OUT / "inputs.json").write_text(json.dumps(inputs, indent=1, sort_keys=True))

    (OUT / "partition.json").write_text(json.dumps(part_rows, indent=0, sort_keys=True))
    (OUT / "schedules.json").write_text(json.dumps(index, indent=0, sort_keys=True))

    # preserver values (preserver.py:97-192)
    pres = []
    rng = random.Random(9)
    for _ in range(50):
        s = rng.uniform(0.0, 0.5)
        b = rng.randint(1, 4096)
        pres.append({"kind": "next", "s": s, "batch": b, "value": ds.expected_next_state(s, b, walk)})
    for ks in ((1,), (2,), (1, 2), (2, 2, 1), (3,), (4, 1), (1, 1, 2)):
        seq = ds.BatchSequence(k_values=ks, base_batch_size=64)
        ok, ratio, merged, base = ds.check_sequence(seq, walk)
        pres.append({"kind": "check", "k_values": list(ks), "batch": 64, "preserved": ok,
                     "ratio": ratio, "merged": merged, "base": base})
    (OUT / "preserver.json").write_text(json.dumps(pres, indent=0, sort_keys=True))


if __name__ == "__main__":
    main()
