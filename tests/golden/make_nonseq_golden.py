"""Golden vectors for the non-sequential baseline (scheduler.py:421-472),
produced by RUNNING THE REFERENCE (oracle/_ref, copied by oracle/copy_ref.py):
for the fixture profiles and random profiles, the sha256 of the reference's
decision stream (JSONL, sorted keys), the chosen block structure and the
simulator's total time of the WFBP order (the scoring rule).

python tests/golden/make_nonseq_golden.py  ->  tests/golden/nonsequential.json"""
import hashlib
import json
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.reference import deftsim  # noqa: E402

R = deftsim()
INPUTS = json.loads((ROOT / "tests" / "golden" / "inputs.json").read_text())


def stream_sha(sched):
    text = "".join(json.dumps(d.to_dict(), sort_keys=True) + "\n" for d in sched.decisions)
    return hashlib.sha256(text.encode()).hexdigest()


def main():
    cases = []
    for name in ("resnet101", "vgg19", "gpt2"):
        for ps, su in ((6_500_000, 0), (6_500_000, 100), (3_000_000, 500), (10**12, 0)):
            cases.append({"profile": INPUTS["profiles"][name], "cluster": INPUTS["clusters"]["dual"],
                          "partition_size": ps, "comm_startup_us": su, "iterations": 6})
    rnd = random.Random(20261019)
    for i in range(40):
        n = rnd.randint(1, 14)
        bs = [dict(id=k + 1, param_count=rnd.randint(1, 5_000_000),
                   forward_us=rnd.randint(0, 3000), backward_us=rnd.randint(0, 6000),
                   comm_fast_us=rnd.randint(1, 9000)) for k in range(n)]
        cases.append({"profile": {"name": f"rand{i}", "batch_size": 32, "learning_rate": 0.01,
                                  "buckets": bs, "notes": {}},
                      "cluster": {"links": [{"name": "nccl", "speed_ratio_to_fast": 1.0,
                                             "startup_us": rnd.choice([0, 20, 300])},
                                            {"name": "gloo", "speed_ratio_to_fast": 1.65}]},
                      "partition_size": rnd.choice([10**12, 3_000_000, 1_000_000]),
                      "comm_startup_us": rnd.choice([0, 50, 500]),
                      "iterations": rnd.choice([1, 3, 8, 12])})
    for c in cases:
        prof, cl = R.profile_from_dict(c["profile"]), R.cluster_from_dict(c["cluster"])
        cfg = R.PartitionConfig(partition_size=c["partition_size"],
                                comm_startup_us=c["comm_startup_us"])
        s = R.build_schedule("nonsequential", prof, cl, cfg, c["iterations"])
        c["want"] = {"sha256": stream_sha(s),
                     "blocks": [b.param_count for b in s.profile.buckets],
                     "wfbp_total_us": R.simulate(R.baseline_wfbp(prof, cl, c["iterations"]))
                     .total_time_us}
    out = ROOT / "tests" / "golden" / "nonsequential.json"
    out.write_text(json.dumps(cases, sort_keys=True))
    print(f"{len(cases)} cases -> {out}")


if __name__ == "__main__":
    main()
