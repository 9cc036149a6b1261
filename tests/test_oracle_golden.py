"""Pin the oracle (oracle/) against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""
import hashlib
import json

import pytest

from conftest import GOLDEN, golden_schedule_text, read_jsonl_gz, spec_inputs
from oracle import deft_oracle as O


def test_c_dp_matches_reference_naive():
    rows = read_jsonl_gz("naive.jsonl.gz")
    assert len(rows) > 800
    for r in rows:
        chosen, val, left = O.naive(list(zip(r["ids"], r["weights"])), r["cap"])
        assert chosen == r["selection"], r
        assert val == r["value"]
        assert left == r["leftovers"]


def test_python_dp_matches_c_dp_small():
    rows = [r for r in read_jsonl_gz("naive.jsonl.gz") if r["cap"] <= 200_000 and r["weights"]]
    for r in rows[:600]:
        pairs = sorted(zip(r["ids"], r["weights"]))
        ws = [w for _, w in pairs]
        take_py, _ = O.subset_sum_py(ws, r["cap"])
        take_c = O.subset_sum_c_batch([(ws, r["cap"])])[0] if r["cap"] > 0 else [False] * len(ws)
        assert take_py == take_c


def test_recursive_matches_reference():
    for r in read_jsonl_gz("recursive.jsonl.gz"):
        got = O.recursive(list(zip(r["ids"], r["weights"])), r["remain"], r["backward"])
        assert got == r["order"], r


def test_greedy_matches_reference():
    for r in read_jsonl_gz("greedy.jsonl.gz"):
        sels, val, left = O.greedy(list(enumerate(r["weights"], 1)), r["caps"])
        assert sels == r["selections"]
        assert val == r["value"]
        assert left == r["leftovers"]


def test_partition_matches_reference(golden_inputs):
    rows = json.loads((GOLDEN / "partition.json").read_text())
    for row in rows:
        pname, cname, bw = row["key"].split("__")
        bw = float(bw[2:])
        prof = golden_inputs["profiles"][pname]
        mu = {"dual": 1.65, "fast": 1.0, "equal_dual": 1.0}[cname]
        b = prof["buckets"] if bw == 1.0 else O.scaled_comm(prof["buckets"], 1.0 / bw)
        fwd = sum(x["forward_us"] for x in b)
        if row.get("infeasible"):
            with pytest.raises(ValueError):
                O.partition(b, fwd, 6_500_000, mu)
            continue
        got = O.partition(b, fwd, 6_500_000, mu)
        assert [{k: x[k] for k in sorted(x)} for x in got] == row["buckets"]


def _oracle_stream(entry, inputs):
    prof, cluster, part, factor, mult, iters = spec_inputs(entry, inputs)
    buckets = prof["buckets"]
    if factor != 1.0:
        buckets = O.scaled_comm(buckets, factor)
    if part is not None:
        buckets = O.partition(buckets, sum(b["forward_us"] for b in buckets),
                              part["partition_size"], part["mu"])
    links = cluster["links"]
    if entry["spec"].get("single_link"):
        links = [l for l in links if l["speed_ratio_to_fast"] == 1.0]
    ratios = [l["speed_ratio_to_fast"] for l in links]
    names = [l["name"] for l in links]
    return O.jsonl(O.schedule(buckets, ratios, names, iters, mult))


def _entries(index, max_buckets):
    return [e for e in index if len(e["partitioned"]) <= max_buckets]


def test_oracle_schedules_match_reference(golden_index, golden_inputs):
    checked = 0
    for e in _entries(golden_index, 60):
        text = _oracle_stream(e, golden_inputs)
        assert hashlib.sha256(text.encode()).hexdigest() == e["sha256"], e["key"]
        assert text == golden_schedule_text(e)
        checked += 1
    assert checked >= 45


def test_preserver_values():
    w = json.loads((GOLDEN / "inputs.json").read_text())["walk"]
    for row in json.loads((GOLDEN / "preserver.json").read_text()):
        if row["kind"] == "next":
            assert O.expected_next(row["s"], row["batch"], w) == row["value"]
        else:
            ok, ratio, merged, base = O.check(row["k_values"], row["batch"], w)
            assert (ok, ratio, merged, base) == (row["preserved"], row["ratio"], row["merged"],
                                                 row["base"])
