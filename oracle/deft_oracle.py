"""ORACLE -- test infrastructure only.

Independent CPU restatement of the reference's DeFT scheduling path, used by
tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs as the checker.  The product package never imports
this module.  Parity of this restatement is pinned against the golden streams
produced by running the reference itself (tests/golden/make_golden.py).

Every function cites the reference (paths relative to
/root/reference/pkg/src/deftsim).  Profiles are plain dicts/tuples here, on
purpose, so nothing is shared with the product's dataclasses.
"""
from __future__ import annotations

import ctypes
import json
import math
from pathlib import Path

import numpy as np

MAX_EXACT = 10_000_000  # knapsack.py:16
_LIB = None
_LIB_PATH = Path(__file__).resolve().parent / "_build" / "liboracle.so"


def _lib():
    global _LIB
    if _LIB is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(f"{_LIB_PATH} missing: run `make -C oracle`")
        L = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.POINTER
        L.oracle_subset_sum_batch.restype = ctypes.c_int32
        L.oracle_subset_sum_batch.argtypes = [ctypes.c_int32, P(ctypes.c_int32),
                                              P(ctypes.c_int64), P(ctypes.c_int64),
                                              P(ctypes.c_uint8), P(ctypes.c_int64)]
        _LIB = L
    return _LIB


# ---------------------------------------------------------------- subset sum

def subset_sum_py(weights, cap):
    """Pure-Python big-int DP (knapsack.py:70-88) -- small cases only."""
    n = len(weights)
    if n == 0 or cap <= 0:
        return [False] * n, 0
    if cap > MAX_EXACT:
        q = math.ceil(cap / MAX_EXACT)
        weights, cap = [math.ceil(w / q) for w in weights], cap // q
    mask = (1 << (cap + 1)) - 1
    rows = [0] * (n + 1)
    rows[n] = 1
    for i in range(n - 1, -1, -1):
        rows[i] = (rows[i + 1] | (rows[i + 1] << weights[i])) & mask
    best = rows[0].bit_length() - 1
    t, take = best, []
    for i in range(n):
        ok = weights[i] <= t and (rows[i + 1] >> (t - weights[i])) & 1 == 1
        take.append(bool(ok))
        if ok:
            t -= weights[i]
    return take, best


def subset_sum_c_batch(problems):
    """C restatement (oracle/subset_sum.c), batched: [(weights asc id, cap)] -> takes."""
    if not problems:
        return []
    n = np.array([len(w) for w, _ in problems], dtype=np.int32)
    caps = np.array([c for _, c in problems], dtype=np.int64)
    ws = np.array([x for w, _ in problems for x in w], dtype=np.int64)
    take = np.zeros(max(1, int(n.sum())), dtype=np.uint8)
    best = np.zeros(len(problems), dtype=np.int64)
    P = ctypes.POINTER
    rc = _lib().oracle_subset_sum_batch(len(problems), n.ctypes.data_as(P(ctypes.c_int32)),
                                        ws.ctypes.data_as(P(ctypes.c_int64)),
                                        caps.ctypes.data_as(P(ctypes.c_int64)),
                                        take.ctypes.data_as(P(ctypes.c_uint8)),
                                        best.ctypes.data_as(P(ctypes.c_int64)))
    if rc != 0:
        raise MemoryError("oracle subset-sum ran out of memory")
    out, pos = [], 0
    for k in n.tolist():
        out.append([bool(x) for x in take[pos:pos + k]])
        pos += k
    return out


def naive(pairs, cap, dp=None):
    """naive_knapsack (knapsack.py:55-94) over (id, weight) pairs.
    Returns (chosen ids asc, value, leftovers asc)."""
    if cap < 0:
        raise ValueError("capacity must be >= 0")
    pairs = sorted(pairs)
    ids = [i for i, _ in pairs]
    if not pairs or cap == 0:
        return [], 0, ids
    take = (dp or subset_sum_c_batch)([([w for _, w in pairs], cap)])[0]
    chosen = [i for i, t in zip(ids, take) if t]
    val = sum(w for (_, w), t in zip(pairs, take) if t)
    return chosen, val, [i for i, t in zip(ids, take) if not t]


def recursive(pairs_desc, remain, bwd, dp=None):
    """recursive_knapsack (knapsack.py:97-127), every level solved."""
    n = len(pairs_desc)
    caps, r = [], remain
    for d in range(n):
        if d:
            r -= bwd[d]
        caps.append(max(0, r))
    levels = [sorted(pairs_desc[d:]) for d in range(n)]
    live = [d for d in range(n) if caps[d] > 0]
    takes = dict(zip(live, (dp or subset_sum_c_batch)(
        [([w for _, w in levels[d]], caps[d]) for d in live])))
    best_v, best_order = None, []
    for d in range(n):
        take = takes.get(d, [False] * len(levels[d]))
        val = sum(w for (_, w), t in zip(levels[d], take) if t)
        if best_v is None or val > best_v:
            pick = {i for (i, _), t in zip(levels[d], take) if t}
            best_v, best_order = val, [i for i, _ in pairs_desc[d:] if i in pick]
    return best_order


def greedy(pairs, caps):
    """greedy_multi_knapsack (knapsack.py:130-159): (selections, value, leftovers)."""
    ranked = sorted(pairs, key=lambda p: (-p[1], p[0]))
    sels = [[] for _ in caps]
    used, value = set(), 0
    for k in sorted(range(len(caps)), key=lambda j: (caps[j], j)):
        room = caps[k]
        for i, w in ranked:
            if i not in used and w <= room:
                used.add(i)
                sels[k].append(i)
                room -= w
                value += w
    return sels, value, sorted(i for i, _ in pairs if i not in used)


# ---------------------------------------------------------------- partition

def partition(buckets, total_fwd, partition_size, mu):
    """partition_buckets (partition.py:67-120) over dict buckets."""
    bound = total_fwd / mu
    out = []
    for b in buckets:
        pc, comm = b["param_count"], b["comm_fast_us"]
        parts = math.ceil(pc / partition_size) if pc > partition_size else 1
        if comm / parts >= bound:
            parts = max(parts, math.ceil(comm / bound))
        while parts <= pc and math.ceil(comm / parts) >= bound:
            parts += 1
        if parts > pc:
            raise ValueError(f"infeasible bucket {b['id']}")
        if parts == 1:
            out.append(dict(b))
            continue
        parts = max(1, min(parts, pc, comm))

        def sp(v):
            q, r = divmod(v, parts)
            return [q + (1 if i < r else 0) for i in range(parts)]
        cols = [sp(b[k]) for k in ("param_count", "forward_us", "backward_us", "comm_fast_us")]
        for p, f, w, c in zip(*cols):
            out.append({"param_count": p, "forward_us": f, "backward_us": w, "comm_fast_us": c})
    for i, b in enumerate(out, 1):
        if b["comm_fast_us"] >= bound:
            raise ValueError(f"infeasible piece {i}")
        b["id"] = i
    return out


def scaled_comm(buckets, factor):
    """ModelProfile.scaled_comm (profiles.py:134-152)."""
    return [dict(b, comm_fast_us=max(1, round(b["comm_fast_us"] * factor))) for b in buckets]


# ---------------------------------------------------------------- state machine

def schedule(buckets, ratios, names, iterations, mult=1.0, dp=None):
    """DeftScheduler.run (scheduler.py:159-342) -> list of decision dicts in the
    exact Schedule.dump_jsonl schema (scheduler.py:82-96)."""
    comm = {b["id"]: b["comm_fast_us"] for b in buckets}
    bwd_t = {b["id"]: b["backward_us"] for b in buckets}
    all_ids = [b["id"] for b in buckets]
    fsum = sum(b["forward_us"] for b in buckets)
    bsum = sum(b["backward_us"] for b in buckets)
    fcaps = [round(r * fsum * mult) for r in ratios]
    bcaps = [round(r * bsum * mult) for r in ratios]
    cur = []             # current queue ids
    cur_group = None     # [origins, k, remaining set]
    fut = None           # [origins, k] -- future queue holds every bucket id
    pending = []
    out = []

    def room_pick(caps, loads, cands):
        return max(cands, key=lambda j: (caps[j] - loads[j], -j))

    def drop(ids):
        nonlocal cur, cur_group
        s = set(ids)
        cur = [i for i in cur if i not in s]
        if cur_group is not None:
            cur_group[2] -= s
            if not cur_group[2]:
                pending.append(cur_group)
                cur_group = None

    def store_or_merge(t):
        nonlocal fut
        if fut is not None:
            fut[0] = fut[0] + [t]
            fut[1] += 1
            return list(all_ids)
        fut = [[t], 1]
        return []

    for t in range(iterations):
        sels, _, _ = greedy([(i, comm[i]) for i in cur], fcaps)
        drop([i for s in sels for i in s])
        out.append({"iteration": t, "stage": "forward",
                    "forward_plan": {n: list(s) for n, s in zip(names, sels)},
                    "backward_plan": {}, "fresh_ids": [], "merged": [], "update_events": [],
                    "update_performed": False, "case_taken": "CASE1"})
        caps = bcaps
        dual = sum(caps)
        plan = [[] for _ in caps]
        loads = [0] * len(caps)
        fresh = []
        backlog = sum(comm[i] for i in cur)
        remain = None
        if cur and backlog > dual:
            case = "CASE2"
            sels, _, _ = greedy([(i, comm[i]) for i in cur], caps)
            for k, s in enumerate(sels):
                plan[k] += s
                loads[k] += sum(comm[i] for i in s)
            drop([i for s in sels for i in s])
            merged = store_or_merge(t)
        elif cur:
            case = "CASE3"
            for i in sorted(cur, key=lambda i: (-comm[i], i)):
                k = room_pick(caps, loads, range(len(caps)))
                plan[k].append(i)
                loads[k] += comm[i]
            drop(list(cur))
            merged = store_or_merge(t)
            remain = max(0, dual - backlog)
        else:
            case = "CASE4"
            merged = store_or_merge(t)
            remain = dual
        if remain is not None and fut is not None:
            desc = sorted(all_ids, reverse=True)
            order = recursive([(i, comm[i]) for i in desc], remain, [bwd_t[i] for i in desc], dp)
            for i in order:
                fits = [j for j in range(len(caps)) if caps[j] - loads[j] >= comm[i]]
                k = room_pick(caps, loads, fits or range(len(caps)))
                plan[k].append(i)
                loads[k] += comm[i]
            fresh = sorted(order)
            left = [i for i in desc if i not in set(order)]
            grp = [fut[0], fut[1], set(left)]
            fut = None
            if left:
                cur, cur_group = sorted(left), grp
            else:
                pending.append(grp)
        events = [{"origins": list(g[0]), "merge_count": g[1]} for g in pending]
        pending = []
        out.append({"iteration": t, "stage": "backward", "forward_plan": {},
                    "backward_plan": {n: list(p) for n, p in zip(names, plan)},
                    "fresh_ids": fresh, "merged": merged, "update_events": events,
                    "update_performed": bool(events), "case_taken": case})
    return out


def jsonl(decisions) -> str:
    return "".join(json.dumps(d, sort_keys=True) + "\n" for d in decisions)


# ---------------------------------------------------------------- preserver

def expected_next(s, batch, w):
    """preserver.py:97-112 (same evaluation order)."""
    m = s - w["s_star"] - w["eta"] * w["mu_t"]
    v = w["eta"] * w["sigma_t"] / math.sqrt(batch)
    a = m / v
    inner = m * math.erf(a / math.sqrt(2.0))
    tail = v * math.sqrt(2.0 / math.pi) * math.exp(-0.5 * a * a)
    return inner + tail + w["s_star"]


def check(ks, batch, w):
    """check_sequence (preserver.py:182-192)."""
    s = w["s0"]
    for k in ks:
        s = expected_next(s, k * batch, w)
    b = w["s0"]
    for _ in range(sum(ks)):
        b = expected_next(b, batch, w)
    denom = s - w["s_star"]
    ratio = 1.0 if denom <= 0 else (b - w["s_star"]) / denom
    return abs(ratio - 1.0) <= w["epsilon"], ratio, s, b


def period(ks):
    """extract_batch_sequence's tail-period search (preserver.py:153-168)."""
    n = len(ks)
    for p in range(1, n // 2 + 1):
        pat = ks[n - p:]
        reps, end = 0, n
        while end >= p and ks[end - p:end] == pat:
            reps += 1
            end -= p
        if reps >= 2:
            return pat
    if n == 1:
        return ks
    raise ValueError("non-steady")


def update_schedule(decisions):
    """(iteration t, [(origins, merge_count)]) for every backward decision that
    reports update events: the input of the delayed-SGD oracle."""
    return [(d["iteration"], [(tuple(u["origins"]), u["merge_count"]) for u in d["update_events"]])
            for d in decisions if d["stage"] == "backward" and d["update_events"]]
