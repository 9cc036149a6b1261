"""Knapsack solvers of the DeFT scheduler (mirrors deftsim/knapsack.py:16-213).

The exact 0/1 subset-sum behind ``naive_knapsack`` / ``recursive_knapsack``
runs on the B200 as the batched bitset kernel ``deft_subset_sum_kernel``
(csrc/subset_sum.cu) reached through the C-ABI (include/deft_b200.h).  The
multi-knapsack greedy is O(n*m) bookkeeping and stays on the host.

Contract with the reference (bit-exact):
  * naive_knapsack: suffix bitsets over items sorted by ascending bucket id,
    best = highest reachable sum <= capacity, include-earliest reconstruction
    (knapsack.py:63-94).  Above ``MAX_EXACT_CAPACITY`` weights are scaled by
    q = ceil(cap/1e7), w' = ceil(w/q), cap' = cap // q (knapsack.py:47-52).
  * recursive_knapsack: level d solves items[d:] at max(0, remain - sum of
    backward_times[1..d]); the shallowest level with the maximal original
    value wins (knapsack.py:97-127).  When every level is exact and the level
    capacities never increase, level 0 always wins (its item set and capacity
    dominate every deeper level), so only level 0 is launched; otherwise all
    levels are solved in ONE batched launch.
"""
from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass
from typing import Callable, Sequence

from .errors import DeftError

MAX_EXACT_CAPACITY = 10_000_000


@dataclass(frozen=True)
class Item:
    """One schedulable bucket communication (knapsack.py:19-28)."""

    bucket_id: int
    weight: int

    def __post_init__(self):
        if self.weight <= 0:
            raise DeftError(f"item {self.bucket_id}: weight must be > 0")


@dataclass(frozen=True)
class KnapsackAssignment:
    """Placement of items into knapsacks (knapsack.py:31-44)."""

    selections: tuple[tuple[int, ...], ...]
    total_value: int
    leftovers: tuple[int, ...]

    def selected_ids(self) -> set[int]:
        return {i for sel in self.selections for i in sel}


# A subset-sum backend takes problems [(weights in ascending-id order, capacity)]
# with capacity >= 1 and non-empty weights, and returns one take-mask per problem
# (list[bool], aligned with the weights).  The product backend is the CUDA kernel;
# tests may swap in the CPU oracle explicitly with ``subset_sum_backend``.
SubsetSumBackend = Callable[[Sequence[tuple[Sequence[int], int]]], list[list[bool]]]
_backend_override: SubsetSumBackend | None = None


def _gpu_backend(problems):
    from . import _native  # imported lazily: loading the .so needs no GPU, solving does
    return _native.subset_sum_solver().solve(problems)


def _solve(problems) -> list[list[bool]]:
    if not problems:
        return []
    fn = _backend_override or _gpu_backend
    return fn(problems)


@contextlib.contextmanager
def subset_sum_backend(fn: SubsetSumBackend):
    """Temporarily route the DP through ``fn`` (used by CPU-only tests to check
    the host logic around the solver; the product path is always the GPU)."""
    global _backend_override
    prev, _backend_override = _backend_override, fn
    try:
        yield
    finally:
        _backend_override = prev


def scaled_weights(weights: Sequence[int], capacity: int) -> tuple[list[int], int]:
    """Host restatement of knapsack.py:47-52 (the kernel applies the same
    double-precision arithmetic on the device)."""
    if capacity <= MAX_EXACT_CAPACITY:
        return list(weights), capacity
    q = math.ceil(capacity / MAX_EXACT_CAPACITY)
    return [math.ceil(w / q) for w in weights], capacity // q


def naive_knapsack(items: list[Item], capacity: int) -> KnapsackAssignment:
    """Exact subset-sum knapsack, include-earliest tie rule (knapsack.py:55-94)."""
    if capacity < 0:
        raise DeftError("capacity must be >= 0")
    ordered = sorted(items, key=lambda it: it.bucket_id)
    ids = tuple(it.bucket_id for it in ordered)
    if not ordered or capacity == 0:
        return KnapsackAssignment(selections=((),), total_value=0, leftovers=ids)
    take = _solve([([it.weight for it in ordered], capacity)])[0]
    chosen = tuple(i for i, t in zip(ids, take) if t)
    return KnapsackAssignment(
        selections=(chosen,),
        total_value=sum(it.weight for it, t in zip(ordered, take) if t),
        leftovers=tuple(i for i, t in zip(ids, take) if not t),
    )


def recursive_level_caps(remain_time: int, backward_times: Sequence[int]) -> list[int]:
    """Capacity of every recursion level (knapsack.py:112-122)."""
    caps, r = [], remain_time
    for d in range(len(backward_times)):
        if d:
            r -= backward_times[d]
        caps.append(max(0, r))
    return caps


def recursive_plan(items: Sequence[Item], remain_time: int,
                   backward_times: Sequence[int]) -> tuple[list[int], list[tuple]]:
    """Which levels must be solved: returns (levels, problems)."""
    caps = recursive_level_caps(remain_time, backward_times)
    monotone = all(caps[d] <= caps[0] for d in range(len(caps)))
    exact = all(c <= MAX_EXACT_CAPACITY for c in caps)
    levels = [0] if (monotone and exact) else list(range(len(items)))
    levels = [d for d in levels if caps[d] > 0]
    problems = []
    for d in levels:
        sub = sorted(items[d:], key=lambda it: it.bucket_id)
        problems.append(([it.weight for it in sub], caps[d]))
    return levels, problems


def recursive_finish(items: Sequence[Item], levels: list[int], problems, takes) -> list[int]:
    """Pick the shallowest level with the largest original value; return its ids
    in ``items`` order (knapsack.py:115-127)."""
    best_val, best_ids = 0, []  # level with value 0 returns [] (cap 0 levels too)
    best_level = None
    for d, (ws, _cap), take in zip(levels, problems, takes):
        sub = sorted(items[d:], key=lambda it: it.bucket_id)
        val = sum(it.weight for it, t in zip(sub, take) if t)
        if best_level is None or val > best_val:
            picked = {it.bucket_id for it, t in zip(sub, take) if t}
            best_val, best_level = val, d
            best_ids = [it.bucket_id for it in items[d:] if it.bucket_id in picked]
    if best_level is None or best_val == 0:
        return []
    return best_ids


def recursive_knapsack(items: list[Item], remain_time: int,
                       backward_times: list[int]) -> list[int]:
    """Drop-or-solve recursion (Alg. 1) over newest-first items (knapsack.py:97-127)."""
    if len(items) != len(backward_times):
        raise DeftError("items and backward_times must be aligned")
    if not items:
        return []
    levels, problems = recursive_plan(items, remain_time, backward_times)
    takes = _solve(problems)
    return recursive_finish(items, levels, problems, takes)


def greedy_multi_knapsack(items: list[Item], capacities: list[int]) -> KnapsackAssignment:
    """Smallest knapsack first, heaviest item first, first fit
    (knapsack.py:130-159).  ``selections[k]`` is in placement order."""
    if any(c < 0 for c in capacities):
        raise DeftError("capacities must be >= 0")
    ranked = sorted(items, key=lambda it: (-it.weight, it.bucket_id))
    placed: list[list[int]] = [[] for _ in capacities]
    taken: set[int] = set()
    value = 0
    for k in sorted(range(len(capacities)), key=lambda j: (capacities[j], j)):
        room = capacities[k]
        for it in ranked:
            if it.weight <= room and it.bucket_id not in taken:
                placed[k].append(it.bucket_id)
                taken.add(it.bucket_id)
                room -= it.weight
                value += it.weight
    left = tuple(sorted(it.bucket_id for it in items if it.bucket_id not in taken))
    return KnapsackAssignment(selections=tuple(tuple(p) for p in placed),
                              total_value=value, leftovers=left)


def brute_force_multi_knapsack(items: list[Item], capacities: list[int]) -> KnapsackAssignment:
    """Exhaustive multi-knapsack optimum for tests (knapsack.py:162-213).
    Among optimal assignments the first one met in depth-first order (item in
    knapsack 0, 1, ..., then skipped) wins."""
    if len(items) > 20:
        raise DeftError("brute force guard: at most 20 items")
    if any(c < 0 for c in capacities):
        raise DeftError("capacities must be >= 0")
    ordered = sorted(items, key=lambda it: it.bucket_id)
    n, m = len(ordered), len(capacities)
    tail = [0] * (n + 1)
    for i in range(n - 1, -1, -1):
        tail[i] = tail[i + 1] + ordered[i].weight
    best = [-1, []]
    where = [-1] * n
    rooms = list(capacities)

    def walk(i: int, value: int):
        if value + tail[i] <= best[0]:
            return
        if i == n:
            best[0], best[1] = value, list(where)
            return
        w = ordered[i].weight
        for k in range(m):
            if rooms[k] >= w:
                rooms[k] -= w
                where[i] = k
                walk(i + 1, value + w)
                rooms[k] += w
        where[i] = -1
        walk(i + 1, value)

    walk(0, 0)
    sels = [[] for _ in range(m)]
    left = []
    for i, it in enumerate(ordered):
        k = best[1][i] if i < len(best[1]) else -1
        (sels[k] if k >= 0 else left).append(it.bucket_id)
    return KnapsackAssignment(selections=tuple(tuple(s) for s in sels),
                              total_value=max(best[0], 0), leftovers=tuple(left))
