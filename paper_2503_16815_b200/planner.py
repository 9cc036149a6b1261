"""Host bookkeeping of the executor, free of any device work.

Turns the decision stream of a ``DeftScheduler`` into per-iteration execution
plans: which gradient slot every transfer reads, which slot this iteration's
gradients accumulate into (store = fresh zeroed slot, merge = the live future
group's slot), and which group updates run in this iteration's backward
(update events of decision (t-1, backward); visible from t+1 = (t-1)+2).
Kept separate from ``executor.py`` so the slot/group invariants can be
checked on CPU over every golden decision stream (tests/test_planner.py).
"""
from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass

from .errors import InternalInvariantError
from .scheduler import DeftScheduler, ScheduleDecision


@dataclass(frozen=True)
class IterPlan:
    t: int
    slot: int                 # gradient slot this iteration accumulates into
    zero: bool                # new group (store): zero the slot first
    fwd: tuple                # (link, slot, bucket index) released at forward start
    bwd: tuple                # ... released at backward start
    fresh: tuple              # (bucket index, ((link, slot), ...)) released at bucket end
    due: tuple                # (slot, merge_count) updates applied per bucket this backward
    freed: tuple              # slots whose group is fully updated after this iteration
    key: tuple                # identifies the device work (CUDA-graph cache key)


class ExecutionPlanner:
    """``lag`` = how many iterations after its decision an update event is applied.
    Delayed schedules (DeFT, visible from t+2): 1 -> during the next backward
    ("end"/"bucket" placement), 2 -> at the start of the iteration it becomes
    visible in ("start" placement).  Synchronous schedules (the wfbp / priority
    baselines, ``delayed_updates=False``, visible from t+1): 0 -> in the same
    backward, 1 -> at the start of the next iteration."""

    def __init__(self, scheduler: DeftScheduler, n_slots: int, lookahead: int = 32,
                 lag: int = 1):
        if lag not in (0, 1, 2):
            raise InternalInvariantError("update lag must be 0, 1 or 2")
        self.scheduler = scheduler
        self.n_slots = n_slots
        self.lookahead = lookahead
        self.lag = lag
        self._event_queue: list[list[tuple[int, int]]] = []
        self._decisions: dict[int, tuple[ScheduleDecision, ScheduleDecision]] = {}
        self._next = 0
        self.decision_log: list[tuple[ScheduleDecision, ScheduleDecision]] = []
        self._slot_of: dict[int, int] = {}
        self._busy = [False] * n_slots

    def decisions(self, t: int) -> tuple[ScheduleDecision, ScheduleDecision]:
        while self._next <= t + self.lookahead:
            k = self._next
            self._decisions[k] = (self.scheduler.schedule_forward(k),
                                  self.scheduler.schedule_backward(k))
            self._next += 1
        if t in self._decisions:
            return self._decisions[t]
        return self.decision_log[t]

    def live_slots(self) -> dict[int, int]:
        return dict(self._slot_of)

    def _alloc(self, uid: int) -> int:
        for cand in range(self.n_slots):
            if not self._busy[cand]:
                self._busy[cand] = True
                self._slot_of[uid] = cand
                return cand
        raise InternalInvariantError(
            f"all {self.n_slots} gradient slots are held by live groups; raise n_slots")

    def take_pending(self) -> tuple[tuple, tuple]:
        """("start" placement) updates that are due at the start of the NEXT
        iteration, handed out early so a caller can make theta^(t) current
        without running iteration t.  Returns (due, freed)."""
        if self.lag == 0 or len(self._event_queue) < self.lag:
            return (), ()
        due_groups = self._event_queue.pop(0)
        due = tuple((self._slot_of[u], k) for u, k in due_groups)
        freed = []
        for u, _ in due_groups:
            s = self._slot_of.pop(u)
            self._busy[s] = False
            freed.append(s)
        self._event_queue.insert(0, [])   # keep the queue's timing for the next plan()
        return due, tuple(freed)

    def plan(self, t: int) -> IterPlan:
        if t != len(self.decision_log):
            raise InternalInvariantError("iterations must be planned in order")
        dF, dB = self.decisions(t)
        self.decision_log.append(self._decisions.pop(t))
        fwd = tuple((tr.link, self._slot_of[tr.group], tr.bucket_id - 1)
                    for tr in dF.exec.transfers)
        uid = dB.exec.grad_group
        if uid is None:
            raise InternalInvariantError("backward decision without a gradient group")
        new = uid not in self._slot_of
        if new and dB.exec.grad_merge:
            raise InternalInvariantError("merge into a group that has no slot")
        if not new and not dB.exec.grad_merge:
            raise InternalInvariantError("store into a group that already has a slot")
        bwd, fresh = [], defaultdict(list)
        for tr in dB.exec.transfers:       # older groups first: their slots exist
            if tr.group != uid:
                bwd.append((tr.link, self._slot_of[tr.group], tr.bucket_id - 1))
        slot = self._slot_of[uid] if not new else self._alloc(uid)
        for tr in dB.exec.transfers:
            if tr.group == uid:
                if tr.fresh:
                    fresh[tr.bucket_id - 1].append((tr.link, slot))
                else:
                    bwd.append((tr.link, slot, tr.bucket_id - 1))
        # groups reported by decision (t-lag, backward) are updated in this iteration
        self._event_queue.append([(u, k) for u, k, _ in dB.exec.updates])
        due_groups = self._event_queue.pop(0) if len(self._event_queue) > self.lag else []
        due = tuple((self._slot_of[u], k) for u, k in due_groups)
        freed = []
        for u, _ in due_groups:
            s = self._slot_of.pop(u)
            self._busy[s] = False
            freed.append(s)
        fresh_t = tuple(sorted((b, tuple(v)) for b, v in fresh.items()))
        key = (fwd, slot, new, tuple(bwd), fresh_t, due)
        return IterPlan(t, slot, new, fwd, tuple(bwd), fresh_t, due, tuple(freed), key)


def start_groups(bucket_sizes: list[int], max_groups: int) -> list[list[int]]:
    """"start" placement: buckets in forward order (input side = last index
    first) coalesced into at most `max_groups` consecutive update launches -- a
    small first group (~1/(4*max_groups) of the parameters: the forward's first
    modules wait for it), then groups of similar size.  Returns bucket indices."""
    order = list(range(len(bucket_sizes) - 1, -1, -1))
    n_groups = max(1, min(max_groups, len(order)))
    total = sum(bucket_sizes)
    first = total / (4 * n_groups)
    step = (total - first) / max(1, n_groups - 1)
    groups, cur, acc = [], [], 0
    for b in order:
        size = bucket_sizes[b]
        target = first + step * len(groups)
        if (cur and len(groups) < n_groups - 1 and acc + size > target
                and acc + size - target > target - acc):
            # b would overshoot the target by more than it fills: the modules
            # before it must not wait for its (large) update -- close first
            groups.append(cur)
            cur = []
            target = first + step * len(groups)
        cur.append(b)
        acc += size
        if acc >= target and len(groups) < n_groups - 1:
            groups.append(cur)
            cur = []
    if cur:
        groups.append(cur)
    return groups


def release_runs(transfers) -> list[tuple[int, int, list[int]]]:
    """Transfers released together, as (link, slot, bucket) in plan order ->
    one (link, slot, [buckets]) launch per consecutive same-slot run on each
    link; per-link order is kept (a link serves its transfers in plan order,
    simulator.py:107-129)."""
    out: list[tuple[int, int, list[int]]] = []
    open_run: dict[int, tuple[int, int, list[int]]] = {}
    for link, slot, bidx in transfers:
        cur = open_run.get(link)
        if cur is None or cur[1] != slot:
            cur = (link, slot, [])
            open_run[link] = cur
            out.append(cur)
        cur[2].append(bidx)
    return out


def start_groups_timed(bucket_sizes: list[int], forward_us: list[float],
                       update_us_per_elem: float, launch_us: float,
                       max_groups: int, report: dict | None = None) -> list[list[int]]:
    """"start" placement from the measured profile: the fewest update launches
    such that each group's update (run back to back on the update stream,
    `launch_us` + size x `update_us_per_elem` each) completes before the forward
    reaches the group's first bucket (forward order = input side first; bucket
    i's forward starts after the forward time of the buckets before it).  The
    first group is the input-side bucket alone (the forward waits for it
    whatever its size).  A bucket that cannot be ready in time starts its own
    group.  Returns bucket indices, like `start_groups`."""
    order = list(range(len(bucket_sizes) - 1, -1, -1))
    feasible = True
    if not order:
        return []
    if max_groups <= 1:
        if report is not None:
            report["feasible"] = len(order) == 1
        return [order]
    arrive, t = [], 0.0
    for b in order:
        arrive.append(t)
        t += forward_us[b]
    groups = [[order[0]]]
    done = launch_us + bucket_sizes[order[0]] * update_us_per_elem
    i = 1
    while i < len(order):
        j, size = i, 0
        # extend while the group's completion precedes the forward's arrival at
        # its first bucket (the binding one: arrival times only grow)
        while j < len(order):
            cand = done + launch_us + (size + bucket_sizes[order[j]]) * update_us_per_elem
            if j > i and cand > arrive[i]:
                break
            size += bucket_sizes[order[j]]
            j += 1
            if cand > arrive[i]:          # even alone it is late: keep it alone
                feasible = False
                break
        if len(groups) >= max_groups - 1 and j < len(order):  # launch cap: the rest
            j = len(order)                                     # in one group
            size = sum(bucket_sizes[order[k]] for k in range(i, j))
            feasible = feasible and done + launch_us + size * update_us_per_elem <= arrive[i]
        groups.append(order[i:j])
        done += launch_us + size * update_us_per_elem
        i = j
    if report is not None:
        report["feasible"] = feasible   # no forward wait predicted after the first group
    return groups


class LinkQueueModel:
    """Which of an iteration's fresh transfers the backward can hide, under
    CUDA-graph execution (every side stream joins the compute stream at the end
    of the iteration).  Each link is a FIFO (simulator.py:107-129) serving a
    transfer for its profiled time (comm_fast_us x the link's speed ratio,
    profiles.py:64-80); a bucket's transfers are released when its backward ends
    (simulator.py:184-196: release = cumulative backward time, output side
    first).  A release whose predicted completion lies past the backward's end
    would be exposed at the join: with delayed updates (lag 2) it is needed an
    iteration later at the earliest, so it is deferred to the start of the next
    iteration (executor ``_buckets_ready``) instead of extending this one.

    ``admit`` is called in release order; deferred transfers do not occupy the
    link in this iteration's model."""

    def __init__(self, backward_us: list[float], comm_fast_us: list[float],
                 link_ratios: list[float], slack: float = 1.0):
        self.release_us = []
        t = 0.0
        for b in backward_us:
            t += b
            self.release_us.append(t)
        self.end_us = t
        self.comm = [[c * r * slack for r in link_ratios] for c in comm_fast_us]
        self.busy = [0.0] * len(link_ratios)

    def reset(self):
        self.busy = [0.0] * len(self.busy)

    def admit(self, link: int, bidxs, ready: list[int]) -> bool:
        """True: issue now (the link drains it before the backward ends); False:
        defer.  `ready` = the buckets whose backward end released it."""
        t = max(self.release_us[b] for b in ready)
        done = max(self.busy[link], t) + sum(self.comm[b][link] for b in bidxs)
        if done > self.end_us:
            return False
        self.busy[link] = done
        return True
