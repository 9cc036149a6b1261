"""K5 front end: run whole DeFT schedules inside one persistent GPU kernel.

``run_schedules`` takes a partitioned profile, a cluster and one capacity
multiplier per instance, launches ``deft_scheduler_kernel`` once (one CTA per
instance, csrc/scheduler_kernel.cu) and decodes its compact records into the
same ``ScheduleDecision`` objects (``to_dict`` schema of scheduler.py:82-96 and
the executor's ``exec`` notes) the host state machine produces.  Stage
capacities are computed here with the reference's float expression and
half-even ``round`` (scheduler.py:121-125), so the kernel is integer-only.
Instances the kernel does not cover (scaled-mode capacities above 1e7 us)
come back as None and are scheduled by the host state machine instead
(which still solves every knapsack on the GPU).
"""
from __future__ import annotations

import numpy as np

from . import _native
from ._native import P, c_i32, c_i64
from .errors import InternalInvariantError
from .profiles import ClusterSpec, ModelProfile
from .scheduler import (CapacityModel, Case, ExecNote, ScheduleDecision, Transfer,
                        UpdateEvent)

_HDR = 7
_CASES = {1: Case.CASE1, 2: Case.CASE2, 3: Case.CASE3, 4: Case.CASE4}


def _decode(rec: np.ndarray, n_used: int, names: list[str], all_ids: tuple[int, ...],
            iterations: int, t0: int = 0) -> list[ScheduleDecision]:
    out: list[ScheduleDecision] = []
    r = rec[:n_used].tolist()
    pos = 0
    L = len(names)
    for t in range(t0, t0 + iterations):
        for expect_stage in (0, 1):
            stage, cas, n_tr, n_ev, merged, grad_uid, grad_merge = r[pos:pos + _HDR]
            pos += _HDR
            if stage != expect_stage:
                raise InternalInvariantError("corrupt scheduler record stream")
            trs = []
            plans: list[list[int]] = [[] for _ in range(L)]
            fresh = set()
            for k in range(n_tr):
                link, bid, grp, fr = r[pos + 4 * k:pos + 4 * k + 4]
                trs.append(Transfer(link, bid, grp, bool(fr)))
                plans[link].append(bid)
                if fr:
                    fresh.add(bid)
            pos += 4 * n_tr
            events, notes = [], []
            for e in range(n_ev):
                uid, first, k = r[pos + 3 * e:pos + 3 * e + 3]
                origins = tuple(range(first, first + k))
                events.append(UpdateEvent(origins, k))
                notes.append((uid, k, origins))
            pos += 3 * n_ev
            plan = {nm: tuple(p) for nm, p in zip(names, plans)}
            if stage == 0:
                out.append(ScheduleDecision(
                    iteration=t, stage="forward", forward_plan=plan, backward_plan={},
                    fresh_ids=frozenset(), merged=(), update_events=(), case_taken=Case.CASE1,
                    exec=ExecNote(transfers=tuple(trs))))
            else:
                out.append(ScheduleDecision(
                    iteration=t, stage="backward", forward_plan={}, backward_plan=plan,
                    fresh_ids=frozenset(fresh), merged=all_ids if merged else (),
                    update_events=tuple(events), case_taken=_CASES[cas],
                    exec=ExecNote(transfers=tuple(trs), grad_group=grad_uid,
                                  grad_merge=bool(grad_merge), updates=tuple(notes))))
    return out


class KernelSchedule:
    """The records of one scheduler instance; decoded on demand (the feedback loop
    only needs the merge counts of most attempts)."""

    def __init__(self, rec: np.ndarray, used: int, names, all_ids, iterations: int):
        self._rec = rec[:used].copy()
        self._names, self._all_ids, self._iterations = names, all_ids, iterations
        self._decoded: list[ScheduleDecision] | None = None

    def merge_counts(self) -> list[int]:
        """merge_count of every update event, in stream order (preserver.py:129-134)."""
        r = self._rec
        ks, pos = [], 0
        for _ in range(2 * self._iterations):
            n_tr, n_ev = int(r[pos + 2]), int(r[pos + 3])
            pos += _HDR + 4 * n_tr
            for e in range(n_ev):
                ks.append(int(r[pos + 3 * e + 2]))
            pos += 3 * n_ev
        return ks

    def decisions(self) -> list[ScheduleDecision]:
        if self._decoded is None:
            self._decoded = _decode(self._rec, len(self._rec), self._names, self._all_ids,
                                    self._iterations)
        return self._decoded


def run_schedules(profile: ModelProfile, cluster: ClusterSpec, multipliers: list[float],
                  iterations: int, schedulers=None) -> list[list[ScheduleDecision] | None]:
    """One persistent launch for every multiplier; decoded decision lists, None for
    unsupported instances."""
    return [None if k is None else k.decisions()
            for k in run_schedules_lazy(profile, cluster, multipliers, iterations, schedulers)]


def run_schedules_lazy(profile: ModelProfile, cluster: ClusterSpec, multipliers: list[float],
                       iterations: int, schedulers=None) -> list[KernelSchedule | None]:
    """One persistent launch for every multiplier; None for unsupported instances.
    ``schedulers``: the DeftScheduler of every instance (the caller's
    configuration objects, as the reference builds one per attempt); their
    capacity models are used instead of rebuilding them from the multipliers."""
    solver = _native.subset_sum_solver()
    n = profile.n_buckets
    L = len(cluster.links)
    inst = len(multipliers)
    comm = np.array([b.comm_fast_us for b in profile.buckets], dtype=np.int64)
    bwd = np.array([b.backward_us for b in profile.buckets], dtype=np.int64)
    fc, bc = [], []
    for i, m in enumerate(multipliers):
        cm = (schedulers[i].caps if schedulers is not None else
              CapacityModel.from_profile(profile, cluster, m))
        fc.extend(cm.stage_capacities("forward"))
        bc.extend(cm.stage_capacities("backward"))
    fcaps = np.array(fc, dtype=np.int64)
    bcaps = np.array(bc, dtype=np.int64)
    stride = iterations * 2 * (_HDR + 8 * n + 12) + 16
    out = np.zeros(inst * stride, dtype=np.int32)
    used = np.zeros(inst, dtype=np.int64)
    status = np.zeros(inst, dtype=np.int32)
    st = _native.lib().deft_solver_schedule(
        solver._h, inst, n, L, iterations, comm.ctypes.data_as(P(c_i64)),
        bwd.ctypes.data_as(P(c_i64)), fcaps.ctypes.data_as(P(c_i64)),
        bcaps.ctypes.data_as(P(c_i64)), out.ctypes.data_as(P(c_i32)), stride,
        used.ctypes.data_as(P(c_i64)), status.ctypes.data_as(P(c_i32)))
    _native.check(st, "deft_solver_schedule")
    solver.kernel_ms += float(_native.lib().deft_solver_last_kernel_ms(solver._h))
    names = [l.name for l in cluster.links]
    all_ids = tuple(b.id for b in profile.buckets)
    res: list[KernelSchedule | None] = []
    for i in range(inst):
        if status[i] == -4:
            res.append(None)
            continue
        if status[i] == -6:
            raise InternalInvariantError("insufficient capacity yet queue drained")
        if status[i] != 0:
            raise InternalInvariantError(f"scheduler kernel status {status[i]}")
        res.append(KernelSchedule(out[i * stride:(i + 1) * stride], int(used[i]), names,
                                  all_ids, iterations))
    return res


class KernelScheduler:
    """``DeftScheduler``'s stage API (schedule_forward / schedule_backward, called in
    order) backed by K5: the decisions are produced on the GPU `chunk` iterations
    at a time, the scheduler state carried between chunks inside the kernel's
    carry records.  Used by the executor for unbounded training runs."""

    def __init__(self, profile: ModelProfile, cluster: ClusterSpec,
                 capacity_multiplier: float = 1.0, chunk: int = 256):
        self.profile, self.cluster, self.chunk = profile, cluster, chunk
        cm = CapacityModel.from_profile(profile, cluster, capacity_multiplier)
        self._fcaps = np.array(cm.stage_capacities("forward"), dtype=np.int64)
        self._bcaps = np.array(cm.stage_capacities("backward"), dtype=np.int64)
        self._comm = np.array([b.comm_fast_us for b in profile.buckets], dtype=np.int64)
        self._bwd = np.array([b.backward_us for b in profile.buckets], dtype=np.int64)
        self._names = [l.name for l in cluster.links]
        self._ids = tuple(b.id for b in profile.buckets)
        self._carry = None
        self._next_t = 0
        self._ready: dict[tuple[int, str], ScheduleDecision] = {}
        self.chunks = 0

    @staticmethod
    def supported(profile: ModelProfile, cluster: ClusterSpec, mult: float = 1.0) -> bool:
        cm = CapacityModel.from_profile(profile, cluster, mult)
        return (sum(cm.stage_capacities("backward")) <= 10_000_000 and profile.n_buckets <= 1024
                and len(cluster.links) <= 4)

    def _fetch(self):
        solver = _native.subset_sum_solver()
        n, L, T, t0 = len(self._ids), len(self._names), self.chunk, self._next_t
        stride = T * 2 * (_HDR + 8 * n + 12) + 16
        out = np.zeros(stride, dtype=np.int32)
        used = np.zeros(1, dtype=np.int64)
        status = np.zeros(1, dtype=np.int32)
        cbytes = int(_native.lib().deft_sched_carry_bytes())
        carry_out = np.zeros(cbytes, dtype=np.uint8)
        cin = None if self._carry is None else self._carry.ctypes.data_as(_native.c_vp)
        st = _native.lib().deft_solver_schedule_chunk(
            solver._h, 1, n, L, t0, T, self._comm.ctypes.data_as(P(c_i64)),
            self._bwd.ctypes.data_as(P(c_i64)), self._fcaps.ctypes.data_as(P(c_i64)),
            self._bcaps.ctypes.data_as(P(c_i64)), cin, carry_out.ctypes.data_as(_native.c_vp),
            out.ctypes.data_as(P(c_i32)), stride, used.ctypes.data_as(P(c_i64)),
            status.ctypes.data_as(P(c_i32)))
        _native.check(st, "deft_solver_schedule_chunk")
        if status[0] != 0:
            raise InternalInvariantError(f"scheduler kernel status {status[0]}")
        for d in _decode(out, int(used[0]), self._names, self._ids, T, t0):
            self._ready[(d.iteration, d.stage)] = d
        self._carry = carry_out
        self._next_t += T
        self.chunks += 1

    def _take(self, iteration: int, stage: str) -> ScheduleDecision:
        while iteration >= self._next_t:
            self._fetch()
        return self._ready.pop((iteration, stage))

    def schedule_forward(self, iteration: int) -> ScheduleDecision:
        return self._take(iteration, "forward")

    def schedule_backward(self, iteration: int) -> ScheduleDecision:
        return self._take(iteration, "backward")

    def run(self, iterations: int) -> list[ScheduleDecision]:
        out = []
        for k in range(iterations):
            out.append(self.schedule_forward(k))
            out.append(self.schedule_backward(k))
        return out


__all__ = ["run_schedules", "run_schedules_lazy", "KernelSchedule", "KernelScheduler"]
