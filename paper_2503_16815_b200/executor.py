"""DeftDataParallel: runs a DeFT decision stream on real GPUs.

The reference plays decisions onto a simulated timeline (simulator.py:150-273);
this executor plays them onto CUDA streams with the same release rules
(simulator.py:184-196):

  * forward-plan transfers are released at the forward-stage start;
  * backward-plan transfers of older groups at the backward-stage start;
  * fresh transfers at their own bucket's backward end (a post-accumulate-grad
    hook records the event and launches the reduce on the link's stream).

Channels: link i of the ClusterSpec maps to an NVLink channel (SM P2P or copy
engines); every link owns one CUDA stream, so a link serves its transfers in
release order like the simulator's per-link queue (simulator.py:94-133).

Delayed update (stale-by-k, SURVEY §8c rule 4).  Update events carried by
decision (t, backward) are applied -- per bucket, fused with the parameter
all-gather -- inside bucket b's no-read window of iteration t+1 (after its
backward, before its next forward) and are therefore visible from iteration
t+2 on, deterministically, whatever the communication timing:
    theta^(s) = theta^(s-1) - lr * v,   v = m*v + sum_{o in origins} mean_ranks(g_o) / k
for every event of decision (s-2, backward).  Compute never waits for a
transfer; it only waits, at each forward start, for the (short) update
kernels due at that version -- the zero-stall property of simulator.py:12-14.

The reference's synchronous baseline schedules (``scheme="wfbp"`` /
``"priority"``, scheduler.py:386-418) run on the same machinery with their
update events visible from t+1 (planner lag 0 / 1).

Memory (B200, 180 GB HBM): the flat fp32 parameter buffer (output-side
bucket first, every module parameter is a view into it), a momentum buffer
and ``n_slots`` gradient group slots, all symmetric (CUDA-IPC mapped by every
peer).  Autograd accumulates straight into the slot of the group the schedule
says this iteration's gradients join (store -> zeroed slot, merge -> the live
future group's slot), so merging k iterations is plain gradient accumulation
 with no extra pass.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import torch

from . import _native
from .comm import BucketComm
from .errors import DeftError, InternalInvariantError
from .partition import PartitionConfig, element_ranges, partition_buckets, partition_by_size
from .preserver import WalkParams, feedback_loop
from .profiles import BucketProfile, ClusterSpec, LinkSpec, ModelProfile
from .planner import (ExecutionPlanner, IterPlan, LinkQueueModel, release_runs, start_groups,
                      start_groups_timed)
from .scheduler import (DeftScheduler, OrderScheduler, ScheduleDecision,
                        nonsequential_candidates, priority_order, sync_schedule_time_us,
                        wfbp_order)

SCHEMES = ("deft", "wfbp", "priority", "nonsequential")

# default one-shot threshold (bytes of one bucket's gradients); see DESIGN.md
ONESHOT_DEFAULT_BYTES = 0


def oneshot_limit(cfg_value: int | None) -> int:
    import os
    if cfg_value is not None:
        return int(cfg_value)
    env = os.environ.get("DEFT_ONESHOT_MAX_BYTES")
    return int(env) if env else ONESHOT_DEFAULT_BYTES


@dataclass
class DeftConfig:
    lr: float = 0.1
    momentum: float = 0.9
    partition: PartitionConfig = field(default_factory=PartitionConfig)
    grad_dtype: torch.dtype = torch.float32
    n_slots: int = 6
    autocast_dtype: torch.dtype | None = torch.bfloat16
    walk: WalkParams | None = None          # run the feedback loop when given
    capacity_multiplier: float = 1.0
    lookahead: int = 32                     # decisions generated ahead of execution
    schedule_engine: str = "auto"           # "kernel" (K5 chunks), "host", "auto"
    use_ce_channel: bool = True             # second link = copy engines
    instrument: bool = False                # CUDA events around every native launch
    # capture + replay each distinct iteration shape; "auto" = keep graphs only if
    # warm_up() measures them faster than eager execution
    cuda_graphs: bool | str = "auto"
    # where the delayed update of bucket b runs inside its no-read window
    # ("auto": "end" on one GPU, "start" on several -- measured best):
    # "bucket" = right after b's backward (overlaps the rest of the backward),
    # "end" = after the whole backward (one launch per event at W == 1),
    # "start" = at the start of the iteration it becomes visible in, input-side
    #           bucket first, each bucket's forward waiting only for its own update
    update_placement: str = "auto"
    # CTAs of every update kernel (0 = the comm default; 32 with "start").  With
    # "start" placement a small budget lets the update overlap the forward instead
    # of displacing it.
    update_blocks: int = 0
    start_groups: int = 8                   # max update launches per event with "start"
    # "timed": as few launches as the measured forward can hide (planner.start_groups_timed);
    # "size": a small first group, then similar sizes (planner.start_groups);
    # "auto": timed when it predicts no forward wait, else size
    start_grouping: str = "auto"
    # "deft" (delayed updates) or one of the reference's synchronous baselines on
    # the same kernels (scheduler.py:386-418): "wfbp" (every bucket at its own
    # backward end, measured buckets) / "priority" (partition_by_size blocks,
    # input layer first).  Synchronous: updates of iteration t visible from t+1.
    scheme: str = "deft"
    graph_warmup: int = 2                   # eager iterations before any capture
    # buckets of at most this many gradient bytes sync "one-shot" at W > 1: no
    # reduce-scatter at the transfer point, the update reads every rank's slot
    # (all-reduce + update in one launch, no all-gather).  None = the measured
    # default (DEFT_ONESHOT_MAX_BYTES, else ONESHOT_DEFAULT_BYTES); 0 = never
    oneshot_max_bytes: int | None = None
    # delayed schedules under CUDA graphs (per-iteration joins): fresh transfers
    # that would be exposed at the join start with the next iteration instead.
    # "last" (or True): the backward's last release only; "predicted": also every
    # release the link-queue model (planner.LinkQueueModel, profiled times)
    # predicts would finish after the backward's end; False: none
    defer_tail: bool | str = True


class _Bucket:
    """Bucket `id` owns elements [lo, hi) of the flat parameter / gradient buffers."""

    __slots__ = ("id", "lo", "hi")

    def __init__(self, bid, lo, hi):
        self.id, self.lo, self.hi = bid, lo, hi


class DeftDataParallel:
    """Wraps a module; ``train_step`` runs one DeFT-scheduled iteration."""

    def __init__(self, module: torch.nn.Module, config: DeftConfig | None = None,
                 process_group=None, device: torch.device | None = None):
        self.cfg = config or DeftConfig()
        self.module = module
        self.group = process_group
        dist = torch.distributed
        # a LoopbackRank (loopback.py): W ranks of one process on one GPU
        from .loopback import LoopbackRank
        self.loopback = process_group if isinstance(process_group, LoopbackRank) else None
        if self.loopback is not None:
            self.world, self.rank = self.loopback.world, self.loopback.rank
        else:
            self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
            self.rank = dist.get_rank(process_group) if dist.is_initialized() else 0
        self.device = device or (self.loopback.device if self.loopback is not None else
                                 torch.device("cuda", torch.cuda.current_device()))
        self.placement = self.cfg.update_placement
        if self.placement == "auto":
            self.placement = "end" if self.world == 1 else "start"
        if self.placement not in ("end", "start", "bucket"):
            raise DeftError(f"unknown update placement {self.placement!r}")
        if self.cfg.scheme not in SCHEMES:
            raise DeftError(f"unknown scheme {self.cfg.scheme!r}")
        self.sync = self.cfg.scheme != "deft"
        if self.device.type != "cuda":
            raise DeftError("DeftDataParallel runs on CUDA devices only (no CPU fallback)")
        # DDP order: output-side parameter first (bucket 1 finishes backward first)
        self.params = [p for p in module.parameters() if p.requires_grad][::-1]
        self.numels = [p.numel() for p in self.params]
        self.total = sum(self.numels)
        dtypes = {p.dtype for p in self.params}
        if len(dtypes) != 1 or next(iter(dtypes)) not in (torch.float32, torch.bfloat16):
            raise DeftError(f"parameters must all be fp32 or all bf16, got {dtypes}")
        # gradients (and the symmetric parameter copies) carry the parameter dtype;
        # bf16 models get an fp32 master inside the update kernel
        self.cfg.grad_dtype = next(iter(dtypes))
        if self.loopback is not None:
            self.comm = self.loopback.comm(self.cfg.n_slots, self.total, self.cfg.grad_dtype)
        else:
            self.comm = BucketComm(self.rank, self.world, self.cfg.n_slots, self.total,
                                   self.cfg.grad_dtype, self.device, process_group)
        self.mom = torch.zeros(self.total, dtype=torch.float32, device=self.device)
        self._bind_params()
        if self.loopback is not None:
            # two streams per rank; links, gathers and updates share one in-order
            # comm stream (identical issue order on every rank: loopback.py)
            self.compute_stream = self.loopback.compute_stream
            self.update_stream = self.gather_stream = self.loopback.comm_stream
        else:
            self.compute_stream = torch.cuda.Stream(self.device)
            prio_lo, prio_hi = torch.cuda.Stream.priority_range()
            self.update_stream = torch.cuda.Stream(self.device, priority=prio_hi)
            # store path: bucket gathers run here, off the backward's critical path
            self.gather_stream = torch.cuda.Stream(self.device)
        self.link_streams: list[torch.cuda.Stream] = []
        self.profile: ModelProfile | None = None
        self.schedule_profile: ModelProfile | None = None
        self.cluster: ClusterSpec | None = None
        self.iteration = 0
        self.updates_applied = 0                # update events issued so far
        self._events_t: list[tuple[str, torch.cuda.Event, torch.cuda.Event, int]] = []

    # ------------------------------------------------------------------ setup

    def _bind_params(self):
        """Move every parameter into the symmetric flat buffer (same strides)."""
        flat = self.comm.params
        self.offsets = []
        off = 0
        with torch.no_grad():
            for p in self.params:
                n = p.numel()
                view = flat[off:off + n].as_strided(p.shape, p.stride())
                if not p.is_contiguous(memory_format=torch.contiguous_format) and \
                        not p.is_contiguous(memory_format=torch.channels_last):
                    raise DeftError("parameters must be dense (contiguous or channels_last)")
                view.copy_(p.detach())
                p.data = view
                self.offsets.append(off)
                off += n
            # every rank starts from rank 0's parameters and module buffers
            # (BatchNorm running statistics; like DDP's broadcast_buffers)
            buffers = [b for b in self.module.buffers() if b.is_floating_point()
                       or b.dtype in (torch.int64, torch.int32)]
            if self.loopback is not None:
                self.loopback.broadcast_(f"params", flat)
                for i, b in enumerate(buffers):
                    self.loopback.broadcast_(f"buffer{i}", b)
            elif self.world > 1:
                torch.distributed.broadcast(flat, src=0, group=self.group)
                for b in buffers:
                    if b.device == flat.device:
                        torch.distributed.broadcast(b, src=0, group=self.group)
            if self.comm.master is not None:
                self.comm.master.copy_(flat.float())
        torch.cuda.synchronize(self.device)
        self._grad_views = []
        for s in range(self.cfg.n_slots):
            row = self.comm.grads[s]
            self._grad_views.append([row[o:o + p.numel()].as_strided(p.shape, p.stride())
                                     for o, p in zip(self.offsets, self.params)])
        self._bound_slot = None

    def initial_buckets(self) -> list[tuple[int, int]]:
        """Consecutive output-side-first tensors packed up to partition_size
        parameters (larger tensors alone; partition_buckets splits them)."""
        cap = self.cfg.partition.partition_size
        out, lo, cur = [], 0, 0
        for n in self.numels:
            if cur and cur + n > cap:
                out.append((lo, lo + cur))
                lo, cur = lo + cur, 0
            cur += n
        if cur:
            out.append((lo, lo + cur))
        return out

    # -------------------------------------------------------------- profiling

    def _make_links(self, ce_ratio: float | None) -> ClusterSpec:
        links = [LinkSpec("nvlink_sm", 1.0)]
        self.channel_of_link = [_native.CHANNEL_SM]
        if ce_ratio is not None:
            if ce_ratio >= 1.0:
                links.append(LinkSpec("nvlink_ce", ce_ratio))
                self.channel_of_link.append(_native.CHANNEL_CE)
            else:  # copy engines faster: they become the fast link
                links = [LinkSpec("nvlink_ce", 1.0), LinkSpec("nvlink_sm", 1.0 / ce_ratio)]
                self.channel_of_link = [_native.CHANNEL_CE, _native.CHANNEL_SM]
        return ClusterSpec(links=tuple(links))

    def measure_profile(self, batch, loss_fn: Callable, iters: int = 3, name: str = "model",
                        batch_size: int = 1) -> ModelProfile:
        """CUDA-event timing of forward/backward per initial bucket plus the
        measured comm time of every bucket on each channel -> ModelProfile.
        (B200 replacement of the paper's Nsight profiler.)
        Like the reference's trace reconstruction (trace.py:240-250) every
        per-bucket time is the median_low over the timed iterations, in integer
        us.  ``self.profile_step_us`` keeps the median_low end-to-end
        forward+backward time of the same iterations (the per-bucket times
        partition it)."""
        import statistics
        ranges = self.initial_buckets()
        if self.loopback is not None and self.rank > 0:
            # loopback: rank 0 measured (all ranks' comm included); same numbers
            fwd_us, bwd_us, comm_sm, ce_ratio, step_us = self.loopback.broadcast_obj(
                "profile", None)
        else:
            fwd_us, bwd_us, step_us = self._time_buckets(ranges, batch, loss_fn, iters)
            comm_sm = self._measure_comm(ranges, _native.CHANNEL_SM)
            ce_ratio = None
            if self.world > 1 and self.cfg.use_ce_channel:
                comm_ce = self._measure_comm(ranges, _native.CHANNEL_CE)
                ratios = sorted(c / s for c, s in zip(comm_ce, comm_sm) if s > 0)
                ce_ratio = statistics.median_low(ratios) if ratios else None
            if self.loopback is not None:
                self.loopback.broadcast_obj("profile",
                                            (fwd_us, bwd_us, comm_sm, ce_ratio, step_us))
        if self.world > 1 and self.loopback is None:
            # every rank must plan the SAME schedule: rank 0's numbers win
            obj = [(fwd_us, bwd_us, comm_sm, ce_ratio, step_us)]
            torch.distributed.broadcast_object_list(obj, src=0, group=self.group)
            fwd_us, bwd_us, comm_sm, ce_ratio, step_us = obj[0]
        self.profile_step_us = step_us
        self.comm_us = {"sm": list(comm_sm)}
        buckets = tuple(
            BucketProfile(i + 1, hi - lo, fwd_us[i], bwd_us[i], max(1, comm_sm[i]))
            for i, (lo, hi) in enumerate(ranges))
        self.cluster = self._make_links(ce_ratio)
        self.profile = ModelProfile(name=name, buckets=buckets, batch_size=batch_size,
                                    learning_rate=self.cfg.lr,
                                    notes={"device": torch.cuda.get_device_name(self.device),
                                           "world": self.world})
        return self.profile

    def _time_buckets(self, ranges, batch, loss_fn, iters):
        """Per-bucket forward / backward us (median_low over `iters` timed
        iterations after one warm-up) and the end-to-end fwd+bwd us."""
        import statistics
        owner = self._owner_map(ranges)
        nb = len(ranges)
        per_f: list[list[int]] = [[] for _ in range(nb)]
        per_b: list[list[int]] = [[] for _ in range(nb)]
        per_step: list[int] = []
        module_first = {}
        for m in self.module.modules():
            ps = [p for p in m.parameters(recurse=False) if p.requires_grad]
            if ps:
                module_first[m] = max(max(owner[id(p)]) for p in ps)
        for it in range(iters + 1):
            starts: dict[int, torch.cuda.Event] = {}
            hooks = []

            def pre(mod, _inp):
                b = module_first[mod]
                if b not in starts:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record()
                    starts[b] = e
            for m in module_first:
                hooks.append(m.register_forward_pre_hook(pre))
            done: dict[int, torch.cuda.Event] = {}
            pending = [len([p for p in self.params if b in owner[id(p)]]) for b in range(nb)]

            def acc(p):
                for b in owner[id(p)]:
                    pending[b] -= 1
                    if pending[b] == 0:
                        e = torch.cuda.Event(enable_timing=True)
                        e.record()
                        done[b] = e
            for p in self.params:
                hooks.append(p.register_post_accumulate_grad_hook(acc))
            self._bind_grads(0)
            self.comm.grads[0].zero_()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
            with self._autocast():
                loss = loss_fn(self.module, batch)
            ev1.record()
            loss.backward()
            ev2 = torch.cuda.Event(enable_timing=True)
            ev2.record()
            for h in hooks:
                h.remove()
            torch.cuda.synchronize(self.device)
            if it == 0:
                continue  # warm-up
            # forward: bucket n first; bucket b spans start[b] .. start[b-1]
            us = lambda ms: int(round(ms * 1000.0))  # noqa: E731
            marks = {b: ev0.elapsed_time(starts[b]) for b in starts}
            prev_t = ev0.elapsed_time(ev1)
            f = [0.0] * nb
            for b in range(nb):  # b = 0 is bucket 1 (output side)
                t0 = marks.get(b, prev_t)
                f[b] = max(0.0, prev_t - t0)
                prev_t = min(prev_t, t0)
            f[nb - 1] += max(0.0, prev_t)  # pre-module prologue -> input bucket
            prev_t = ev0.elapsed_time(ev1)
            t_end = ev0.elapsed_time(ev2)
            for b in range(nb):
                t1 = ev0.elapsed_time(done[b]) if b in done else t_end
                per_b[b].append(us(max(0.0, t1 - prev_t)))
                prev_t = max(prev_t, t1)
                per_f[b].append(us(f[b]))
            per_b[nb - 1][-1] += us(max(0.0, t_end - prev_t))   # backward tail -> last bucket
            per_step.append(us(t_end))
        med = statistics.median_low
        return ([max(0, med(x)) for x in per_f], [max(0, med(x)) for x in per_b],
                med(per_step))

    def _owner_map(self, ranges):
        owner = {}
        for p, off in zip(self.params, self.offsets):
            lo, hi = off, off + p.numel()
            owner[id(p)] = [b for b, (a, z) in enumerate(ranges) if a < hi and lo < z]
        return owner

    def _measure_comm(self, ranges, channel, reps: int = 3) -> list[int]:
        """Reduce-scatter time (us, median_low of `reps` after one warm-up) of
        every bucket on one channel.  W = 1: no transfer, 0."""
        import statistics
        if self.world == 1:
            return [0] * len(ranges)
        if self.loopback is not None:
            # every rank's launch, then one synchronize (rank 0 alone would wait
            # for its peers forever); the last-launched rank's time is the one
            # without launch skew
            ranks = self.loopback.lb.ranks
            comms = self.loopback.peers()
            streams = [rk.comm_stream for rk in ranks]
        else:
            comms, streams = [self.comm], [torch.cuda.Stream(self.device)]
        out = []
        torch.cuda.synchronize(self.device)
        for lo, hi in ranges:
            times = []
            for rep in range(reps + 1):
                evs = []
                for c, s in zip(comms, streams):
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(s)
                    c.reduce_scatter(channel, 0, lo, hi - lo, s)
                    b.record(s)
                    evs.append((a, b))
                torch.cuda.synchronize(self.device)
                if rep:
                    times.append(int(round(evs[-1][0].elapsed_time(evs[-1][1]) * 1000.0)))
            out.append(statistics.median_low(times))
        for c in comms:
            c.grads[0].zero_()
        torch.cuda.synchronize(self.device)
        return out

    # ---------------------------------------------------------------- planning

    def plan(self, profile: ModelProfile | None = None, cluster: ClusterSpec | None = None,
             feedback_iterations: int = 200, probe: tuple | None = None,
             _candidate: tuple | None = None):
        """Partition the profile, pick the capacity multiplier (feedback loop when
        walk parameters are configured) and start the incremental scheduler.

        ``scheme="nonsequential"`` (scheduler.py:421-472): the four candidate
        block structures x orders are scored -- with ``probe=(batch, loss_fn)``
        by timing 8 iterations of each on this hardware (parameters, momentum
        and iteration count restored afterwards; the slowest rank's time decides
        on every rank), otherwise with the reference's simulator rules
        (scheduler.sync_schedule_time_us) -- and the fastest is planned."""
        profile = profile or self.profile
        cluster = cluster or self.cluster
        if profile is None or cluster is None:
            raise DeftError("measure_profile() or an explicit profile/cluster is required")
        if self.cfg.scheme == "nonsequential" and _candidate is None:
            cands = nonsequential_candidates(profile, self.cfg.partition)
            if probe is None:
                fast = cluster.fast_link
                scores = [(sync_schedule_time_us(p, fast, order, 8), i)
                          for i, (p, order) in enumerate(cands)]
            else:
                scores = self._probe_candidates(profile, cluster, cands, probe)
            self.nonsequential_scores = sorted(scores)
            return self.plan(profile, cluster, feedback_iterations,
                             _candidate=cands[min(scores)[1]])
        if getattr(self, "_planned", False):
            # re-planning: drop the previous plan's hooks and per-plan caches (a
            # new schedule starts; groups of the old one still in flight are
            # dropped, as unaccounted iterations are in the reference)
            if self._deferred:
                raise DeftError("plan() again with deferred transfers pending: "
                                "call finish() first")
            for h in getattr(self, "_hooks", []):
                h.remove()
            self._hooks = []
        self._groups_cache = None
        self._fwd_wait = {}
        self._deferred = []
        if cluster is not self.cluster:
            self.cluster = cluster
            # measured links carry their channel in the name (_make_links); any
            # other cluster: the fast link is the SM channel, the rest copy engines
            self.channel_of_link = [
                _native.CHANNEL_CE if l.name == "nvlink_ce" else
                _native.CHANNEL_SM if l.name == "nvlink_sm" or l.is_fast else
                _native.CHANNEL_CE for l in cluster.links]
        if self.world > 1 and len(set(self.channel_of_link)) != len(self.channel_of_link):
            # one stream, one barrier set and one staging area per channel: two
            # links on the same channel would interleave their barriers and share
            # the copy-engine staging buffer
            raise DeftError(f"links {[l.name for l in cluster.links]} map to channels "
                            f"{self.channel_of_link}: at most one link per channel "
                            "(nvlink_sm, nvlink_ce)")
        mult = self.cfg.capacity_multiplier
        self.verdict = None
        if self.cfg.walk is not None and not self.sync:
            _, self.verdict = feedback_loop(profile, cluster, self.cfg.partition, self.cfg.walk,
                                            iterations=feedback_iterations)
            mult = self.verdict.capacity_multiplier
        if _candidate is not None:
            part = _candidate[0]
        elif self.cfg.scheme == "wfbp":
            part = profile
        elif self.cfg.scheme == "priority":
            part = partition_by_size(profile, self.cfg.partition.partition_size)
        else:
            part = partition_buckets(profile, self.cfg.partition)
        if part.total_param_count != self.total:
            raise DeftError(f"profile covers {part.total_param_count} parameters, "
                            f"model has {self.total}")
        self.schedule_profile = part
        self.buckets = [_Bucket(b.id, lo, hi) for b, (lo, hi) in
                        zip(part.buckets, element_ranges(part, None))]
        owner = self._owner_map([(b.lo, b.hi) for b in self.buckets])
        self._param_buckets = [owner[id(p)] for p in self.params]
        esz = 2 if self.cfg.grad_dtype == torch.bfloat16 else 4
        lim = oneshot_limit(self.cfg.oneshot_max_bytes)
        self._oneshot = [self.world > 1 and (b.hi - b.lo) * esz <= lim for b in self.buckets]
        self._bucket_nparams = [0] * len(self.buckets)
        self._bucket_params: list[list[int]] = [[] for _ in self.buckets]
        for i, bl in enumerate(self._param_buckets):
            for b in bl:
                self._bucket_nparams[b] += 1
                self._bucket_params[b].append(i)
        self._gather_slot = None
        from .gpu_scheduler import KernelScheduler
        from .scheduler import use_kernel_engine
        self.iteration = 0
        if self.sync:
            order = (list(_candidate[1]) if _candidate is not None else
                     wfbp_order(part) if self.cfg.scheme == "wfbp" else priority_order(part))
            self.scheduler = OrderScheduler(part, cluster.fast_link.name, order,
                                            link=cluster.links.index(cluster.fast_link))
        elif (use_kernel_engine(self.cfg.schedule_engine)
                and KernelScheduler.supported(part, cluster, mult)):
            self.scheduler = KernelScheduler(part, cluster, mult)   # K5, in chunks
        else:
            self.scheduler = DeftScheduler(part, cluster, mult)
        self.capacity_multiplier = mult
        self._update_blocks = self.cfg.update_blocks or (
            32 if self.placement in ("start", "bucket") else 0)
        self.comm.set_update_blocks(self._update_blocks)
        # delayed (DeFT): visible from t+2; synchronous baselines: from t+1
        lag = (1 if self.placement == "start" else 0) if self.sync else \
            (2 if self.placement == "start" else 1)
        self.planner = ExecutionPlanner(self.scheduler, self.cfg.n_slots, self.cfg.lookahead,
                                        lag=lag)
        if self.loopback is not None:
            self.link_streams = [self.loopback.comm_stream for _ in cluster.links]
        else:
            self.link_streams = [torch.cuda.Stream(self.device) for _ in cluster.links]
        # runtime state
        self._slot_free = [None] * self.cfg.n_slots   # event: slot reusable (async mode)
        self._rs_done: dict[tuple[int, int], torch.cuda.Event] = {}
        self._version_ready: torch.cuda.Event | None = None
        self._in_step = False
        # CUDA graphs: iterations run strictly one after another (side streams
        # join the compute stream at the end of each iteration)
        self._sequential = bool(self.cfg.cuda_graphs)
        self._use_graphs = bool(self.cfg.cuda_graphs)
        self._freeze_graphs = False
        self.graph_choice = None
        self._graphs: dict = {}
        self._eager_runs = 0
        self._static = None
        self._pool = torch.cuda.graph_pool_handle() if self._use_graphs else None
        self._captured_native = 0
        self._replayed_native = 0
        self.last_step_kind = None
        self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad)
                       for p in self.params]
        self._fwd_wait = {}
        if self.placement == "start":
            self._install_forward_waits()
        # delayed schedules at W > 1 with per-iteration joins: the backward's last
        # fresh transfers start with the next iteration (see _buckets_ready)
        self._deferred: list[tuple[int, int, tuple]] = []
        self._defer_tail = (not self.sync and self.world > 1 and self._sequential
                            and bool(self.cfg.defer_tail))
        self._link_model = None
        if self._defer_tail and self.cfg.defer_tail == "predicted":
            self._link_model = LinkQueueModel(
                [b.backward_us for b in part.buckets], [b.comm_fast_us for b in part.buckets],
                [l.speed_ratio_to_fast for l in cluster.links])
        elif self._defer_tail and self.cfg.defer_tail not in (True, "last"):
            raise DeftError(f"unknown defer_tail {self.cfg.defer_tail!r}")
        self._planned = True
        return part

    def _probe_candidates(self, profile, cluster, cands, probe, warm: int = 4,
                          timed: int = 8) -> list[tuple[float, int]]:
        """Hardware score of each non-sequential candidate: `timed` iterations
        after `warm`, CUDA events, max over ranks; the training state is put back
        after every candidate."""
        if self.loopback is not None:
            raise DeftError("the hardware probe needs one process per GPU (not loopback)")
        batch, loss_fn = probe
        saved = [self.comm.params.clone(), self.mom.clone()]
        if self.comm.master is not None:
            saved.append(self.comm.master.clone())
        scores = []
        for i, cand in enumerate(cands):
            self.plan(profile, cluster, _candidate=cand)
            for _ in range(warm):
                self.train_step(batch, loss_fn)
            ms = self._time_steps(batch, loss_fn, timed)
            scores.append((ms, i))
            self.finish()
            self._release_graphs()
            self.comm.params.copy_(saved[0])
            self.mom.copy_(saved[1])
            if self.comm.master is not None:
                self.comm.master.copy_(saved[2])
            torch.cuda.synchronize(self.device)
        self.updates_applied = 0
        return scores

    def decisions(self, t: int) -> tuple[ScheduleDecision, ScheduleDecision]:
        return self.planner.decisions(t)

    @property
    def decision_log(self):
        return self.planner.decision_log

    # ---------------------------------------------------------------- runtime

    def _autocast(self):
        if self.cfg.autocast_dtype is None:
            return torch.autocast("cuda", enabled=False)
        # the weight-cast cache must not outlive a CUDA-graph capture
        return torch.autocast("cuda", dtype=self.cfg.autocast_dtype,
                              cache_enabled=not getattr(self, "_sequential", False))

    def _bind_grads(self, slot: int):
        if self._bound_slot == slot:
            return
        for p, g in zip(self.params, self._grad_views[slot]):
            p.grad = g
        self._bound_slot = slot

    def _timed(self, kind: str, stream, fn, nbytes: int):
        if not self.cfg.instrument:
            fn()
            return
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        self._events_t.append((kind, a, b, nbytes))

    def _issue_rs(self, link: int, slot: int, bidxs: list[int], release: torch.cuda.Event,
                  track: bool = False):
        """The buckets one release point puts on one link, in plan order: ONE
        reduce-scatter launch (one cross-rank barrier) on the link's stream.
        One-shot buckets have no transfer of their own: their update reads every
        rank's slot (deft_bucket_sync_update_multi)."""
        bidxs = [b for b in bidxs if not self._oneshot[b]]
        if self.world == 1 or not bidxs:
            return
        s = self.link_streams[link]
        s.wait_event(release)
        self._touched[id(s)] = s
        esz = 2 if self.cfg.grad_dtype == torch.bfloat16 else 4
        ranges = [(self.buckets[b].lo, self.buckets[b].hi) for b in bidxs]
        elems = sum(hi - lo for lo, hi in ranges)
        nbytes = elems * esz * (self.world - 1) // self.world  # crossing NVLink
        self._timed("reduce_scatter", s,
                    lambda: self.comm.reduce_scatter_multi(self.channel_of_link[link], slot,
                                                           ranges, s), nbytes)
        if track or not self._sequential or self.planner.lag == 0:
            # an update waits for it: always when streams run ahead (eager, async),
            # within the iteration for synchronous schedules (lag 0), and for
            # transfers deferred into the next iteration
            ev = torch.cuda.Event()
            ev.record(s)
            for b in bidxs:
                self._rs_done[(slot, b)] = ev

    def _launch_update(self, slot: int, bidxs, k: int, stream, nbytes: int):
        """One update event over buckets `bidxs`: the two-shot buckets (reduce-
        scattered at their transfer) get the fused update + parameter all-gather,
        the one-shot buckets the fused all-reduce + update -- one launch each."""
        two = [(self.buckets[b].lo, self.buckets[b].hi) for b in bidxs if not self._oneshot[b]]
        one = [(self.buckets[b].lo, self.buckets[b].hi) for b in bidxs if self._oneshot[b]]
        scale = 1.0 / (self.world * k)
        if two:
            self._timed("update", stream, lambda: self.comm.update_multi(
                slot, two, scale, self.cfg.lr, self.cfg.momentum, self.mom, stream), nbytes)
        if one:
            esz = 2 if self.cfg.grad_dtype == torch.bfloat16 else 4
            ob = sum(hi - lo for lo, hi in one) * esz * (self.world - 1)   # peer reads
            self._timed("oneshot", stream, lambda: self.comm.sync_update_multi(
                slot, one, scale, self.cfg.lr, self.cfg.momentum, self.mom, stream), ob)

    def _issue_planned(self, transfers, release: torch.cuda.Event):
        """Stage-plan transfers (link, slot, bucket) released together: per link,
        consecutive same-slot runs in plan order become one launch each."""
        for link, slot, bl in release_runs(transfers):
            self._issue_rs(link, slot, bl, release)

    def _issue_updates(self, bidxs: list[int], window_open: torch.cuda.Event):
        """"bucket" placement: the due updates of the buckets whose backward just
        ended, one multi-segment launch per update event on the update stream
        (small CTA budget: it runs beside the rest of the backward)."""
        s = self.update_stream
        s.wait_event(window_open)
        self._touched[id(s)] = s
        ranges = [(self.buckets[b].lo, self.buckets[b].hi) for b in bidxs]
        elems = sum(hi - lo for lo, hi in ranges)
        esz = 2 if self.cfg.grad_dtype == torch.bfloat16 else 4
        nbytes = elems * 20 if self.world == 1 else elems * esz * (self.world - 1) // self.world
        for slot, k in self._due_now:
            for b in bidxs:
                rs = self._rs_done.pop((slot, b), None)
                if rs is not None:
                    s.wait_event(rs)
            self._launch_update(slot, bidxs, k, s, nbytes)

    def _install_forward_waits(self):
        """"start" placement: the forward pre-hook of every module that owns
        parameters makes the compute stream wait for the update of the buckets
        those parameters live in (only the first wait per bucket does anything).
        A parameter read without its owning module's forward running (a
        ParameterList a parent iterates, a weight a parent uses directly) gets
        no pre-hook: the first forward records which buckets the hooks cover,
        and the others wait before the forward starts (``_unhooked``)."""
        owner = {id(p): bl for p, bl in zip(self.params, self._param_buckets)}
        self._fwd_wait: dict[int, torch.cuda.Event] = {}
        self._fwd_seen: set | None = None      # buckets the hooks covered (first forward)
        self._unhooked: set | None = None      # None = not known yet: wait for all

        def pre(mod, _args):
            if self._fwd_seen is not None:
                self._fwd_seen.update(self._module_buckets[mod])
            if not self._fwd_wait:
                return
            stream = torch.cuda.current_stream(self.device)
            for b in self._module_buckets[mod]:
                ev = self._fwd_wait.pop(b, None)
                if ev is not None:
                    stream.wait_event(ev)

        self._module_buckets = {}
        for m in self.module.modules():
            bl = sorted({b for p in m.parameters(recurse=False) if id(p) in owner
                         for b in owner[id(p)]})
            if bl:
                self._module_buckets[m] = bl
                self._hooks.append(m.register_forward_pre_hook(pre))

    def _start_groups(self) -> list[list[int]]:
        if getattr(self, "_groups_cache", None) is None:
            sizes = [b.hi - b.lo for b in self.buckets]
            groups = None
            if self.cfg.start_grouping in ("auto", "timed") and self.schedule_profile is not None:
                # update-stream cost model under the start budget (conservative:
                # measured 300-630 GB/s isolated, less beside the forward)
                esz = 2 if self.cfg.grad_dtype == torch.bfloat16 else 4
                per_elem_us = esz * max(1, self.world - 1) / max(1, self.world) / 200e3
                fwd = [b.forward_us for b in self.schedule_profile.buckets]
                rep: dict = {}
                groups = start_groups_timed(sizes, fwd, per_elem_us, 20.0,
                                            self.cfg.start_groups, rep)
                if self.cfg.start_grouping == "auto" and not rep["feasible"]:
                    groups = None   # the forward cannot hide them: size-based groups
            self._groups_cache = groups or start_groups(sizes, self.cfg.start_groups)
        return self._groups_cache

    def _updates_at_start(self, comp, due):
        """Updates of decision (t-2, backward) at the start of iteration t, input-side
        buckets first, overlapping the forward: a bucket's forward waits only for its
        own group's update launch."""
        ev0 = torch.cuda.Event()
        ev0.record(comp)
        s = self.update_stream
        s.wait_event(ev0)
        self._touched[id(s)] = s
        self._fwd_wait = {}
        esz = 2 if self.cfg.grad_dtype == torch.bfloat16 else 4
        for gi, group in enumerate(self._start_groups()):
            # the forward waits for the first group with the GPU otherwise idle:
            # full grid; later groups overlap the forward on the small budget
            self.comm.set_update_blocks(0 if gi == 0 else self._update_blocks)
            ranges = [(self.buckets[b].lo, self.buckets[b].hi) for b in group]
            elems = sum(hi - lo for lo, hi in ranges)
            nbytes = elems * 20 if self.world == 1 else elems * esz * (self.world - 1) // self.world
            for slot, k in due:
                if self.world > 1:
                    for b in group:          # the reduce-scatters of this group are done
                        rs = self._rs_done.pop((slot, b), None)
                        if rs is not None:
                            s.wait_event(rs)
                self._launch_update(slot, group, k, s, nbytes)
            ev = torch.cuda.Event()
            ev.record(s)
            for b in group:
                self._fwd_wait[b] = ev
        self.comm.set_update_blocks(self._update_blocks)

    def _updates_at_end(self, comp):
        """All due updates after the whole backward (every no-read window is open):
        one multi-bucket launch per update event on the compute stream -- the local
        fused update at W == 1, the fused update + parameter all-gather at W > 1."""
        ranges = [(b.lo, b.hi) for b in self.buckets]
        esz = 2 if self.cfg.grad_dtype == torch.bfloat16 else 4
        if self.world == 1:
            nbytes = self.total * 20  # read g, v, p(master); write v, p (+bf16 copy)
        else:
            nbytes = self.total * esz * (self.world - 1) // self.world  # crossing NVLink
        for slot, k in self._due_now:
            if self.world > 1:   # the group's reduce-scatters still in flight
                for b in range(len(self.buckets)):
                    rs = self._rs_done.pop((slot, b), None)
                    if rs is not None:
                        comp.wait_event(rs)
            self._launch_update(slot, range(len(self.buckets)), k, comp, nbytes)

    def _on_grad(self, p):
        if not self._in_step:
            return
        idx = self._param_index[id(p)]
        ready = []
        for b in self._param_buckets[idx]:
            self._pending[b] -= 1
            if self._pending[b] == 0:
                ready.append(b)
        if ready:   # e.g. every piece of a partitioned layer at once
            self._buckets_ready(ready)

    def _gather_buckets(self, bidxs: list[int], slot: int):
        """Copy the buckets' fresh per-parameter gradients into their slot ranges
        (one gather launch)."""
        esz = 2 if self.cfg.grad_dtype == torch.bfloat16 else 4
        srcs, offs, lens = [], [], []
        for bidx in bidxs:
            b = self.buckets[bidx]
            for i in self._bucket_params[bidx]:
                p, o = self.params[i], self.offsets[i]
                lo, hi = max(b.lo, o), min(b.hi, o + p.numel())
                g = p.grad
                if g is None or g.stride() != p.stride() or g.dtype != p.dtype:
                    view = self.comm.grads[slot][lo:hi]
                    if g is None:
                        view.zero_()
                    else:   # layout differs: a strided copy of the whole parameter
                        self._grad_views[slot][i].copy_(g)
                    continue
                srcs.append(g.data_ptr() + (lo - o) * esz)
                offs.append(lo * esz)
                lens.append((hi - lo) * esz)
        if srcs:
            stream = torch.cuda.current_stream(self.device)
            # beside the backward (W > 1) large ranges use the copy engines
            self.comm.gather(slot, srcs, offs, lens, stream,
                             ce_min_bytes=-1 if self.world > 1 else 0)

    def _buckets_ready(self, bidxs: list[int]):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        if self._gather_slot is not None and self.world == 1:
            # one GPU: no transfer follows -- copy in line on the compute stream
            self._gather_buckets(bidxs, self._gather_slot)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
        elif self._gather_slot is not None:
            # copy the fresh gradients into the slot on the gather stream: the
            # backward continues while they move (the compute stream joins it
            # once, after the whole backward); the buckets' transfers wait for it
            gs = self.gather_stream
            gs.wait_event(ev)
            self._touched[id(gs)] = gs
            with torch.cuda.stream(gs):
                self._gather_buckets(bidxs, self._gather_slot)
            ev = torch.cuda.Event()
            ev.record(gs)
        # the backward's last release: with delayed updates its transfers may
        # start with the next iteration instead (they are needed an iteration
        # later), so the per-iteration join does not wait for them
        last = self._defer_tail and sum(self._fired) + len(bidxs) == len(self.buckets)
        fresh = [(link, slot, bidx) for bidx in bidxs
                 for link, slot in self._fresh_now.pop(bidx, ())]
        for link, slot, bl in release_runs(fresh):
            if last or (self._link_model is not None and
                        not self._link_model.admit(link, bl, bidxs)):
                self._deferred.append((link, slot, tuple(bl)))
            else:
                self._issue_rs(link, slot, bl, ev)
        if self.placement == "bucket" and self._due_now:
            self._issue_updates(bidxs, ev)
        for bidx in bidxs:
            self._fired[bidx] = True

    def _issue_deferred(self, release: torch.cuda.Event):
        """Transfers the previous iteration deferred from its backward's end."""
        deferred, self._deferred = self._deferred, []
        for link, slot, bl in deferred:
            self._issue_rs(link, slot, list(bl), release, track=True)

    def _run_iteration(self, it: IterPlan, batch, loss_fn: Callable) -> torch.Tensor:
        """Issue one iteration's device work on the current stream (+ link and
        update streams).  Runs eagerly or inside a CUDA-graph capture."""
        comp = torch.cuda.current_stream(self.device)
        self._touched = {}      # side streams forked from `comp` in this iteration
        if not self._sequential and self._version_ready is not None:
            comp.wait_event(self._version_ready)   # theta^(t) complete
        ev_fwd = torch.cuda.Event()
        ev_fwd.record(comp)
        self._issue_deferred(ev_fwd)
        if self.placement == "start":
            if self._unhooked is None:
                self._fwd_seen = set()
            if it.due:
                self._updates_at_start(comp, it.due)
                for b in (range(len(self.buckets)) if self._unhooked is None
                          else self._unhooked):
                    ev = self._fwd_wait.pop(b, None)    # no pre-hook will wait for it
                    if ev is not None:
                        comp.wait_event(ev)
        self._issue_planned(it.fwd, ev_fwd)
        with self._autocast():
            loss = loss_fn(self.module, batch)
        if self.placement == "start":
            for ev in self._fwd_wait.values():   # buckets no forward module touched
                comp.wait_event(ev)
            self._fwd_wait = {}
            if self._fwd_seen is not None:
                self._unhooked = set(range(len(self.buckets))) - self._fwd_seen
                self._fwd_seen = None
        if it.zero:
            # store: autograd allocates fresh gradients (no accumulate kernels) and
            # each bucket is gathered into the group slot when its backward ends
            if not self._sequential and self._slot_free[it.slot] is not None:
                comp.wait_event(self._slot_free[it.slot])
            for p in self.params:
                p.grad = None
            self._bound_slot = None
            self._gather_slot = it.slot
        else:
            # merge: accumulate straight into the live group's slot
            self._bind_grads(it.slot)
            self._gather_slot = None
        ev_bwd = torch.cuda.Event()
        ev_bwd.record(comp)
        self._issue_planned(it.bwd, ev_bwd)
        self._fresh_now = dict(it.fresh)
        self._due_now = it.due if self.placement != "start" else ()
        self._pending = list(self._bucket_nparams)
        self._fired = [False] * len(self.buckets)
        if self._link_model is not None:
            self._link_model.reset()
        self._in_step = True
        try:
            loss.backward()
        finally:
            self._in_step = False
        unfired = [b for b in range(len(self.buckets)) if not self._fired[b]]
        if unfired:                             # buckets whose params got no gradient
            self._buckets_ready(unfired)
        if self._gather_slot is not None and self.world > 1:
            # every gather done before the slot is read by an update on this
            # stream and before autograd's gradient buffers can be reused
            comp.wait_stream(self.gather_stream)
        if self.placement == "end" and self._due_now:
            self._updates_at_end(comp)
        if self._fresh_now:
            raise InternalInvariantError("fresh transfers left unreleased")
        loss = loss.detach()  # drop the autograd graph (no stale AccumulateGrad nodes)
        if self._sequential:
            for s in self._touched.values():   # join (only streams forked this iteration)
                comp.wait_stream(s)
            # everything issued so far is complete once the join is: no event may
            # carry over (inside a CUDA-graph capture it could not be waited on)
            self._rs_done.clear()
        else:
            ev = torch.cuda.Event()
            ev.record(self.update_stream)
            self._version_ready = ev
            for fs in it.freed:
                self._slot_free[fs] = ev
        return loss

    def _static_inputs(self, batch):
        if self._static is None:
            self._static = tuple(x.detach().clone() for x in batch)
        if any(a is not b for a, b in zip(self._static, batch)):
            for dst, src in zip(self._static, batch):
                dst.copy_(src, non_blocking=True)
        return self._static

    @property
    def static_batch(self):
        """The input tensors captured graphs read (CUDA-graph mode); writing the
        next batch straight into them saves a device copy."""
        return self._static

    def native_launches(self) -> int:
        """Native kernels launched (captured kernels count once per replay)."""
        return _native.launch_count() - self._captured_native + self._replayed_native

    def train_step(self, batch, loss_fn: Callable) -> torch.Tensor:
        """One DeFT iteration: forward (Case 1 transfers released), backward
        (Case 2/3/4 transfers, fresh ones per bucket), delayed updates.
        Returns the (detached) loss.  With ``cuda_graphs`` the device work of
        every distinct iteration shape is captured once (after one eager run)
        and replayed; the loss is then a static tensor, valid until the next step.
        All device work runs on the executor's own compute stream, ordered after
        the caller's current stream and before its next work."""
        if not hasattr(self, "scheduler"):
            raise DeftError("call plan() before train_step()")
        if not hasattr(self, "_param_index"):
            self._param_index = {id(p): i for i, p in enumerate(self.params)}
        it = self.planner.plan(self.iteration)
        self.iteration += 1
        self.updates_applied += len(it.due)
        caller = torch.cuda.current_stream(self.device)
        self.compute_stream.wait_stream(caller)
        with torch.cuda.stream(self.compute_stream):
            loss = self._dispatch(it, batch, loss_fn)
        caller.wait_stream(self.compute_stream)
        return loss

    def warm_up(self, batch, loss_fn: Callable, min_steps: int = 3, max_steps: int = 96,
                steady: int = 6, compare: int = 4) -> int:
        """Run steps until the last `steady` were all graph replays (every
        steady-state iteration shape captured).  Then, with ``cuda_graphs="auto"``,
        time `compare` replayed steps against `compare` eager ones and keep the
        faster mode (some models' captured kernels are slower than their eager
        ones).  Returns the number of steps run."""
        streak, n = 0, 0
        while n < max_steps and (n < min_steps or streak < steady):
            self.train_step(batch, loss_fn)
            n += 1
            streak = streak + 1 if self.last_step_kind == "replay" else 0
            if not self._use_graphs:
                streak = steady
        if self._use_graphs and streak < steady:
            # the iteration shapes never settled (e.g. irregular merge patterns):
            # capturing on the fly would keep paying for captures -- run eagerly,
            # and give the captured graphs' memory pool back to the allocator
            # (left resident it starves eager execution: 134 vs 26 ms per step)
            self._use_graphs = False
            self._release_graphs()
            self.graph_choice = {"use_graphs": False, "reason": "no steady-state shape",
                                 "graphs_released": True}
            for _ in range(min_steps):        # the allocator re-grows eagerly
                self.train_step(batch, loss_fn)
            return n + min_steps
        # from now on unseen iteration shapes run eagerly instead of being captured
        self._freeze_graphs = True
        if self.cfg.cuda_graphs == "auto" and self._use_graphs and compare > 0:
            t_graph = self._time_steps(batch, loss_fn, compare)
            self._use_graphs = False
            for _ in range(2):                    # eager warm-up: allocator, autotuning
                self.train_step(batch, loss_fn)
            t_eager = self._time_steps(batch, loss_fn, compare)
            self._use_graphs = t_graph <= t_eager
            self.graph_choice = {"graph_ms": t_graph / compare, "eager_ms": t_eager / compare,
                                 "use_graphs": self._use_graphs}
            if not self._use_graphs:
                self._release_graphs()
                for _ in range(2):            # the allocator re-grows eagerly
                    self.train_step(batch, loss_fn)
                n += 2
            n += 2 * compare + 2
        return n

    def _release_graphs(self):
        import gc
        torch.cuda.synchronize(self.device)
        self._graphs.clear()
        gc.collect()
        torch.cuda.empty_cache()

    def _time_steps(self, batch, loss_fn, k) -> float:
        ms = 0.0
        if self.world > 1:
            torch.distributed.barrier(group=self.group)
        torch.cuda.synchronize(self.device)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            self.train_step(batch, loss_fn)
        b.record()
        torch.cuda.synchronize(self.device)
        ms = a.elapsed_time(b)
        if self.world > 1:   # every rank must take the same decision
            t = torch.tensor([ms], device=self.device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=self.group)
            ms = float(t.item())
        return ms

    def _dispatch(self, it: IterPlan, batch, loss_fn: Callable) -> torch.Tensor:
        if not self._sequential or self.cfg.instrument or not self._use_graphs:
            self.last_step_kind = "eager"
            if self._sequential and self._static is not None:
                batch = self._static_inputs(batch)
            return self._run_iteration(it, batch, loss_fn)
        static = self._static_inputs(batch)
        key = (it.key, tuple(self._deferred))   # deferred transfers run in this graph
        hit = self._graphs.get(key)
        if hit is not None:
            g, loss, n, deferred = hit
            self._deferred = list(deferred)
            g.replay()
            self._replayed_native += n
            self.last_step_kind = "replay"
            return loss
        # a new shape is captured on first sight once the process itself is warm
        # (allocator, library handles, autotuning: `graph_warmup` eager
        # iterations of any shape) -- the model's compute is the same in every
        # shape, only the communication plan differs
        if self._eager_runs < self.cfg.graph_warmup or self._freeze_graphs:
            self._eager_runs += 1
            self.last_step_kind = "eager"
            return self._run_iteration(it, static, loss_fn)
        self.compute_stream.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = _native.launch_count()
        if self.loopback is not None:
            # torch.cuda.graph() synchronizes the whole device first, which in a
            # loopback world would wait for peers whose iteration is not issued
            with torch.cuda.stream(self.compute_stream):
                g.capture_begin(pool=self._pool)
                try:
                    loss = self._run_iteration(it, static, loss_fn)
                finally:
                    g.capture_end()
        else:
            with torch.cuda.graph(g, pool=self._pool, stream=self.compute_stream):
                loss = self._run_iteration(it, static, loss_fn)
        n = _native.launch_count() - n0
        self._captured_native += n
        self._graphs[key] = (g, loss, n, tuple(self._deferred))
        if self.loopback is not None:
            # graph instantiation synchronizes the device: no rank may replay a
            # new shape before every rank has captured it (LoopbackWorld.flush)
            self.loopback.defer_replay(g, self.compute_stream)
        else:
            g.replay()
        self._replayed_native += n
        self.last_step_kind = "capture"
        return loss

    def finish(self, sync: bool = True):
        """Make theta^(t) current (t = iterations run) and drain every stream
        (``sync=False``: only issue the work -- a loopback world issues every
        rank's finish before it synchronizes).
        With "start" placement the updates that become visible at iteration t are
        applied here (they would otherwise run at the start of iteration t); groups
        still in flight stay unapplied, as in the reference where unaccounted
        iterations are still in flight."""
        if getattr(self, "_deferred", None):
            caller = torch.cuda.current_stream(self.device)
            self.compute_stream.wait_stream(caller)
            with torch.cuda.stream(self.compute_stream):
                self._touched = {}
                ev = torch.cuda.Event()
                ev.record(self.compute_stream)
                self._issue_deferred(ev)
                for st in self._touched.values():
                    self.compute_stream.wait_stream(st)
            caller.wait_stream(self.compute_stream)
        if self.placement == "start" and hasattr(self, "planner"):
            due, freed = self.planner.take_pending()
            self.updates_applied += len(due)
            if due:
                caller = torch.cuda.current_stream(self.device)
                self.compute_stream.wait_stream(caller)
                with torch.cuda.stream(self.compute_stream):
                    comp = self.compute_stream
                    self._touched = {}
                    self._updates_at_start(comp, due)
                    for ev in self._fwd_wait.values():
                        comp.wait_event(ev)
                    self._fwd_wait = {}
                caller.wait_stream(self.compute_stream)
        if sync:
            torch.cuda.synchronize(self.device)

    def timing_summary(self) -> dict:
        """Per-kind (count, total ms, bytes) of the instrumented launches."""
        torch.cuda.synchronize(self.device)
        out: dict[str, list[float]] = {}
        for kind, a, b, nbytes in self._events_t:
            r = out.setdefault(kind, [0, 0.0, 0])
            r[0] += 1
            r[1] += a.elapsed_time(b)
            r[2] += nbytes
        self._events_t = []
        return {k: {"launches": int(v[0]), "ms": v[1], "bytes": int(v[2])} for k, v in out.items()}

    def close(self):
        for h in getattr(self, "_hooks", []):
            h.remove()
        self._hooks = []
        self.comm.close()
