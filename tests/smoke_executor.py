"""Delayed-update executor parity harness (used by __graft_entry__.smoke(),
tests/test_gpu_executor.py and tests/test_gpu_loopback.py).

The probe model's loss is 1/2 sum_i <x_i, theta_i^2> with every x_i element
+-2^-e: the gradient x * theta depends on the parameter version the forward
and backward read (a stale or racing parameter read changes it), and autograd
computes it EXACTLY in fp32 and in bf16 (power-of-two scaling; the two
product-rule terms are equal halves).  The oracle (oracle/delayed_sgd.py
``run_kernel_order``) replays the same decision stream on the CPU in the
kernels' arithmetic order, so the only floating-point difference left is the
order of the cross-rank fp32 sum: fp32 is checked ELEMENTWISE at 1e-6
relative, bf16 bit for bit.
"""
from __future__ import annotations

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2503_16815_b200 as D  # noqa: E402
from oracle import delayed_sgd  # noqa: E402

# elementwise relative tolerance, fp32 (north_star: "within 1e-6 relative (fp32)");
# |a - b| <= TOL * max(|b|, FLOOR) -- the probe's per-element dynamics are linear
# in theta_i, so relative errors do not grow for small |theta_i|; FLOOR only
# guards exact zeros
TOL = 1e-6
FLOOR = 1e-30


class Probe(torch.nn.Module):
    def __init__(self, sizes, seed=0):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.ps = torch.nn.ParameterList(
            [torch.nn.Parameter(torch.randn(n, generator=g)) for n in sizes])

    def forward(self, xs):
        # d/dtheta = 0.5 * (x*theta) + (0.5*theta) * x = x * theta, exactly
        return 0.5 * sum((x * p * p).sum() for p, x in zip(self.ps, xs))


def probe_sizes(total=48_000, n=31, seed=3):
    g = torch.Generator().manual_seed(seed)
    cuts = sorted(torch.randperm(total - 1, generator=g)[: n - 1].add(1).tolist())
    edges = [0] + cuts + [total]
    return [b - a for a, b in zip(edges, edges[1:])]


def flat_x(total, rank, t, seed=11):
    """+-2^-e, e in {1, 2, 3}: exact in bf16, and x * theta is exact in any dtype."""
    g = torch.Generator().manual_seed(seed * 1_000_003 + 7919 * t + rank)
    e = torch.randint(1, 4, (total,), generator=g).float()
    s = torch.randint(0, 2, (total,), generator=g).float() * 2 - 1
    return s * torch.pow(2.0, -e)


def uniform_profile(n, param_count, comm_us=900, fwd_total=3600, bwd_total=7200):
    fwd = [fwd_total // n] * n
    bwd = [bwd_total // n] * n
    for i in range(fwd_total - sum(fwd)):
        fwd[i] += 1
    for i in range(bwd_total - sum(bwd)):
        bwd[i] += 1
    return D.ModelProfile(
        name=f"uniform{n}", batch_size=256,
        buckets=tuple(D.BucketProfile(i + 1, param_count, fwd[i], bwd[i], comm_us)
                      for i in range(n)))


def equal_dual():
    """The reference's equal_dual_cluster (tests/conftest.py:17-19, 52-57): the
    twin link maps to the copy-engine channel."""
    return D.ClusterSpec(links=(D.LinkSpec("fast"), D.LinkSpec("twin", 1.0000001)))


def _config(lr, momentum, partition_size, cuda_graphs, placement, scheme, lookahead=32,
            n_slots=6, startup_us=0, oneshot=0, defer=True):
    return D.DeftConfig(lr=lr, momentum=momentum, autocast_dtype=None,
                        partition=D.PartitionConfig(partition_size=partition_size,
                                                    comm_startup_us=startup_us),
                        cuda_graphs=cuda_graphs, update_placement=placement, scheme=scheme,
                        lookahead=lookahead, n_slots=n_slots, oneshot_max_bytes=oneshot,
                        defer_tail=defer)


def _xs_for(ddp, model, flat):
    order = list(model.ps)[::-1]  # executor flat order: output-side parameter first
    xs_exec = [flat[o:o + p.numel()].view_as(p) for o, p in zip(ddp.offsets, order)]
    return xs_exec[::-1]


def _loss_fn(module, batch):
    return module(batch)


def theta0_for(total, dtype):
    """theta^(0) in the executor's flat order (dtype-rounded, as fp32)."""
    return torch.cat([p.detach().to(dtype).float().reshape(-1) for p in
                      Probe(probe_sizes(total)).ps][::-1])


def run_executor(world, rank, iterations, n_buckets=48, total=48_000, lr=0.05, momentum=0.9,
                 dtype=torch.float32, comm_us=900, group=None, cuda_graphs=True,
                 x_fn=flat_x, placement="end", scheme="deft", partition_size=10**9,
                 model_cls=None, startup_us=0, hw_probe=False, oneshot=0, defer=True):
    """One rank of a real (one process per GPU) run on the probe.  Returns
    (master fp32 CPU -- the parameters for fp32 models --, params CPU in the
    model dtype, theta0, decisions as dicts, bucket ranges).  ``hw_probe``: the
    non-sequential scheme scores its candidates by timing them on the GPU."""
    model = (model_cls or Probe)(probe_sizes(total)).cuda().to(dtype)
    cfg = _config(lr, momentum, partition_size, cuda_graphs, placement, scheme,
                  startup_us=startup_us, oneshot=oneshot, defer=defer)
    ddp = D.DeftDataParallel(model, cfg, process_group=group)
    prof = uniform_profile(n_buckets, total // n_buckets, comm_us=comm_us)
    probe = None
    if hw_probe:
        probe = (_xs_for(ddp, model, x_fn(total, rank, 0).cuda().to(dtype)), _loss_fn)
    ddp.plan(prof, equal_dual(), probe=probe)
    ddp.probe_scores = getattr(ddp, "nonsequential_scores", None)
    for t in range(iterations):
        flat = x_fn(total, rank, t).cuda().to(dtype)
        ddp.train_step(_xs_for(ddp, model, flat), _loss_fn)
    ddp.finish()
    master = ddp.comm.master if ddp.comm.master is not None else ddp.comm.params
    theta = master.detach().float().cpu().clone()
    params = ddp.comm.params.detach().cpu().clone()
    decisions = [d.to_dict() for k in range(iterations) for d in ddp.decisions(k)]
    buckets = [(b.lo, b.hi) for b in ddp.buckets]
    ddp.close()
    return theta, params, theta0_for(total, dtype), decisions, buckets


def run_loopback(world, iterations, n_buckets=48, total=48_000, lr=0.05, momentum=0.9,
                 dtype=torch.float32, comm_us=900, cuda_graphs=True, x_fn=flat_x,
                 placement="end", scheme="deft", partition_size=10**9, model_cls=None,
                 profile=None, cluster=None, startup_us=0, oneshot=0, defer=True):
    """W ranks in this process on cuda:current (loopback.py), driven round-robin
    from this thread.  Returns per-rank (master, params) lists, theta0 and the
    (identical) decision stream of rank 0."""
    lbw = D.LoopbackWorld(world)
    models, execs = [], []
    look = iterations + 4        # every decision generated before the first step
    for r in range(world):
        model = (model_cls or Probe)(probe_sizes(total)).cuda().to(dtype)
        cfg = _config(lr, momentum, partition_size, cuda_graphs, placement, scheme,
                      lookahead=look, startup_us=startup_us, oneshot=oneshot, defer=defer)
        models.append(model)
        execs.append(D.DeftDataParallel(model, cfg, process_group=lbw.rank(r)))
    prof = profile or uniform_profile(n_buckets, total // n_buckets, comm_us=comm_us)
    for ddp in execs:
        ddp.plan(prof, cluster or equal_dual())
        ddp.decisions(iterations - 1)
    # inputs resident before the loop: the host must not block mid-iteration
    xs = [[_xs_for(execs[r], models[r], x_fn(total, r, t).to(dtype).cuda())
           for t in range(iterations)] for r in range(world)]
    torch.cuda.synchronize()
    marks = _watch_install(execs) if _WATCH else None
    with lbw.issuing():
        for t in range(iterations):
            for r in range(world):
                with torch.cuda.stream(lbw.rank(r).compute_stream):
                    execs[r].train_step(xs[r][t], _loss_fn)
            lbw.flush()            # graphs captured this round replay now
        for r in range(world):
            with torch.cuda.stream(lbw.rank(r).compute_stream):
                execs[r].finish(sync=False)
        if marks is not None:
            _watch_wait(marks)
        torch.cuda.synchronize()
    masters, params = [], []
    for ddp in execs:
        m = ddp.comm.master if ddp.comm.master is not None else ddp.comm.params
        masters.append(m.detach().float().cpu().clone())
        params.append(ddp.comm.params.detach().cpu().clone())
    decisions = [[d.to_dict() for k in range(iterations) for d in ddp.decisions(k)]
                 for ddp in execs]
    kinds = [ddp.last_step_kind for ddp in execs]
    buckets = [(b.lo, b.hi) for b in execs[0].buckets]
    for ddp in execs:
        ddp.close()
    return masters, params, theta0_for(total, dtype), decisions, buckets, kinds


# DEFT_LOOPBACK_WATCH=1: record an event after every comm launch and every
# train_step of every rank, and before synchronizing poll them; if nothing
# completes for 5 s, print the last completed / first pending op of each
# rank's streams (diagnoses a loopback stall before the barrier spin traps)
import os as _os  # noqa: E402
_WATCH = _os.environ.get("DEFT_LOOPBACK_WATCH") == "1"


def _watch_install(execs):
    from paper_2503_16815_b200 import comm as C
    marks = []        # (rank, label, stream id, event)

    def wrap(name):
        orig = getattr(C.BucketComm, name)

        def f(self, *a, **k):
            out = orig(self, *a, **k)
            st = [x for x in a if hasattr(x, "cuda_stream")][0]
            if torch.cuda.is_current_stream_capturing():
                return out
            ev = torch.cuda.Event()
            ev.record(st)
            marks.append((self.rank, f"{name}{[x for x in a[:2] if isinstance(x, int)]}",
                          st.cuda_stream, ev))
            return out
        f._orig = orig
        setattr(C.BucketComm, name, f)
    for n in ("reduce_scatter_multi", "update_multi", "gather"):
        if not hasattr(getattr(C.BucketComm, n), "_orig"):
            wrap(n)
    for ddp in execs:
        orig_step = ddp.train_step

        def step(*a, _o=orig_step, _d=ddp, **k):
            out = _o(*a, **k)
            if _d.last_step_kind == "capture":
                return out
            ev = torch.cuda.Event()
            ev.record(_d.compute_stream)
            marks.append((_d.rank, f"step{_d.iteration - 1}", _d.compute_stream.cuda_stream, ev))
            return out
        ddp.train_step = step
    return marks


def _watch_wait(marks, quiet_s=5.0):
    import time
    last, t0 = -1, time.time()
    while True:
        done = sum(1 for m in marks if m[3].query())
        if done == len(marks):
            return
        if done != last:
            last, t0 = done, time.time()
        elif time.time() - t0 > quiet_s:
            break
        time.sleep(0.05)
    by_rank: dict = {}
    for i, (r, label, sid, ev) in enumerate(marks):
        by_rank.setdefault(r, []).append((i, label, sid % 100000, ev.query()))
    for r, ms in sorted(by_rank.items()):
        pend = [m for m in ms if not m[3]]
        okk = [m for m in ms if m[3]]
        print(f"WATCH rank {r}: {len(okk)}/{len(ms)} done; last done {okk[-1][:3] if okk else None}; "
              f"first pending {pend[0][:3] if pend else None}", flush=True)
    raise RuntimeError("loopback stall (see WATCH lines)")


def oracle_theta(theta0, decisions, world, iterations, total=48_000, lr=0.05, momentum=0.9,
                 x_fn=flat_x, lag=2, dtype=torch.float32):
    """lag 2: DeFT (visible from t+2); lag 1: the synchronous wfbp/priority schemes.
    Returns (master fp32, params in dtype)."""
    return delayed_sgd.run_kernel_order(theta0, lambda r, t: x_fn(total, r, t), decisions,
                                        world, lr, momentum, iterations, dtype=dtype, lag=lag)


def elem_err(a, b):
    """max_i |a_i - b_i| / max(|b_i|, FLOOR)  (elementwise relative error)."""
    a, b = a.double(), b.double()
    return float(((a - b).abs() / b.abs().clamp_min(FLOOR)).max())


def shard_range(offset, numel, r, world, align):
    """Python copy of shard_of() (csrc/common.cuh)."""
    per = (numel + world - 1) // world

    def bound(k):
        if k <= 0:
            return offset
        if k >= world:
            return offset + numel
        b = -(-(offset + k * per) // align) * align
        return min(b, offset + numel)
    return bound(r), bound(r + 1)


def check_ranks(masters, params, want_master, want_params, world, dtype, buckets):
    """Every rank's parameters equal the oracle's (fp32: elementwise 1e-6; bf16:
    bit for bit) and each other; the fp32 master is checked where the rank owns
    it (W > 1: its 1/W shard of every bucket; bf16 models keep the master
    ZeRO-1 style).  Returns the worst elementwise error."""
    worst = 0.0
    align = 4 if dtype == torch.float32 else 8
    for r in range(world):
        p = params[r].float()
        if dtype == torch.float32:
            worst = max(worst, elem_err(p, want_params.float()))
        else:
            assert torch.equal(params[r], want_params), f"rank {r}: bf16 params differ"
        assert torch.equal(params[r], params[0]), f"rank {r}: replicas differ"
        for blo, bhi in buckets:
            lo, hi = shard_range(blo, bhi - blo, r, world, align)
            if hi > lo:
                worst = max(worst, elem_err(masters[r][lo:hi], want_master[lo:hi]))
    assert worst <= TOL, f"elementwise relative error {worst:.3e} > {TOL}"
    return worst


def run_smoke_executor(iterations=12):
    """One GPU: the fused local update (W = 1) against the oracle."""
    theta, params, theta0, decisions, buckets = run_executor(1, 0, iterations)
    merges = [u["merge_count"] for d in decisions for u in d["update_events"]]
    want_m, want_p = oracle_theta(theta0, decisions, 1, iterations)
    err = check_ranks([theta], [params], want_m, want_p, 1, torch.float32, buckets)
    assert max(merges) >= 2, "the smoke profile should merge iterations"
    assert not torch.equal(theta, theta0), "parameters never moved"
    return err


def run_smoke_loopback(world=4, iterations=10, dtype=torch.float32, placement="start",
                       oneshot=0, partition_size=10**9):
    """W ranks on this GPU: reduce-scatter (SM + copy-engine channels), fused
    update + parameter all-gather, barriers (and, with ``oneshot``, the one-shot
    all-reduce + update for buckets of at most that many bytes) -- against the
    oracle."""
    masters, params, theta0, decisions, buckets, _ = run_loopback(
        world, iterations, dtype=dtype, placement=placement, oneshot=oneshot,
        partition_size=partition_size)
    for r in range(1, world):
        assert decisions[r] == decisions[0], "ranks planned different streams"
    want_m, want_p = oracle_theta(theta0, decisions[0], world, iterations, dtype=dtype)
    return check_ranks(masters, params, want_m, want_p, world, dtype, buckets)


def run_collective(world, iterations=8, dtype=torch.float32, total=48_000, n_buckets=48,
                   lr=0.05, momentum=0.9, x_fn=flat_x):
    """Kernel-level delayed-update parity in a loopback world with ONE launch per
    collective (deft_loopback_reduce_scatter / deft_loopback_update): pairs of
    iterations merge into one gradient group (store, then merge), every group
    is reduce-scattered -- even buckets on the SM channel, odd ones on the
    copy-engine channel -- and applied as one fused update + parameter
    all-gather with scale 1/(2W), visible from the next iteration (oracle lag 1).
    Works when the device serializes kernels (the driver's profiled smoke run).
    Returns the worst elementwise error."""
    from paper_2503_16815_b200 import _native
    lbw = D.LoopbackWorld(world)
    comms = lbw.make_comms(2, total, dtype)
    dev = lbw.device
    theta0 = theta0_for(total, dtype)
    for c in comms:
        c.params.copy_(theta0.to(dtype))
        if c.master is not None:
            c.master.copy_(theta0)
    moms = [torch.zeros(total, dtype=torch.float32, device=dev) for _ in range(world)]
    size = total // n_buckets
    ranges = [(b * size, (b + 1) * size) for b in range(n_buckets)]
    sm, ce = ranges[0::2], ranges[1::2]
    s = torch.cuda.current_stream(dev)
    decisions = []
    torch.cuda.synchronize()
    for t in range(iterations):
        slot = (t // 2) % 2
        for r in range(world):
            g = (x_fn(total, r, t).to(dtype).to(dev) * comms[r].params).to(dtype)
            if t % 2 == 0:
                comms[r].grads[slot].copy_(g)
            else:
                comms[r].grads[slot].add_(g)      # merge (autograd's accumulate)
        if t % 2 == 1:
            torch.cuda.synchronize()
            lbw.collective_reduce_scatter(comms, _native.CHANNEL_SM, slot, sm, s)
            lbw.collective_reduce_scatter(comms, _native.CHANNEL_CE, slot, ce, s)
            lbw.collective_update(comms, slot, ranges, 1.0 / (world * 2), lr, momentum, moms, s)
            decisions.append({"iteration": t, "stage": "backward",
                              "update_events": [{"origins": [t - 1, t], "merge_count": 2}]})
    torch.cuda.synchronize()
    masters = [(c.master if c.master is not None else c.params).float().cpu() for c in comms]
    params = [c.params.cpu() for c in comms]
    want_m, want_p = delayed_sgd.run_kernel_order(
        theta0, lambda r, t: x_fn(total, r, t), decisions, world, lr, momentum, iterations,
        dtype=dtype, lag=1)
    err = check_ranks(masters, params, want_m, want_p, world, dtype, ranges)
    for c in comms:
        c.close()
    return err
