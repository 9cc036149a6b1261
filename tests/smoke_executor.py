"""Delayed-update executor parity harness (used by __graft_entry__.smoke() and
tests/test_gpu_executor.py).

The probe model's loss is sum_i <theta_i, x_i>, so the gradient of every
parameter IS the data tensor x_i -- computed exactly (no rounding) by autograd
on any device.  All floating-point work left is the communication + delayed
SGD/momentum path under test, which is what makes a 1e-6 relative tolerance
against the CPU oracle meaningful.
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

TOL = 1e-6  # relative, fp32 (north_star: "within 1e-6 relative (fp32)")


class Probe(torch.nn.Module):
    def __init__(self, sizes, seed=0):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.ps = torch.nn.ParameterList(
            [torch.nn.Parameter(torch.randn(n, generator=g)) for n in sizes])

    def forward(self, xs):
        return sum((p * x).sum() for p, x in zip(self.ps, xs))


def probe_sizes(total=48_000, n=31, seed=3):
    g = torch.Generator().manual_seed(seed)
    cuts = sorted(torch.randperm(total - 1, generator=g)[: n - 1].add(1).tolist())
    edges = [0] + cuts + [total]
    return [b - a for a, b in zip(edges, edges[1:])]


def flat_grad(total, rank, t, seed=11):
    g = torch.Generator().manual_seed(seed * 1_000_003 + 7919 * t + rank)
    return torch.randn(total, generator=g)


def flat_grad_dyadic(total, rank, t, seed=13):
    """Small multiples of 1/16: exact in bf16, and so are sums of a few of them
    (merges accumulate in the bf16 slot; the reduce-scatter rounds to bf16)."""
    g = torch.Generator().manual_seed(seed * 1_000_003 + 7919 * t + rank)
    return torch.randint(-8, 9, (total,), generator=g).float() / 16


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
    return D.ClusterSpec(links=(D.LinkSpec("fast"), D.LinkSpec("twin", 1.0000001)))


def run_executor(world, rank, iterations, n_buckets=48, total=48_000, lr=0.05, momentum=0.9,
                 dtype=torch.float32, comm_us=900, group=None, cuda_graphs=True,
                 grad_fn=flat_grad, placement="end", scheme="deft", partition_size=10**9):
    """Run the executor on the probe; return (theta^(T) flat fp32 CPU -- the fp32
    master for bf16 models --, theta0, decisions as dicts[, bf16 params])."""
    model = Probe(probe_sizes(total)).cuda().to(dtype)
    cfg = D.DeftConfig(lr=lr, momentum=momentum, autocast_dtype=None,
                       partition=D.PartitionConfig(partition_size=partition_size),
                       cuda_graphs=cuda_graphs, update_placement=placement, scheme=scheme)
    ddp = D.DeftDataParallel(model, cfg, process_group=group)
    prof = uniform_profile(n_buckets, total // n_buckets, comm_us=comm_us)
    ddp.plan(prof, equal_dual())
    order = list(model.ps)[::-1]  # executor flat order: output-side parameter first

    def loss_fn(module, batch):
        return module(batch)

    for t in range(iterations):
        flat = grad_fn(total, rank, t).cuda().to(dtype)
        xs_exec = [flat[o:o + p.numel()].view_as(p) for o, p in zip(ddp.offsets, order)]
        ddp.train_step(xs_exec[::-1], loss_fn)
    ddp.finish()
    master = ddp.comm.master if ddp.comm.master is not None else ddp.comm.params
    theta = master.detach().float().cpu().clone()
    params = ddp.comm.params.detach().cpu().clone()
    decisions = [d.to_dict() for k in range(iterations) for d in ddp.decisions(k)]
    theta0 = torch.cat([p.detach().to(dtype).float().reshape(-1) for p in
                        Probe(probe_sizes(total)).ps][::-1])
    ddp.close()
    if dtype == torch.bfloat16:
        return theta, theta0, decisions, params
    return theta, theta0, decisions


def oracle_theta(theta0, decisions, world, iterations, total=48_000, lr=0.05, momentum=0.9,
                 grad_fn=flat_grad, lag=2):
    """lag 2: DeFT (visible from t+2); lag 1: the synchronous wfbp/priority schemes."""
    return delayed_sgd.run(theta0, lambda th, r, t: grad_fn(total, r, t), decisions, world,
                           lr, momentum, iterations, lag=lag)


def rel_err(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def run_smoke_executor(iterations=12):
    theta, theta0, decisions = run_executor(1, 0, iterations)
    merges = [u["merge_count"] for d in decisions for u in d["update_events"]]
    want = oracle_theta(theta0, decisions, 1, iterations)
    err = rel_err(theta, want)
    assert err <= TOL, f"executor vs delayed-SGD oracle: rel err {err:.3e}"
    assert max(merges) >= 2, "the smoke profile should merge iterations"
    assert not torch.equal(theta, theta0), "parameters never moved"
    return err
