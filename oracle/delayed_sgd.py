"""ORACLE -- test infrastructure only.

CPU restatement of DeFT's delayed-update data-parallel SGD, driven by a
decision stream in the reference's JSONL schema (scheduler.py:82-96).  The
reference defines WHEN gradients merge and when a group is declared updated
(UpdateEvent, scheduler.py:56-61; merges scheduler.py:223-233) but not the
arithmetic, which SURVEY.md §8c fixes (and DESIGN.md restates):

  * a group's gradient is sum_{o in origins} sum_{ranks} g_o / (W * merge_count)
    (the k*B*W mean, preserver.py:93-94);
  * the step is torch.optim.SGD momentum: v <- m*v + g ; theta <- theta - lr*v
    (dampening 0, no nesterov, no weight decay);
  * events of decision (t, backward) are visible from iteration t+2 (``lag=2``);
    the synchronous baseline schedules (wfbp / priority, ``delayed_updates=False``,
    scheduler.py:386-418) make them visible from t+1 (``lag=1``).

``reduce`` selects how the per-rank gradients are summed: "local" (all ranks'
gradients are known to the caller) or "gloo" (this process is one rank of an
initialised gloo group; torch.distributed.all_reduce does the sum).
"""
from __future__ import annotations

from typing import Callable

import torch


def events_by_iteration(decisions) -> dict[int, list[tuple[tuple[int, ...], int]]]:
    out: dict[int, list] = {}
    for d in decisions:
        if d["stage"] == "backward" and d["update_events"]:
            out[d["iteration"]] = [(tuple(u["origins"]), u["merge_count"])
                                   for u in d["update_events"]]
    return out


def run(theta0: torch.Tensor, grad_of: Callable[[torch.Tensor, int, int], torch.Tensor],
        decisions, world: int, lr: float, momentum: float, iterations: int,
        reduce: str = "local", rank: int = 0, lag: int = 2) -> torch.Tensor:
    """Return theta^(iterations): the parameters the next forward would use.

    grad_of(theta, rank, t) -> this rank's flat fp32 gradient at iteration t,
    evaluated at the parameters iteration t computes with.
    """
    theta = theta0.detach().to(torch.float32).clone()
    v = torch.zeros_like(theta)
    events = events_by_iteration(decisions)
    summed: dict[int, torch.Tensor] = {}
    for s in range(iterations + 1):
        for origins, k in events.get(s - lag, ()):
            g = torch.zeros_like(theta)
            for o in origins:
                g += summed.pop(o)
            g /= world * k
            v.mul_(momentum).add_(g)
            theta.add_(v, alpha=-lr)
        if s == iterations:
            break
        if reduce == "gloo":
            import torch.distributed as dist
            g = grad_of(theta, rank, s).to(torch.float32).clone()
            dist.all_reduce(g)
        else:
            g = torch.zeros_like(theta)
            for r in range(world):
                g += grad_of(theta, r, s).to(torch.float32)
        summed[s] = g
    return theta


def _fma32(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor) -> torch.Tensor:
    """fp32 fused multiply-add (the kernels' fmaf): the product of two fp32
    values is exact in fp64, the sum is rounded once to fp64 and then to fp32
    (double rounding can differ from a single rounding with probability ~2^-29
    per operation)."""
    return (a.double() * b.double() + c.double()).float()


def run_kernel_order(theta0: torch.Tensor, x_of: Callable[[int, int], torch.Tensor],
                     decisions, world: int, lr: float, momentum: float, iterations: int,
                     dtype: torch.dtype = torch.float32, lag: int = 2):
    """Delayed-update SGD for the theta-DEPENDENT probe gradient g = x * theta
    (tests/smoke_executor.py: loss = 1/2 sum x theta^2, x = +-2^-e, so autograd
    computes g exactly in fp32 and bf16), with the same rules as ``run`` but in
    the arithmetic order of the B200 path, so that only the
    order of the cross-rank fp32 sum can differ from it:

      * rank r's gradient at iteration s is  x_of(r, s) * theta_read, in the
        parameter dtype, where theta_read is the dtype copy of the master the
        forward of iteration s reads;
      * a group's gradient on rank r accumulates its origins in origin order in
        the gradient dtype (store, then autograd's in-place adds = merges);
      * the reduce-scatter sums the ranks in fp32 and rounds to the dtype;
      * the update is the kernels' fmaf form with scale = fp32(1/(W*k)):
            v = fma(m, v, g*scale) ; master = fma(-lr, v, master)
        and the parameters are the dtype copy (round to nearest even) of master.

    Returns (master fp32, params in ``dtype``) after ``iterations`` iterations.
    """
    master = theta0.detach().to(torch.float32).clone()
    params = master.to(dtype)
    v = torch.zeros_like(master)
    m32 = torch.tensor(momentum, dtype=torch.float32)
    nlr32 = torch.tensor(-lr, dtype=torch.float32)
    events = events_by_iteration(decisions)
    grads: dict[int, list[torch.Tensor]] = {}
    for s in range(iterations + 1):
        for origins, k in events.get(s - lag, ()):
            acc = None
            for r in range(world):
                slot = None
                for o in origins:
                    g = grads[o][r]
                    slot = g.clone() if slot is None else (slot.float() + g.float()).to(dtype)
                acc = slot.float() if acc is None else acc + slot.float()
            for o in origins:
                grads.pop(o)
            red = acc.to(dtype).float()
            scale = torch.tensor(1.0 / (world * k), dtype=torch.float32)
            v = _fma32(m32, v, red * scale)
            master = _fma32(nlr32, v, master)
            params = master.to(dtype)
        if s == iterations:
            break
        grads[s] = [(x_of(r, s).to(dtype) * params).to(dtype) for r in range(world)]
    return master, params
