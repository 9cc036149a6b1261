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
