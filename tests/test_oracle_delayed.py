"""CPU checks of the delayed-SGD oracle (oracle/delayed_sgd.py): the
kernel-order restatement used by the GPU parity tests is the same math as the
plain torch.optim.SGD semantics of SURVEY §8c, on the theta-dependent probe
and the decision stream of the reference's uniform48 / equal_dual fixture."""
import json

import pytest

torch = pytest.importorskip("torch")

import smoke_executor as S  # noqa: E402
from conftest import uniform_buckets  # noqa: E402
from oracle import deft_oracle as O  # noqa: E402
from oracle import delayed_sgd  # noqa: E402


@pytest.fixture(scope="module")
def decisions():
    lines = O.schedule(uniform_buckets(48), [1.0, 1.0000001], ["fast", "twin"], 14)
    return [json.loads(x) if isinstance(x, str) else x for x in lines]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("lag", [1, 2])
def test_kernel_order_equals_sgd_semantics(decisions, world, lag):
    th0 = S.theta0_for(48_000, torch.float32)
    m, p = S.oracle_theta(th0, decisions, world, 14, lag=lag)
    ref = delayed_sgd.run(th0, lambda th, r, t: S.flat_x(48_000, r, t) * th, decisions,
                          world, 0.05, 0.9, 14, lag=lag)
    assert S.elem_err(m, ref) <= 1e-6
    assert torch.equal(p, m)
    assert float((m - th0).abs().max()) > 0.1          # the probe really trains


def test_merges_present(decisions):
    assert max(u["merge_count"] for d in decisions for u in d["update_events"]) >= 2


def test_bf16_params_are_rounded_master(decisions):
    th0 = S.theta0_for(48_000, torch.bfloat16)
    m, p = S.oracle_theta(th0, decisions, 4, 14, dtype=torch.bfloat16)
    assert p.dtype == torch.bfloat16 and torch.equal(p, m.bfloat16())


def test_probe_gradient_is_exact():
    """autograd's gradient of 1/2 sum x theta^2 is x * theta bit for bit
    (fp32 and bf16) for x = +-2^-e -- what makes the GPU parity exact."""
    sizes = S.probe_sizes()
    for dtype in (torch.float32, torch.bfloat16):
        model = S.Probe(sizes).to(dtype)
        xs = [S.flat_x(n, 0, 3)[:n].to(dtype) for n in sizes]
        model(xs).backward()
        for p, x in zip(model.ps, xs):
            assert torch.equal(p.grad, (x * p.detach()).to(dtype))


@pytest.mark.parametrize("world", [1, 4])
@pytest.mark.parametrize("lag", [1, 2])
@pytest.mark.parametrize("foreach", [False, True])
def test_oracle_is_torch_optim_sgd(decisions, world, lag, foreach):
    """Pins the oracle's update arithmetic to a library implementation: the same
    delayed group gradients fed to torch.optim.SGD(momentum=0.9, dampening 0) --
    one .step() per update event, p.grad = the k*W mean of the group -- give
    theta bit for bit (the reference fixes only WHICH gradients form a group and
    WHEN it applies, scheduler.py:56-61, 223-233; preserver.py:93-94)."""
    total, iters, lr, m = 48_000, 14, 0.05, 0.9
    th0 = S.theta0_for(total, torch.float32)
    grad_of = lambda th, r, t: S.flat_x(total, r, t) * th   # noqa: E731
    want = delayed_sgd.run(th0, grad_of, decisions, world, lr, m, iters, lag=lag)
    p = torch.nn.Parameter(th0.clone())
    opt = torch.optim.SGD([p], lr=lr, momentum=m, foreach=foreach)
    events = delayed_sgd.events_by_iteration(decisions)
    summed = {}
    for s in range(iters + 1):
        for origins, k in events.get(s - lag, ()):
            g = torch.zeros_like(th0)
            for o in origins:
                g += summed.pop(o)
            g /= world * k
            p.grad = g
            opt.step()
        if s == iters:
            break
        with torch.no_grad():
            summed[s] = sum(grad_of(p.detach(), r, s) for r in range(world))
    assert torch.equal(p.detach(), want)
