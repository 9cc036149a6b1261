"""Delayed-update parity of the executor (comm + fused SGD/momentum kernels)
against the CPU oracle, on 1 GPU and -- when the box has them -- 2+ GPUs."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import smoke_executor as S  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("placement", ["end", "bucket", "start"])
@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("iterations,comm_us", [(12, 900), (25, 900), (20, 300), (16, 1900)])
def test_single_gpu_matches_oracle(iterations, comm_us, graphs, placement):
    theta, theta0, decisions = S.run_executor(1, 0, iterations, comm_us=comm_us,
                                              cuda_graphs=graphs, placement=placement)
    want = S.oracle_theta(theta0, decisions, 1, iterations)
    assert S.rel_err(theta, want) <= S.TOL


@pytest.mark.parametrize("scheme", ["wfbp", "priority"])
@pytest.mark.parametrize("placement", ["end", "bucket", "start"])
@pytest.mark.parametrize("graphs", [True, False])
def test_single_gpu_synchronous_baselines(scheme, placement, graphs):
    """The reference's synchronous schedules (scheduler.py:386-418) on the same
    executor and kernels: updates of iteration t visible from t+1 (oracle lag 1).
    priority: partition_by_size blocks (1000-element buckets cut into 334/333/333)."""
    iters = 12
    theta, theta0, decisions = S.run_executor(
        1, 0, iters, cuda_graphs=graphs, placement=placement, scheme=scheme,
        partition_size=400 if scheme == "priority" else 10**9)
    assert all(u["merge_count"] == 1 for d in decisions for u in d["update_events"])
    want = S.oracle_theta(theta0, decisions, 1, iters, lag=1)
    assert S.rel_err(theta, want) <= S.TOL
    # and it is NOT the delayed trajectory
    assert S.rel_err(theta, S.oracle_theta(theta0, decisions, 1, iters, lag=2)) > 1e-4


@pytest.mark.parametrize("placement", ["end", "start"])
@pytest.mark.parametrize("graphs", [True, False])
def test_bf16_params_single_gpu(graphs, placement):
    """bf16 model (bf16 grads, as the GPT-2 config): the fp32 master follows the
    oracle within 1e-6 and the bf16 parameters are its round-to-nearest copy."""
    iters = 16
    theta, theta0, decisions, params = S.run_executor(
        1, 0, iters, dtype=torch.bfloat16, cuda_graphs=graphs, grad_fn=S.flat_grad_dyadic,
        placement=placement)
    assert max(u["merge_count"] for d in decisions for u in d["update_events"]) >= 2
    want = S.oracle_theta(theta0, decisions, 1, iters, grad_fn=S.flat_grad_dyadic)
    assert S.rel_err(theta, want) <= S.TOL
    assert torch.equal(params, theta.bfloat16())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, iterations, comm_us, graphs, q, bf16=False, placement="end",
            scheme="deft"):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        if bf16:
            theta, theta0, decisions, params = S.run_executor(
                world, rank, iterations, comm_us=comm_us, cuda_graphs=graphs,
                dtype=torch.bfloat16, grad_fn=S.flat_grad_dyadic, placement=placement)
            q.put((rank, theta, theta0, decisions, params))
        else:
            theta, theta0, decisions = S.run_executor(
                world, rank, iterations, comm_us=comm_us, cuda_graphs=graphs,
                placement=placement, scheme=scheme,
                partition_size=400 if scheme == "priority" else 10**9)
            q.put((rank, theta, theta0, decisions))
    finally:
        dist.destroy_process_group()


@pytest.mark.multigpu
@pytest.mark.parametrize("graphs,placement", [(True, "end"), (False, "end"), (True, "start"),
                                              (False, "bucket")])
@pytest.mark.parametrize("iterations,comm_us", [(14, 900), (20, 1900)])
def test_multi_gpu_matches_oracle(iterations, comm_us, graphs, placement):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, iterations, comm_us, graphs, q, False,
                                             placement))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, theta, theta0, decisions = q.get(timeout=300)
        res[r] = (theta, theta0, decisions)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    theta0, decisions = res[0][1], res[0][2]
    want = S.oracle_theta(theta0, decisions, world, iterations)
    for r in range(world):
        assert res[r][2] == decisions          # every rank planned the same stream
        assert S.rel_err(res[r][0], want) <= S.TOL, r
        assert torch.equal(res[r][0], res[0][0])  # replicas bit-identical


@pytest.mark.multigpu
@pytest.mark.parametrize("scheme,graphs,placement", [
    ("wfbp", True, "end"), ("wfbp", False, "bucket"), ("priority", True, "start"),
    ("priority", False, "end")])
def test_multi_gpu_synchronous_baselines(scheme, graphs, placement):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    iterations = 10
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, iterations, 900, graphs, q,
                                             False, placement, scheme))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, theta, theta0, decisions = q.get(timeout=300)
        res[r] = (theta, theta0, decisions)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    theta0, decisions = res[0][1], res[0][2]
    want = S.oracle_theta(theta0, decisions, world, iterations, lag=1)
    for r in range(world):
        assert res[r][2] == decisions
        assert S.rel_err(res[r][0], want) <= S.TOL, r
        assert torch.equal(res[r][0], res[0][0])


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


@pytest.mark.multigpu
@pytest.mark.parametrize("placement", ["end", "start"])
def test_multi_gpu_bf16_matches_oracle(placement):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world, iterations = min(n, 4), 14
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, iterations, 900, True, q, True,
                                               placement))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, theta, theta0, decisions, params = q.get(timeout=300)
        res[r] = (theta, theta0, decisions, params)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    theta0, decisions = res[0][1], res[0][2]
    want = S.oracle_theta(theta0, decisions, world, iterations, grad_fn=S.flat_grad_dyadic)
    for r in range(world):
        theta, _, dec, params = res[r]
        assert dec == decisions
        assert torch.equal(params, res[0][3])        # every rank holds the same bf16 params
        for b in range(48):                          # uniform48 probe buckets of 1000
            lo, hi = shard_range(1000 * b, 1000, r, world, 8)
            # the owner's fp32 master shard follows the oracle within 1e-6
            assert S.rel_err(theta[lo:hi], want[lo:hi]) <= S.TOL, (r, b)
            assert torch.equal(params[lo:hi], theta[lo:hi].bfloat16())


class _ProbeWithUnused(S.Probe):
    """One parameter never takes part in the loss: its gradient is None every
    iteration, and the executor must treat its bucket range as a zero gradient."""

    def forward(self, xs):
        return sum((p * x).sum() for i, (p, x) in enumerate(zip(self.ps, xs)) if i != 3)


@pytest.mark.parametrize("graphs", [True, False])
def test_unused_parameter_gets_zero_gradient(graphs, monkeypatch):
    monkeypatch.setattr(S, "Probe", _ProbeWithUnused)
    iters = 10
    theta, theta0, decisions = S.run_executor(1, 0, iters, cuda_graphs=graphs)
    sizes = S.probe_sizes()
    order = list(range(len(sizes)))[::-1]            # executor flat order
    offs, o = {}, 0
    for i in order:
        offs[i] = (o, o + sizes[i])
        o += sizes[i]
    lo, hi = offs[3]

    def grad(total, r, t):
        g = S.flat_grad(total, r, t)
        g[lo:hi] = 0
        return g
    want = S.oracle_theta(theta0, decisions, 1, iters, grad_fn=grad)
    assert S.rel_err(theta, want) <= S.TOL
    assert torch.equal(theta[lo:hi], theta0[lo:hi])   # zero grads, zero momentum: unchanged
