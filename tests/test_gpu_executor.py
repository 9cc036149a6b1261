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
    theta, params, theta0, decisions, buckets = S.run_executor(
        1, 0, iterations, comm_us=comm_us, cuda_graphs=graphs, placement=placement)
    want_m, want_p = S.oracle_theta(theta0, decisions, 1, iterations)
    S.check_ranks([theta], [params], want_m, want_p, 1, torch.float32, buckets)


@pytest.mark.parametrize("scheme", ["wfbp", "priority"])
@pytest.mark.parametrize("placement", ["end", "bucket", "start"])
@pytest.mark.parametrize("graphs", [True, False])
def test_single_gpu_synchronous_baselines(scheme, placement, graphs):
    """The reference's synchronous schedules (scheduler.py:386-418) on the same
    executor and kernels: updates of iteration t visible from t+1 (oracle lag 1).
    priority: partition_by_size blocks (1000-element buckets cut into 334/333/333)."""
    iters = 12
    theta, params, theta0, decisions, buckets = S.run_executor(
        1, 0, iters, cuda_graphs=graphs, placement=placement, scheme=scheme,
        partition_size=400 if scheme == "priority" else 10**9)
    assert all(u["merge_count"] == 1 for d in decisions for u in d["update_events"])
    want_m, want_p = S.oracle_theta(theta0, decisions, 1, iters, lag=1)
    S.check_ranks([theta], [params], want_m, want_p, 1, torch.float32, buckets)
    # and it is NOT the delayed trajectory
    assert S.elem_err(theta, S.oracle_theta(theta0, decisions, 1, iters, lag=2)[0]) > 1e-4


@pytest.mark.parametrize("placement", ["end", "start"])
@pytest.mark.parametrize("graphs", [True, False])
def test_bf16_params_single_gpu(graphs, placement):
    """bf16 model (bf16 grads, as the GPT-2 config): the fp32 master follows the
    oracle within 1e-6 and the bf16 parameters are its round-to-nearest copy."""
    iters = 16
    theta, params, theta0, decisions, buckets = S.run_executor(
        1, 0, iters, dtype=torch.bfloat16, cuda_graphs=graphs, placement=placement)
    assert max(u["merge_count"] for d in decisions for u in d["update_events"]) >= 2
    want_m, want_p = S.oracle_theta(theta0, decisions, 1, iters, dtype=torch.bfloat16)
    S.check_ranks([theta], [params], want_m, want_p, 1, torch.bfloat16, buckets)
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
        out = S.run_executor(
            world, rank, iterations, comm_us=comm_us, cuda_graphs=graphs,
            dtype=torch.bfloat16 if bf16 else torch.float32, placement=placement,
            scheme=scheme, partition_size=400 if scheme == "priority" else 10**9)
        q.put((rank,) + out)
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
    _collect_and_check(q, procs, world, iterations, lag=2)


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
    _collect_and_check(q, procs, world, iterations, lag=1)


def _collect_and_check(q, procs, world, iterations, lag, dtype=torch.float32):
    res = {}
    for _ in range(world):
        r, theta, params, theta0, decisions, buckets = q.get(timeout=300)
        res[r] = (theta, params, theta0, decisions, buckets)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    theta0, decisions, buckets = res[0][2], res[0][3], res[0][4]
    for r in range(world):
        assert res[r][3] == decisions          # every rank planned the same stream
    want_m, want_p = S.oracle_theta(theta0, decisions, world, iterations, lag=lag,
                                    dtype=dtype)
    S.check_ranks([res[r][0] for r in range(world)], [res[r][1] for r in range(world)],
                  want_m, want_p, world, dtype, buckets)


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
    _collect_and_check(q, procs, world, iterations, lag=2, dtype=torch.bfloat16)


class _ProbeWithUnused(S.Probe):
    """One parameter never takes part in the loss: its gradient is None every
    iteration, and the executor must treat its bucket range as a zero gradient."""

    def forward(self, xs):
        return 0.5 * sum((x * p * p).sum() for i, (p, x) in enumerate(zip(self.ps, xs))
                         if i != 3)


@pytest.mark.parametrize("graphs", [True, False])
def test_unused_parameter_gets_zero_gradient(graphs):
    iters = 10
    theta, params, theta0, decisions, buckets = S.run_executor(
        1, 0, iters, cuda_graphs=graphs, model_cls=_ProbeWithUnused)
    sizes = S.probe_sizes()
    order = list(range(len(sizes)))[::-1]            # executor flat order
    offs, o = {}, 0
    for i in order:
        offs[i] = (o, o + sizes[i])
        o += sizes[i]
    lo, hi = offs[3]

    def x_fn(total, r, t):
        x = S.flat_x(total, r, t)
        x[lo:hi] = 0
        return x
    want_m, want_p = S.oracle_theta(theta0, decisions, 1, iters, x_fn=x_fn)
    S.check_ranks([theta], [params], want_m, want_p, 1, torch.float32, buckets)
    assert torch.equal(theta[lo:hi], theta0[lo:hi])   # zero grads, zero momentum: unchanged


@pytest.mark.parametrize("hw_probe", [True, False])
@pytest.mark.parametrize("placement", ["end", "start"])
def test_single_gpu_nonsequential(hw_probe, placement):
    """The reference's non-sequential baseline (scheduler.py:421-472) on the
    executor: four candidate block structures x orders scored by timing 8
    iterations of each on the GPU (or by the reference's simulator rules),
    the state restored after the probe; the run then matches the lag-1 oracle
    from theta0."""
    iters = 10
    theta, params, theta0, decisions, buckets = S.run_executor(
        1, 0, iters, placement=placement, scheme="nonsequential", partition_size=400,
        startup_us=500, hw_probe=hw_probe)
    assert all(u["merge_count"] == 1 for d in decisions for u in d["update_events"])
    want_m, want_p = S.oracle_theta(theta0, decisions, 1, iters, lag=1)
    S.check_ranks([theta], [params], want_m, want_p, 1, torch.float32, buckets)
