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


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("iterations,comm_us", [(12, 900), (25, 900), (20, 300), (16, 1900)])
def test_single_gpu_matches_oracle(iterations, comm_us, graphs):
    theta, theta0, decisions = S.run_executor(1, 0, iterations, comm_us=comm_us,
                                              cuda_graphs=graphs)
    want = S.oracle_theta(theta0, decisions, 1, iterations)
    assert S.rel_err(theta, want) <= S.TOL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, iterations, comm_us, graphs, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        theta, theta0, decisions = S.run_executor(world, rank, iterations, comm_us=comm_us,
                                                  cuda_graphs=graphs)
        q.put((rank, theta, theta0, decisions))
    finally:
        dist.destroy_process_group()


@pytest.mark.multigpu
@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("iterations,comm_us", [(14, 900), (20, 1900)])
def test_multi_gpu_matches_oracle(iterations, comm_us, graphs):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, iterations, comm_us, graphs, q))
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
