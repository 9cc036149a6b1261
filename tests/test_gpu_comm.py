"""Reduce-scatter kernels on 2+ GPUs: the one-launch multi-bucket form equals
the per-bucket form and the exact sum, on both channels, f32 and bf16, with
ragged, tiny and unaligned buckets (csrc/bucket_comm.cu, capi.cu)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# (offset, numel) buckets inside one slot: ragged, unaligned, tiny, empty shards
BUCKETS = [(0, 1_000_003), (1_000_003, 7), (1_000_010, 65_536), (1_065_546, 3),
           (1_065_549, 250_001), (1_315_550, 1), (1_315_551, 2_000_000)]


def shard_of(offset, numel, r, world, align):
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


def _run(rank, world, dev):
    import torch.distributed as dist
    from paper_2503_16815_b200 import _native
    from paper_2503_16815_b200.comm import BucketComm
    errs = []
    total = BUCKETS[-1][0] + BUCKETS[-1][1]
    for dtype in (torch.float32, torch.bfloat16):
        comm = BucketComm(rank, world, 2, total, dtype, dev)
        s = torch.cuda.Stream(dev)
        idx = torch.arange(total, device=dev, dtype=torch.float32)
        mine = torch.sin(idx * 0.37 + rank).to(dtype)
        want = sum(torch.sin(idx * 0.37 + r).to(dtype).float() for r in range(world))
        align = 4 if dtype == torch.float32 else 8
        for ch in (_native.CHANNEL_SM, _native.CHANNEL_CE):
            for multi in (True, False):
                comm.grads[1].copy_(mine)
                torch.cuda.synchronize()
                dist.barrier()
                if multi:
                    comm.reduce_scatter_multi(ch, 1, [(o, o + n) for o, n in BUCKETS], s)
                else:
                    for o, n in BUCKETS:
                        comm.reduce_scatter(ch, 1, o, n, s)
                torch.cuda.synchronize()
                got = comm.grads[1].float()
                err = 0.0
                for o, n in BUCKETS:
                    lo, hi = shard_of(o, n, rank, world, align)
                    if hi > lo:
                        ref = want[lo:hi].to(dtype).float()
                        err = max(err, float((got[lo:hi] - ref).abs().max()))
                errs.append((str(dtype), ch, multi, err))
                dist.barrier()
        comm.close()
    return errs


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        q.put((rank, _run(rank, world, dev)))
    except BaseException:
        import traceback
        q.put((rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def test_reduce_scatter_multi_matches_exact_sum():
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(n, 4)
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for rank, errs in res:
        assert not isinstance(errs, str), errs       # a worker's traceback
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errs in res:
        for dtype, ch, multi, err in errs:
            # f32: W-term sums in fp32 (the order may differ from torch's);
            # bf16: one rounding of the fp32 sum (1 ulp at |x| < 4 is 2^-6)
            tol = 1e-5 if dtype == "torch.float32" else 0.02
            assert err <= tol, (rank, dtype, ch, multi, err)
