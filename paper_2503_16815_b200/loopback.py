"""Loopback world: W data-parallel ranks in ONE process on ONE GPU.

The bucket communication kernels (csrc/bucket_comm.cu) only need, per rank,
the device pointers of every rank's gradient arena, parameter buffer and
barrier flags.  In a loopback world those are ordinary allocations on the same
device, so the unchanged reduce-scatter / copy-engine / fused update +
all-gather kernels run -- barriers, epochs and all -- for W = 2..8 on a single
B200.  That is how the multi-rank paths are checked against the delayed-SGD
oracle on a one-GPU box (tests/test_gpu_loopback.py, ``smoke()``).

What makes it safe to drive every rank from one host thread:

* every kernel that meets its peers in a barrier is capped at
  ``grid_cap`` = 148 / (2W) CTAs (deft_comm_configure), so all ranks' blocks of
  one barrier kernel are co-resident with room left for the ranks' compute;
* each rank has exactly two streams -- compute and ONE in-order comm stream
  (its links, gathers and updates collapse onto it).  Every rank issues the
  same program in the same order, so the k-th barrier kernel of every rank's
  comm stream is the same logical transfer, and the host can issue rank 0's
  whole iteration before rank 1's: rank 0's kernels simply wait on the device;
* 2W streams stay within CUDA_DEVICE_MAX_CONNECTIONS (set to 32 before the
  CUDA context exists) so no two ranks' streams share a hardware queue;
* nothing may make the host or the device wait for the WHOLE device while a
  rank's barrier kernel waits for a peer whose work is not issued yet (no
  cudaFree either: ``issuing()`` keeps the garbage collector off the loop):
  kernels are loaded eagerly (CUDA_MODULE_LOADING=EAGER, set before the CUDA
  context exists -- a lazily loaded kernel's first launch waits for the
  device), and a new CUDA-graph shape is captured by every rank before any
  rank replays it (``flush``; cudaGraphInstantiate synchronizes the device);
* the barrier spin is bounded (``spin_timeout_ms``): a violated assumption
  traps instead of hanging the GPU.

The host must never block on device work while some rank's iteration is only
partly issued (no device-wide synchronize, no ``.item()``, no pageable H2D
copies inside the loop): ``DeftDataParallel`` follows that in loopback mode.

This is a test / bring-up harness: NVLink is not involved, all W ranks share
one GPU's HBM bandwidth.
"""
from __future__ import annotations

import os

import torch

# must be in the environment before the CUDA context is created (no effect after)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

SMS = 148  # B200


class LoopbackRank:
    """The process-group stand-in one rank's executor receives."""

    def __init__(self, world: "LoopbackWorld", rank: int):
        self.lb = world
        self.rank = rank
        self.world = world.world
        self.device = world.device
        self.compute_stream = torch.cuda.Stream(world.device)
        self.comm_stream = torch.cuda.Stream(world.device)

    # -- the few collectives the executor needs, in rank order (rank 0 first)
    def broadcast_(self, key: str, t: torch.Tensor) -> None:
        """Overwrite ``t`` with rank 0's tensor of the same key (ranks are set
        up in rank order, so rank 0's is registered first)."""
        if self.rank == 0:
            self.lb._shared[key] = t
        else:
            t.copy_(self.lb._shared[key])

    def broadcast_obj(self, key: str, obj):
        if self.rank == 0:
            self.lb._shared[key] = obj
            return obj
        return self.lb._shared[key]

    def defer_replay(self, graph, stream) -> None:
        """A freshly captured graph is replayed by LoopbackWorld.flush() once
        every rank has captured its own: cudaGraphInstantiate synchronizes the
        device, which would wait for a peer's replayed kernels that wait for
        this rank."""
        self.lb._pending.append((self.rank, graph, stream))

    def comm(self, n_slots: int, slot_elems: int, grad_dtype: torch.dtype):
        self._key = (n_slots, slot_elems, grad_dtype)
        return self.lb._comm(self.rank, n_slots, slot_elems, grad_dtype)

    def peers(self) -> list:
        """Every rank's communicator of the world this rank's comm belongs to."""
        return self.lb._comms[self._key]


class LoopbackWorld:
    def __init__(self, world: int, device: torch.device | int | None = None,
                 grid_cap: int | None = None, spin_timeout_ms: int = 60_000):
        if not 1 <= world <= 8:
            raise ValueError("loopback world size must be 1..8")
        self.world = world
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else (device.index if isinstance(device, torch.device)
                                         else device))
        self.grid_cap = grid_cap or max(1, SMS // (2 * world))
        self.spin_timeout_ms = spin_timeout_ms
        self._shared: dict = {}
        self._comms: dict = {}
        self._pending: list = []
        self.ranks = [LoopbackRank(self, r) for r in range(world)]

    def rank(self, r: int) -> LoopbackRank:
        return self.ranks[r]

    def make_comms(self, n_slots: int, slot_elems: int, grad_dtype: torch.dtype) -> list:
        """One BucketComm per rank over the same device, every rank's pointers
        mapped into every communicator (no IPC: they are all local)."""
        from .comm import BucketComm, PeerMaps
        comms = [BucketComm(r, self.world, n_slots, slot_elems, grad_dtype, self.device,
                            connect=False) for r in range(self.world)]
        maps = PeerMaps([c._g.ptr.value for c in comms], [c._p.ptr.value for c in comms],
                        [c._f.ptr.value for c in comms])
        for c in comms:
            c._connect(maps)
            c.configure(self.grid_cap, self.spin_timeout_ms)
        return comms

    def _comm(self, rank, n_slots, slot_elems, grad_dtype):
        key = (n_slots, slot_elems, grad_dtype)
        if rank == 0 or key not in self._comms:
            self._comms[key] = self.make_comms(n_slots, slot_elems, grad_dtype)
        return self._comms[key][rank]

    # -- collectives: one launch for all ranks (work under kernel serialization)
    def collective_reduce_scatter(self, comms, channel: int, slot: int, ranges, stream) -> None:
        """deft_loopback_reduce_scatter: every rank's reduce-scatter of the bucket
        list in ONE launch (synchronous)."""
        import ctypes

        from . import _native
        n, w = len(ranges), self.world
        _native.check(_native.lib().deft_loopback_reduce_scatter(
            (ctypes.c_void_p * w)(*[c._h.value for c in comms]), w, channel, slot, n,
            (ctypes.c_int64 * n)(*[lo for lo, _ in ranges]),
            (ctypes.c_int64 * n)(*[hi - lo for lo, hi in ranges]),
            ctypes.c_void_p(stream.cuda_stream)), "deft_loopback_reduce_scatter")

    def collective_update(self, comms, slot: int, ranges, scale: float, lr: float,
                          momentum: float, moms, stream) -> None:
        """deft_loopback_update: every rank's fused update of its owned shards +
        parameter all-gather in ONE launch (synchronous)."""
        import ctypes

        from . import _native
        n, w = len(ranges), self.world
        _native.check(_native.lib().deft_loopback_update(
            (ctypes.c_void_p * w)(*[c._h.value for c in comms]), w, slot, n,
            (ctypes.c_int64 * n)(*[lo for lo, _ in ranges]),
            (ctypes.c_int64 * n)(*[hi - lo for lo, hi in ranges]), lr, momentum, scale,
            (ctypes.c_void_p * w)(*[m.data_ptr() for m in moms]),
            ctypes.c_void_p(stream.cuda_stream)), "deft_loopback_update")

    def kernels_run_concurrently(self, timeout_us: int = 50_000) -> bool:
        """False when the device serializes kernels (a kernel profiler): then the
        ranks' separate launches can never meet in a barrier and only the
        collectives above work.  Measured with deft_stream_alias_probe."""
        import ctypes

        from . import _native
        lib = _native.lib()
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(lib.deft_stream_create(0, ctypes.byref(a)), "deft_stream_create")
        _native.check(lib.deft_stream_create(0, ctypes.byref(b)), "deft_stream_create")
        try:
            out = ctypes.c_int32()
            _native.check(lib.deft_stream_alias_probe(a, b, timeout_us, 0, ctypes.byref(out)),
                          "deft_stream_alias_probe")
            return out.value == 0
        finally:
            lib.deft_stream_destroy(a)
            lib.deft_stream_destroy(b)

    def issuing(self):
        """Context for the round-robin issue loop: garbage from earlier objects
        is collected (and the device drained) BEFORE it, and the cyclic garbage
        collector is off DURING it -- a region freed by the collector mid-loop
        means cudaFree, which synchronizes the device and so waits for a rank's
        barrier kernel whose peers this thread has not issued yet."""
        import contextlib
        import gc

        @contextlib.contextmanager
        def ctx():
            gc.collect()
            torch.cuda.synchronize(self.device)
            was = gc.isenabled()
            gc.disable()
            try:
                yield self
            finally:
                if was:
                    gc.enable()
        return ctx()

    def flush(self) -> None:
        """Replay the graphs the ranks captured this round, in rank order.  Call
        after every rank's train_step of an iteration."""
        pending, self._pending = self._pending, []
        for _, g, stream in sorted(pending, key=lambda x: x[0]):
            with torch.cuda.stream(stream):
                g.replay()

    def synchronize(self) -> None:
        self.flush()
        torch.cuda.synchronize(self.device)


__all__ = ["LoopbackWorld", "LoopbackRank"]
