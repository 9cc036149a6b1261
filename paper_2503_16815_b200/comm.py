"""Symmetric device memory and the bucket communicator (one process per GPU).

Each rank cudaMalloc's its gradient arena, parameter buffer and barrier flags
inside libdeft_b200.so, exports CUDA IPC handles, exchanges them through
``torch.distributed`` (plumbing only -- no collective touches the data path)
and maps every peer's buffers.  The kernels then read peers' gradient slots and
write peers' parameters directly over NVLink / NVSwitch.

This replaces the reference's abstract links (profiles.py:18-40; durations
simulator.py:136-147): link 0 / "fast" is the SM-driven P2P channel, the
second link is the copy-engine channel.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native
from ._native import CHANNEL_CE, CHANNEL_SM, DTYPE_BF16, DTYPE_F32, IPC_HANDLE_BYTES, c_vp, check

_TYPESTR = {torch.float32: "<f4", torch.bfloat16: "<i2", torch.uint8: "|u1"}


class _Region:
    """A raw device allocation exposed through __cuda_array_interface__ so that
    torch.as_tensor wraps it without a copy.  Freed when the last tensor dies."""

    def __init__(self, nbytes: int, ipc: bool):
        self.ptr = c_vp()
        self.nbytes = nbytes
        self.handle = (ctypes.c_uint8 * IPC_HANDLE_BYTES)() if ipc else None
        check(_native.lib().deft_mem_alloc(nbytes, ctypes.byref(self.ptr), self.handle),
              "deft_mem_alloc")
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (self.ptr.value, False), "version": 3}

    def __del__(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value and _native._lib is not None:
            _native.lib().deft_mem_free(self.ptr)
            self.ptr = None


def region_tensor(nbytes: int, dtype: torch.dtype, ipc: bool, device: torch.device):
    reg = _Region(nbytes, ipc)
    raw = torch.as_tensor(reg, device=device)  # uint8 view, keeps `reg` alive
    if raw.data_ptr() != reg.ptr.value:
        raise RuntimeError("torch.as_tensor copied the symmetric region")
    t = raw.view(torch.int16 if dtype == torch.bfloat16 else dtype)
    return (t.view(torch.bfloat16) if dtype == torch.bfloat16 else t), reg


@dataclass
class PeerMaps:
    grads: list[int]
    params: list[int]
    flags: list[int]


class BucketComm:
    """Per-rank communicator over the symmetric gradient arena / params / flags."""

    def __init__(self, rank: int, world: int, n_slots: int, slot_elems: int,
                 grad_dtype: torch.dtype, device: torch.device, group=None,
                 connect: bool = True):
        """``connect=False`` only allocates this rank's regions; a loopback
        world (loopback.py) maps every rank's pointers and calls ``_connect``."""
        self.rank, self.world = rank, world
        self.group = group
        self.n_slots, self.slot_elems = n_slots, slot_elems
        self.grad_dtype = grad_dtype
        self.device = device
        esz = 2 if grad_dtype == torch.bfloat16 else 4
        ipc = world > 1 and connect
        # slots start 256-byte aligned (the kernels' vector and TMA bulk accesses
        # are aligned relative to the slot base)
        self.slot_stride = -(-slot_elems // 128) * 128
        self.grads, self._g = region_tensor(n_slots * self.slot_stride * esz, grad_dtype, ipc,
                                            device)
        self.grads = self.grads.view(n_slots, self.slot_stride)[:, :slot_elems]
        # parameters share the gradient dtype (autograd requires it); bf16 models
        # keep an fp32 master copy that only the update kernel touches
        # padded like a slot, so every range the C-ABI accepts is inside all buffers
        self.params, self._p = region_tensor(self.slot_stride * esz, grad_dtype, ipc, device)
        self.params = self.params[:slot_elems]
        self._master_buf = (torch.zeros(self.slot_stride, dtype=torch.float32, device=device)
                            if grad_dtype == torch.bfloat16 else None)
        self.master = self._master_buf[:slot_elems] if self._master_buf is not None else None
        fbytes = int(_native.lib().deft_comm_flag_bytes(world))
        self.flags, self._f = region_tensor(fbytes, torch.uint8, ipc, device)
        self._opened: list[c_vp] = []
        self._h = None
        self.loopback = not connect
        if not connect:
            return
        if world > 1:
            maps = self._exchange(group)
        else:
            maps = self.own_maps()
        self._connect(maps)

    def own_maps(self) -> PeerMaps:
        return PeerMaps([self._g.ptr.value], [self._p.ptr.value], [self._f.ptr.value])

    def _connect(self, maps: PeerMaps) -> None:
        arr = lambda xs: (c_vp * self.world)(*xs)  # noqa: E731
        h = c_vp()
        check(_native.lib().deft_comm_create(
            self.rank, self.world, arr(maps.grads), arr(maps.params), arr(maps.flags),
            c_vp(self.master.data_ptr() if self.master is not None else None), self.slot_stride,
            self.n_slots,
            DTYPE_BF16 if self.grad_dtype == torch.bfloat16 else DTYPE_F32, ctypes.byref(h)),
            "deft_comm_create")
        self._h = h

    def configure(self, grid_cap: int = -1, spin_timeout_ms: int = -1) -> None:
        """deft_comm_configure: CTA cap of the peer-barrier kernels and the
        barrier spin timeout (negative = unchanged); equal on every rank."""
        check(_native.lib().deft_comm_configure(self._h, int(grid_cap), int(spin_timeout_ms)),
              "deft_comm_configure")

    def set_phase_trace(self, stamps) -> None:
        """Diagnostics: a device uint64 tensor (>= 256 x 8) that the TMA reduce-
        scatter / update and one-shot kernels stamp with globaltimer ns at their
        phase boundaries (deft_comm_set_phase_trace), or None to stop.  Every launch
        captures the pointer by value: keep the tensor alive until those launches
        have completed (e.g. a synchronize before it is freed)."""
        ptr = None if stamps is None else _native.c_vp(stamps.data_ptr())
        check(_native.lib().deft_comm_set_phase_trace(self._h, ptr), "deft_comm_set_phase_trace")

    def _exchange(self, group) -> PeerMaps:
        import torch.distributed as dist
        mine = [bytes(r.handle) for r in (self._g, self._p, self._f)]
        allh: list = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        out = PeerMaps([], [], [])
        for r in range(self.world):
            if r == self.rank:
                out.grads.append(self._g.ptr.value)
                out.params.append(self._p.ptr.value)
                out.flags.append(self._f.ptr.value)
                continue
            for lst, hbytes in zip((out.grads, out.params, out.flags), allh[r]):
                p = c_vp()
                hb = (ctypes.c_uint8 * IPC_HANDLE_BYTES).from_buffer_copy(hbytes)
                check(_native.lib().deft_mem_open(hb, ctypes.byref(p)), "deft_mem_open")
                self._opened.append(p)
                lst.append(p.value)
        dist.barrier(group=group)
        return out

    def reduce_scatter(self, channel: int, slot: int, offset: int, numel: int, stream) -> None:
        check(_native.lib().deft_bucket_reduce_scatter(self._h, channel, slot, offset, numel,
                                                       c_vp(stream.cuda_stream)),
              "deft_bucket_reduce_scatter")

    def reduce_scatter_multi(self, channel: int, slot: int, ranges, stream) -> None:
        """Buckets released together on one link, one launch / one barrier
        (deft_bucket_reduce_scatter_multi); ``ranges`` = [(lo, hi), ...] in plan order."""
        n = len(ranges)
        offs = (ctypes.c_int64 * n)(*[lo for lo, _ in ranges])
        lens = (ctypes.c_int64 * n)(*[hi - lo for lo, hi in ranges])
        check(_native.lib().deft_bucket_reduce_scatter_multi(
            self._h, channel, slot, n, offs, lens, c_vp(stream.cuda_stream)),
            "deft_bucket_reduce_scatter_multi")

    def set_update_blocks(self, blocks: int) -> None:
        """CTA budget of the update kernels (0 = default); identical on every rank."""
        check(_native.lib().deft_comm_set_update_blocks(self._h, int(blocks)),
              "deft_comm_set_update_blocks")

    def update(self, slot: int, offset: int, numel: int, lr: float, momentum: float,
               grad_scale: float, mom: torch.Tensor, stream) -> None:
        check(_native.lib().deft_bucket_update(self._h, slot, offset, numel, lr, momentum,
                                               grad_scale, c_vp(mom.data_ptr()),
                                               c_vp(stream.cuda_stream)),
              "deft_bucket_update")

    def gather(self, slot: int, srcs, byte_offsets, byte_lens, stream,
               ce_min_bytes: int = 0) -> None:
        """Gather device byte ranges into slot `slot` (deft_gather_segments);
        ranges >= ce_min_bytes (> 0) are copied by the copy engines."""
        n = len(srcs)
        esz = 2 if self.grad_dtype == torch.bfloat16 else 4
        dst = self._g.ptr.value + slot * self.slot_stride * esz
        check(_native.lib().deft_gather_segments(
            c_vp(dst), (c_vp * n)(*srcs), (ctypes.c_int64 * n)(*byte_offsets),
            (ctypes.c_int64 * n)(*byte_lens), n, int(ce_min_bytes), c_vp(stream.cuda_stream)),
            "deft_gather_segments")

    def update_multi(self, slot: int, ranges, scale: float, lr: float, momentum: float,
                     mom: torch.Tensor, stream) -> None:
        """Every bucket of one update event in ONE launch (deft_bucket_update_multi):
        the local fused update at W == 1, update + parameter all-gather at W > 1."""
        n = len(ranges)
        offs = (ctypes.c_int64 * n)(*[lo for lo, _ in ranges])
        lens = (ctypes.c_int64 * n)(*[hi - lo for lo, hi in ranges])
        check(_native.lib().deft_bucket_update_multi(
            self._h, slot, n, offs, lens, lr, momentum, scale, c_vp(mom.data_ptr()),
            c_vp(stream.cuda_stream)), "deft_bucket_update_multi")

    def sync_update_multi(self, slot: int, ranges, scale: float, lr: float, momentum: float,
                          mom: torch.Tensor, stream) -> None:
        """One-shot bucket sync (deft_bucket_sync_update_multi): the all-reduce of
        the full buckets fused with their update, one launch, no reduce-scatter
        before it and no all-gather after it."""
        n = len(ranges)
        offs = (ctypes.c_int64 * n)(*[lo for lo, _ in ranges])
        lens = (ctypes.c_int64 * n)(*[hi - lo for lo, hi in ranges])
        check(_native.lib().deft_bucket_sync_update_multi(
            self._h, slot, n, offs, lens, lr, momentum, scale, c_vp(mom.data_ptr()),
            c_vp(stream.cuda_stream)), "deft_bucket_sync_update_multi")

    def close(self, barrier: bool = True) -> None:
        if getattr(self, "_h", None) is not None:
            torch.cuda.synchronize(self.device)
            if barrier and self.world > 1 and not self.loopback:
                # a peer's last kernels may still read our gradient slots / write
                # our parameters over NVLink: nobody unmaps before everyone is done
                import torch.distributed as dist
                if dist.is_initialized():
                    dist.barrier(group=self.group)
            _native.lib().deft_comm_destroy(self._h)
            self._h = None
            for p in self._opened:
                _native.lib().deft_mem_close(p)
            self._opened = []

    def __del__(self):
        try:
            self.close(barrier=False)
        except Exception:
            pass


__all__ = ["BucketComm", "region_tensor", "CHANNEL_SM", "CHANNEL_CE"]
