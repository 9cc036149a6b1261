"""ctypes binding of libdeft_b200.so (include/deft_b200.h).

The library is the product path: if it is missing, or there is no CUDA
device, every call raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import DeftError, DeviceError, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libdeft_b200.so"

# every symbol include/deft_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTED = (
    "deft_abi_version", "deft_last_error", "deft_launch_count",
    "deft_subset_sum_workspace_bytes", "deft_subset_sum_batched",
    "deft_solver_create", "deft_solver_destroy", "deft_solver_solve",
    "deft_solver_last_kernel_ms", "deft_solver_schedule", "deft_solver_schedule_chunk",
    "deft_sched_carry_bytes",
    "deft_mem_alloc", "deft_mem_free", "deft_mem_open", "deft_mem_close",
    "deft_comm_flag_bytes", "deft_comm_create", "deft_comm_destroy",
    "deft_comm_set_update_blocks", "deft_comm_configure", "deft_comm_set_phase_trace",
    "deft_bucket_reduce_scatter", "deft_bucket_reduce_scatter_multi", "deft_bucket_update",
    "deft_bucket_update_multi",
    "deft_sgd_momentum_update", "deft_sgd_momentum_update_multi", "deft_gather_segments",
    "deft_stream_create", "deft_stream_destroy", "deft_stream_alias_probe",
    "deft_loopback_reduce_scatter", "deft_loopback_update", "deft_bucket_sync_update_multi",
)

DTYPE_F32, DTYPE_BF16 = 0, 1
CHANNEL_SM, CHANNEL_CE = 0, 1
IPC_HANDLE_BYTES = 64

_lib = None
_lib_lock = threading.Lock()

c_i32, c_i64, c_u64, c_f32, c_sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                    ctypes.c_float, ctypes.c_size_t)
c_vp = ctypes.c_void_p
P = ctypes.POINTER


def _declare(lib):
    sig = {
        "deft_abi_version": (c_i32, []),
        "deft_last_error": (ctypes.c_char_p, []),
        "deft_launch_count": (c_u64, []),
        "deft_subset_sum_workspace_bytes": (c_sz, [c_i32, P(c_i32), P(c_i64)]),
        "deft_subset_sum_batched": (c_i32, [c_vp, c_vp, c_vp, c_i32, P(c_i32), P(c_i64), c_vp,
                                            c_vp, c_vp, c_sz, c_vp]),
        "deft_solver_create": (c_i32, [c_i32, P(c_vp)]),
        "deft_solver_destroy": (c_i32, [c_vp]),
        "deft_solver_solve": (c_i32, [c_vp, c_i32, P(c_i32), P(c_i64), P(c_i64),
                                      P(ctypes.c_uint8), P(c_i64)]),
        "deft_solver_last_kernel_ms": (c_f32, [c_vp]),
        "deft_sched_carry_bytes": (c_sz, []),
        "deft_solver_schedule_chunk": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, c_i32,
                                               P(c_i64), P(c_i64), P(c_i64), P(c_i64), c_vp,
                                               c_vp, P(c_i32), c_i64, P(c_i64), P(c_i32)]),
        "deft_solver_schedule": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, P(c_i64), P(c_i64),
                                         P(c_i64), P(c_i64), P(c_i32), c_i64, P(c_i64),
                                         P(c_i32)]),
        "deft_mem_alloc": (c_i32, [c_sz, P(c_vp), P(ctypes.c_uint8)]),
        "deft_mem_free": (c_i32, [c_vp]),
        "deft_mem_open": (c_i32, [P(ctypes.c_uint8), P(c_vp)]),
        "deft_mem_close": (c_i32, [c_vp]),
        "deft_comm_flag_bytes": (c_sz, [c_i32]),
        "deft_comm_create": (c_i32, [c_i32, c_i32, P(c_vp), P(c_vp), P(c_vp), c_vp, c_i64,
                                     c_i32, c_i32, P(c_vp)]),
        "deft_comm_destroy": (c_i32, [c_vp]),
        "deft_comm_set_update_blocks": (c_i32, [c_vp, c_i32]),
        "deft_comm_configure": (c_i32, [c_vp, c_i32, c_i64]),
        "deft_comm_set_phase_trace": (c_i32, [c_vp, c_vp]),
        "deft_bucket_sync_update_multi": (c_i32, [c_vp, c_i32, c_i32, P(c_i64), P(c_i64),
                                                  c_f32, c_f32, c_f32, c_vp, c_vp]),
        "deft_stream_create": (c_i32, [c_i32, P(c_vp)]),
        "deft_loopback_reduce_scatter": (c_i32, [P(c_vp), c_i32, c_i32, c_i32, c_i32,
                                                 P(c_i64), P(c_i64), c_vp]),
        "deft_loopback_update": (c_i32, [P(c_vp), c_i32, c_i32, c_i32, P(c_i64), P(c_i64),
                                         c_f32, c_f32, c_f32, P(c_vp), c_vp]),
        "deft_stream_destroy": (c_i32, [c_vp]),
        "deft_stream_alias_probe": (c_i32, [c_vp, c_vp, c_i32, c_i32, P(c_i32)]),
        "deft_bucket_reduce_scatter": (c_i32, [c_vp, c_i32, c_i32, c_i64, c_i64, c_vp]),
        "deft_bucket_reduce_scatter_multi": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp,
                                                     c_vp]),
        "deft_bucket_update": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_f32, c_f32, c_f32, c_vp,
                                       c_vp]),
        "deft_bucket_update_multi": (c_i32, [c_vp, c_i32, c_i32, P(c_i64), P(c_i64), c_f32,
                                             c_f32, c_f32, c_vp, c_vp]),
        "deft_sgd_momentum_update": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i64, c_f32,
                                             c_f32, c_f32, c_vp]),
        "deft_gather_segments": (c_i32, [c_vp, P(c_vp), P(c_i64), P(c_i64), c_i32, c_i64,
                                         c_vp]),
        "deft_sgd_momentum_update_multi": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i32,
                                                   P(c_i64), P(c_i64), P(c_f32), c_f32, c_f32,
                                                   c_vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """Load libdeft_b200.so (no GPU needed just to load it)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise DeftError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (make -C paper_2503_16815_b200/csrc)")
            _lib = _declare(ctypes.CDLL(str(LIB_PATH)))
        return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        raise_for_status(status, what, lib().deft_last_error().decode(errors="replace"))


def launch_count() -> int:
    return int(lib().deft_launch_count())


def _require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("the DeFT B200 path needs a CUDA device; no CPU fallback exists")
    return torch


class SubsetSumSolver:
    """Owns a deft_solver (high-priority stream, pinned staging) on one device."""

    def __init__(self, device: int | None = None):
        torch = _require_cuda()
        self.device = torch.cuda.current_device() if device is None else device
        h = c_vp()
        check(lib().deft_solver_create(self.device, ctypes.byref(h)), "deft_solver_create")
        self._h = h
        self.calls = 0
        self.problems = 0
        self.kernel_ms = 0.0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.deft_solver_destroy(h)

    def solve(self, problems) -> list[list[bool]]:
        """problems: [(weights in ascending-id order, capacity >= 1)]."""
        b = len(problems)
        if b == 0:
            return []
        n = np.fromiter((len(w) for w, _ in problems), dtype=np.int32, count=b)
        caps = np.fromiter((c for _, c in problems), dtype=np.int64, count=b)
        ws = np.fromiter((x for w, _ in problems for x in w), dtype=np.int64, count=int(n.sum()))
        take = np.empty(int(n.sum()), dtype=np.uint8)
        best = np.empty(b, dtype=np.int64)
        st = lib().deft_solver_solve(
            self._h, b, n.ctypes.data_as(P(c_i32)), ws.ctypes.data_as(P(c_i64)),
            caps.ctypes.data_as(P(c_i64)), take.ctypes.data_as(P(ctypes.c_uint8)),
            best.ctypes.data_as(P(c_i64)))
        check(st, "deft_solver_solve")
        self.calls += 1
        self.problems += b
        self.kernel_ms += float(lib().deft_solver_last_kernel_ms(self._h))
        out, pos = [], 0
        tl = take.astype(bool).tolist()
        for k in n.tolist():
            out.append(tl[pos:pos + k])
            pos += k
        self.last_best = best
        return out


_solvers: dict[int, SubsetSumSolver] = {}


def subset_sum_solver() -> SubsetSumSolver:
    torch = _require_cuda()
    dev = torch.cuda.current_device()
    s = _solvers.get(dev)
    if s is None:
        s = _solvers[dev] = SubsetSumSolver(dev)
    return s
