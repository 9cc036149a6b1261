"""Measure how CUDA streams map onto hardware work queues (deft_stream_alias_probe).

python tools/stream_queues.py [n_raw] [n_pool]
Prints the queue class of each of n_raw streams created with deft_stream_create
and of n_pool torch pool streams (classes = sets of mutually aliasing streams).
Run with and without CUDA_DEVICE_MAX_CONNECTIONS=32 to see its effect.
"""
import ctypes
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2503_16815_b200 import _native  # noqa: E402


def classify(ptrs, timeout_us=20000, mode=0):
    lib = _native.lib()
    reps, cls = [], []
    for p in ptrs:
        c = None
        for k, rep in enumerate(reps):
            a = ctypes.c_int32()
            _native.check(lib.deft_stream_alias_probe(ctypes.c_void_p(rep), ctypes.c_void_p(p),
                                                      timeout_us, mode, ctypes.byref(a)), "probe")
            if a.value:
                c = k
                break
        if c is None:
            reps.append(p)
            c = len(reps) - 1
        cls.append(c)
    return cls


def main():
    n_raw = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    n_pool = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    torch.cuda.init()
    lib = _native.lib()
    raw = []
    for _ in range(n_raw):
        h = ctypes.c_void_p()
        _native.check(lib.deft_stream_create(0, ctypes.byref(h)), "create")
        raw.append(h.value)
    t0 = time.time()
    mode = int(os.environ.get("PROBE_MODE", "0"))
    c_raw = classify(raw, mode=mode)
    pool = [torch.cuda.Stream().cuda_stream for _ in range(n_pool)]
    c_pool = classify(pool, mode=mode)
    # symmetry check of one aliasing pair, if any
    out = {"CUDA_DEVICE_MAX_CONNECTIONS": os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"),
           "mode": mode,
           "raw_classes": c_raw, "n_raw_classes": len(set(c_raw)),
           "pool_classes": c_pool, "n_pool_classes": len(set(c_pool)),
           "probe_s": round(time.time() - t0, 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
