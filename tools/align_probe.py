"""Does the alignment of parameter views inside one flat buffer change the
model's compute time?  fwd+bwd, CUDA-graphed, ResNet-101 bs64 (1 GPU):
  native   -- parameters as allocated by torch
  packed   -- views into one flat buffer, packed back to back (DeFT round 1)
  aligned  -- views into one flat buffer, every parameter at a 256-byte boundary
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def rebind(model, align_elems):
    ps = [p for p in model.parameters()][::-1]
    offs, o = [], 0
    for p in ps:
        o = -(-o // align_elems) * align_elems
        offs.append(o)
        o += p.numel()
    flat = torch.zeros(o + 64, device="cuda")
    for p, off in zip(ps, offs):
        v = torch.as_strided(flat, p.shape, p.stride(), off)
        v.copy_(p.data)
        p.data = v
    return flat


def timed(model, batch, loss_fn, steps=30):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())

    def step():
        for p in model.parameters():
            p.grad = None
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_fn(model, batch)
        loss.backward()
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    torch.backends.cudnn.benchmark = True
    name = sys.argv[1] if len(sys.argv) > 1 else "resnet101"
    batch = bench.make_batch(name, 64 if name != "gpt2" else 16, "cuda")
    loss_fn = bench.loss_fn_for(name)
    for rep in range(2):
        for mode in ("native", "packed", "aligned"):
            m = bench.build_model(name, "cuda")
            if mode != "native":
                keep = rebind(m, 1 if mode == "packed" else 64)
            print(name, rep, mode, round(timed(m, batch, loss_fn), 3), "ms", flush=True)
            del m
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
