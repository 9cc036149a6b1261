"""Where does a ResNet-101 bs64 training step spend its time on one B200?
eager fwd+bwd (host vs device time), CUDA-graphed fwd+bwd, DeFT step."""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main(model_name="resnet101", steps=20):
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda", 0)
    model = bench.build_model(model_name, dev)
    batch = bench.make_batch(model_name, 64, dev)
    loss_fn = bench.loss_fn_for(model_name)

    def plain():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_fn(model, batch)
        loss.backward()
        return loss

    for _ in range(5):
        plain()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    a.record()
    for _ in range(steps):
        plain()
    b.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"eager fwd+bwd: device {a.elapsed_time(b)/steps:.3f} ms/step, "
          f"host {(h1-h0)*1e3/steps:.3f} ms/step")

    # CUDA graph of fwd+bwd (grads accumulate into static .grad)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            plain()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plain()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"graphed fwd+bwd: device {a.elapsed_time(b)/steps:.3f} ms/step")

    # forward only / backward only split
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps):
        with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
            loss_fn(model, batch)
    b.record()
    torch.cuda.synchronize()
    print(f"eager fwd (no_grad): {a.elapsed_time(b)/steps:.3f} ms/step")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["resnet101"]))
