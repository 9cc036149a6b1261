"""Debug: run a small loopback world with every comm launch logged per rank.
python tools/loopback_trace.py W placement graphs(0|1) [iters] [dtype]"""
import os
import sys
from pathlib import Path

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

from paper_2503_16815_b200 import comm as C  # noqa: E402
from paper_2503_16815_b200 import executor as E  # noqa: E402

LOG = []


def wrap(name):
    orig = getattr(C.BucketComm, name)

    def f(self, *a, **k):
        short = [x if not isinstance(x, (list, tuple)) or len(x) < 6 else f"<{len(x)}>"
                 for x in a if not isinstance(x, torch.Tensor)]
        short = [s if not hasattr(s, "cuda_stream") else f"s{s.cuda_stream % 100000}"
                 for s in short]
        LOG.append((self.rank, name, short))
        print("R", self.rank, name, short, flush=True)
        return orig(self, *a, **k)
    setattr(C.BucketComm, name, f)


for n in ("reduce_scatter", "reduce_scatter_multi", "update_multi", "gather", "update"):
    wrap(n)

orig_step = E.DeftDataParallel.train_step


def step(self, *a, **k):
    print("STEP rank", self.rank, "it", self.iteration, flush=True)
    return orig_step(self, *a, **k)


E.DeftDataParallel.train_step = step
orig_ready = E.DeftDataParallel._buckets_ready


def ready(self, bidxs):
    print("READY rank", self.rank, bidxs, "current stream",
          torch.cuda.current_stream(self.device).cuda_stream % 100000, flush=True)
    return orig_ready(self, bidxs)


E.DeftDataParallel._buckets_ready = ready
orig_sync = torch.cuda.Stream.synchronize


def ssync(self):
    print("STREAM SYNC", self.cuda_stream % 100000, flush=True)
    return orig_sync(self)


torch.cuda.Stream.synchronize = ssync
import smoke_executor as S  # noqa: E402

W = int(sys.argv[1])
placement = sys.argv[2]
graphs = bool(int(sys.argv[3]))
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 6
dtype = torch.bfloat16 if len(sys.argv) > 5 and sys.argv[5] == "bf16" else torch.float32
import paper_2503_16815_b200.loopback as L  # noqa: E402
orig_init = L.LoopbackWorld.__init__


def init(self, *a, **k):
    k["spin_timeout_ms"] = 8000
    orig_init(self, *a, **k)
    for r in self.ranks:
        print("rank", r.rank, "compute", r.compute_stream.cuda_stream % 100000,
              "comm", r.comm_stream.cuda_stream % 100000, flush=True)


L.LoopbackWorld.__init__ = init
res = S.run_loopback(W, iters, placement=placement, cuda_graphs=graphs, dtype=dtype)
want_m, want_p = S.oracle_theta(res[2], res[3][0], W, iters, dtype=dtype)
print("ERR", S.check_ranks(res[0], res[1], want_m, want_p, W, dtype, res[4]))
