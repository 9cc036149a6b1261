"""DeFT delayed-update data-parallel training step on B200s.

python bench.py [--gpus N --steps K --warmup W --model resnet101|vgg19|gpt2]
    [--impl deft|reference]

A step = one DeFT-scheduled training iteration (forward, backward, bucket
reduce-scatter on the schedule's NVLink channels, fused delayed SGD/momentum
update + parameter all-gather) of the named model on synthetic data,
batch 64 per GPU (BASELINE.json configs[1]: ResNet-101, 224x224).
Under torchrun (N > 1) every rank runs one GPU; rank 0 prints ONE JSON line.

--impl reference runs the CPU path (the oracle port of the reference's
scheduler plus the delayed-SGD oracle, oracle/), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# rank 0 prints exactly ONE JSON line on stdout: keep NCCL's version banner off it
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"

BATCH = 64
METRIC = "samples/sec (DeFT delayed-update DP training step)"
# The convergence walk the update-frequency controller is driven by: the values the
# reference ships for its merged-update experiments (pkg/fixtures/
# walk_merged_updates.json = experiment_vgg.json:18-25).  --walk FILE overrides.
DEFAULT_WALK = {"s0": 0.2103, "s_star": 0.0, "eta": 0.01, "mu_t": 0.851934758267416,
                "sigma_t": 181.21080499210186, "epsilon": 0.01}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--model", default="resnet101", choices=["resnet101", "vgg19", "gpt2"])
    ap.add_argument("--impl", default="deft", choices=["deft", "reference", "ddp"],
                    help="deft (this repo), reference (CPU oracle port), ddp (PyTorch DDP + "
                         "NCCL WFBP baseline)")
    ap.add_argument("--batch", type=int, default=None,
                    help="per-GPU batch (default 64; GPT-2: 16 sequences of 1024)")
    ap.add_argument("--update-placement", default="auto",
                    choices=["auto", "bucket", "end", "start"])
    ap.add_argument("--update-blocks", type=int, default=0,
                    help="CTA budget of the update kernels (0 = default)")
    ap.add_argument("--scheme", default="deft", choices=["deft", "wfbp", "priority"],
                    help="schedule run on the executor: DeFT, or one of the reference's "
                         "synchronous baselines (scheduler.py:386-418) on the same kernels")
    ap.add_argument("--start-grouping", default="auto", choices=["auto", "size", "timed"],
                    help="how start-placement updates are grouped into launches")
    ap.add_argument("--eager", action="store_true", help="no CUDA graphs")
    ap.add_argument("--walk", default=None,
                    help="JSON file of the convergence walk (preserver.WalkParams fields); "
                         "default: the reference's walk_merged_updates values")
    ap.add_argument("--oneshot-mb", type=float, default=None,
                    help="buckets of at most this many MB of gradients sync one-shot "
                         "(DeftConfig.oneshot_max_bytes; default: the executor's)")
    ap.add_argument("--defer", default="last", choices=["last", "predicted", "none"],
                    help="graph mode: which fresh transfers start with the next iteration "
                         "(DeftConfig.defer_tail)")
    ap.add_argument("--bucket-mb", type=float, default=None,
                    help="partition size in MB of fp32 (default: the reference's 6.5M params)")
    ap.add_argument("--links", default="both", choices=["both", "sm", "ce"],
                    help="NVLink channels the schedule may use (both = measured SM + CE)")
    ap.add_argument("--dump-profile", default=None,
                    help="write the B200-measured ModelProfile + ClusterSpec JSON here")
    ap.add_argument("--comm-scale", type=float, default=1.0,
                    help="scale the measured comm times before planning (slower-link / "
                         "update-frequency sweep: >1 makes DeFT merge iterations)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--solver-full", action="store_true",
                    help="solver block: also time the reference's GPT-2 / VGG-19 feedback "
                         "loops (about 50 s of single-core Python)")
    ap.add_argument("--ddp-graphs", action="store_true",
                    help="--impl ddp: capture the DDP step (static_graph=True) in a CUDA graph")
    ap.add_argument("--h2d-chunks", type=int, default=32,
                    help="e2e: split each step's host->device input copy into this many "
                         "batch slices")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


# ----------------------------------------------------------------- workloads

def build_model(name, device):
    import torch
    import torchvision
    torch.manual_seed(0)
    if name == "resnet101":
        m = torchvision.models.resnet101()
    elif name == "vgg19":
        m = torchvision.models.vgg19()
    else:
        from transformers import GPT2Config, GPT2LMHeadModel
        m = GPT2LMHeadModel(GPT2Config(n_positions=1024))
        m.config.use_cache = False
    m = m.to(device)
    if name == "gpt2" and device != "cpu":
        m = m.to(torch.bfloat16)  # BASELINE configs[3]: bf16 gradient buckets
    if name != "gpt2":
        m = m.to(memory_format=torch.channels_last)
    return m


def make_batch(name, batch, device, seed=1234):
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    if name == "gpt2":
        x = torch.randint(0, 50257, (batch, 1024), generator=g)
        return (x.to(device), x.to(device))
    x = torch.randn(batch, 3, 224, 224, generator=g)
    y = torch.randint(0, 1000, (batch,), generator=g)
    if device != "cpu":
        x = x.to(device).contiguous(memory_format=torch.channels_last)
        y = y.to(device)
    return (x, y)


def loss_fn_for(name):
    import torch.nn.functional as F

    if name == "gpt2":
        def loss_fn(module, batch):
            out = module(batch[0], labels=batch[1])
            return out.loss
    else:
        def loss_fn(module, batch):
            return F.cross_entropy(module(batch[0]), batch[1])
    return loss_fn


# ----------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period_ms=50):
        self.index = index
        self.period_ms = period_ms
        self.rows = []
        self.proc = None
        self.window = None
        self.load = [time.monotonic(), None]

    def mark(self, start: bool):
        """Open / close the timed region; summary() reports the samples inside."""
        if start:
            self.window = [time.monotonic(), None]
        else:
            self.window[1] = time.monotonic()

    def end_load(self):
        """Close the load window (opened by __enter__, before the warm-up): the
        throttle reasons are taken over all of it, so they cover >= 1 s of load
        even when the timed region itself is shorter."""
        self.load[1] = time.monotonic()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([time.monotonic()] + [x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        rows = [r[1:] for r in self.rows]
        win = None
        if self.window and self.window[1] is not None:
            win = [r[1:] for r in self.rows if self.window[0] <= r[0] <= self.window[1]]
        lo, hi = self.load[0], self.load[1] or time.monotonic()
        load = [r[1:] for r in self.rows if lo <= r[0] <= hi]
        use = win if win else rows
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def med(rs):
            sm = sorted(float(r[0]) for r in rs if r[0].replace(".", "").isdigit())
            return sm[len(sm) // 2] if sm else None
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # reasons: the timed region AND the whole load window around it
        reasons = sorted({n for r in use + load for n, v in zip(names, r[2:6])
                          if v == "Active"})
        return {"sm_mhz": med(use), "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(use),
                "samples_all": len(rows), "period_ms": self.period_ms,
                "window": "timed region" if win else "whole run (no sample in the timed region)",
                "window_s": round(self.window[1] - self.window[0], 3) if win else None,
                "load_window": "warm-up start to end of the last timed region",
                "load_window_s": round(hi - lo, 3), "load_samples": len(load),
                "load_sm_mhz": med(load),
                "load_sm_min_mhz": min((float(r[0]) for r in load
                                        if r[0].replace(".", "").isdigit()), default=None)}


def pad_load(clk, step_fn, ms_per_step, world, dist, device, min_s=1.0):
    """Untimed extra steps so the clock sampler's load window spans >= min_s;
    the same count on every rank (the steps contain collectives)."""
    import math

    import torch
    need = max(0.0, min_s - (time.monotonic() - clk.load[0]))
    n = min(5000, int(math.ceil(need * 1e3 / max(ms_per_step, 1e-3))))
    if world > 1:
        t = torch.tensor([n], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        n = int(t.item())
    for _ in range(n):
        step_fn()
    torch.cuda.synchronize()


# ----------------------------------------------------------------- CPU path

def reference_schedule(n_iter):
    """The DeFT decision stream of the reference's ResNet-101 fixture on its
    dual-link cluster (6.5M partition, mu 1.65) from the UNMODIFIED reference
    (deftsim, oracle/_ref -- copied there by build()), as dicts; the oracle port
    when the copy is absent.  Returns (decisions, seconds, kind)."""
    from oracle import reference
    inputs = json.loads((ROOT / "tests" / "golden" / "inputs.json").read_text())
    prof_d, cl_d = inputs["profiles"]["resnet101"], inputs["clusters"]["dual"]
    t0 = time.perf_counter()
    if reference.available():
        R = reference.deftsim()
        sched = R.deft_schedule(R.profile_from_dict(prof_d), R.cluster_from_dict(cl_d),
                                R.PartitionConfig(partition_size=6_500_000, mu=1.65), n_iter)
        dec = [d.to_dict() for d in sched.decisions]
        kind = "reference"
    else:
        from oracle import deft_oracle as O
        part = O.partition(prof_d["buckets"], sum(b["forward_us"] for b in prof_d["buckets"]),
                           6_500_000, 1.65)
        dec = O.schedule(part, [l["speed_ratio_to_fast"] for l in cl_d["links"]],
                         [l["name"] for l in cl_d["links"]], n_iter)
        kind = "port"
    return dec, time.perf_counter() - t0, kind


def cpu_reference_run(model_name, steps, warmup, batch):
    """The reference's CPU path on this host: the DeFT schedule from the
    reference itself (deftsim, reference_schedule), CPU fwd/bwd of the named
    model, and the delayed SGD/momentum the schedule's update events call for
    (oracle/delayed_sgd.py rules -- the reference defines no update arithmetic
    and no training loop).  Bounded sample: `batch` samples per step."""
    import torch

    torch.set_num_threads(os.cpu_count() or 1)
    model = build_model(model_name, "cpu")
    params = [p for p in model.parameters() if p.requires_grad][::-1]
    loss_fn = loss_fn_for(model_name)
    data = make_batch(model_name, batch, "cpu")
    total = sum(p.numel() for p in params)
    v = torch.zeros(total)
    summed = {}
    n = warmup + steps
    decisions, t_sched, kind = reference_schedule(n + 2)
    events = {d["iteration"]: d["update_events"] for d in decisions if d["stage"] == "backward"}
    t0 = None
    for s in range(n):
        if s == warmup:
            t0 = time.perf_counter()
        flat = torch.cat([p.detach().reshape(-1) for p in params])
        for u in events.get(s - 2, ()):
            g = sum(summed.pop(o) for o in u["origins"]) / u["merge_count"]
            v.mul_(0.9).add_(g)
            flat.add_(v, alpha=-0.1)
        off = 0
        with torch.no_grad():
            for p in params:
                p.copy_(flat[off:off + p.numel()].view_as(p))
                off += p.numel()
        for p in params:
            p.grad = None
        loss = loss_fn(model, data)
        loss.backward()
        summed[s] = torch.cat([p.grad.reshape(-1) for p in params])
    dt = time.perf_counter() - t0
    src = ("the reference itself (deftsim from oracle/_ref)" if kind == "reference"
           else "the oracle port (oracle/_ref absent)")
    return {"value": steps * batch / dt, "unit": "samples/s", "cores": torch.get_num_threads(),
            "kind": kind,
            "sample": f"{model_name} fp32 CPU fwd+bwd, batch {batch} x {steps} timed steps "
                      f"(+{warmup} warm-up); DeFT schedule (ResNet-101 fixture, dual link, "
                      f"6.5M partition) by {src}: {t_sched * 1e3:.0f} ms for {n + 2} "
                      "iterations; delayed SGD/momentum per its update events"}


# ----------------------------------------------------------------- GPU path

def solver_measurement(full: bool = False):
    """The scheduling side of the path, timed on THIS host in the same run: the
    reference itself (deftsim from oracle/_ref, single-threaded Python: 1 core)
    against this package (K5 persistent GPU state machine), on the SURVEY §6.3
    workloads -- feedback_loop (200 iterations, up to 10 capacity retries) on the
    ResNet-101 fixture at quarter bandwidth (and VGG-19 / GPT-2 with ``full``),
    and deft_schedule (200 iterations) of the three fixtures -- with the decision
    streams compared byte for byte."""
    import gc

    import paper_2503_16815_b200 as D
    from paper_2503_16815_b200 import gpu_scheduler
    from oracle import reference
    # this runs after the training measurement: move the large training heap out
    # of the cyclic GC's reach, so a collection triggered inside either timed
    # region (both arms allocate thousands of decision objects) does not walk it
    # -- measured: one VGG-19 deft_schedule read 96 ms in-process vs 10-13 ms alone
    gc.collect()
    gc.freeze()
    inputs = json.loads((ROOT / "tests" / "golden" / "inputs.json").read_text())
    walk_d, cl_d = inputs["walk"], inputs["clusters"]["dual"]
    R = reference.deftsim() if reference.available() else None
    cfg = D.PartitionConfig(6_500_000, mu=1.65)
    warm = D.partition_buckets(D.profile_from_dict(inputs["profiles"]["resnet101"]), cfg)
    gpu_scheduler.run_schedules_lazy(warm, D.cluster_from_dict(cl_d), [1.0], 4)   # warm
    out = {"reference": "deftsim (oracle/_ref, unmodified)" if R else "absent",
           "reference_cores": 1, "host_nproc": os.cpu_count(), "runs": []}

    def text(decisions):
        return "".join(json.dumps(d.to_dict(), sort_keys=True) + "\n" for d in decisions)

    loops = [("resnet101", 4.0)] + ([("gpt2", 4.0), ("vgg19", 4.0)] if full else [])
    for name, scale in loops:
        prof = D.profile_from_dict(inputs["profiles"][name]).scaled_comm(scale)
        t0 = time.perf_counter()
        sched, verdict = D.feedback_loop(prof, D.cluster_from_dict(cl_d), cfg,
                                         D.WalkParams.from_dict(walk_d), iterations=200)
        t_gpu = time.perf_counter() - t0
        run = {"workload": f"feedback_loop {name} bw x{1 / scale:g}, dual link, 200 iterations",
               "retries": verdict.retries, "gpu_s": round(t_gpu, 4)}
        if R:
            rp = R.profile_from_dict(inputs["profiles"][name]).scaled_comm(scale)
            t0 = time.perf_counter()
            rs, rv = R.feedback_loop(rp, R.cluster_from_dict(cl_d),
                                     R.PartitionConfig(6_500_000, mu=1.65),
                                     R.WalkParams.from_dict(walk_d), iterations=200)
            run["reference_cpu_s"] = round(time.perf_counter() - t0, 3)
            run["speedup"] = round(run["reference_cpu_s"] / t_gpu, 1)
            run["identical"] = (text(rs.decisions) == text(sched.decisions)
                                and rv.retries == verdict.retries)
        out["runs"].append(run)
    for name in ("resnet101", "vgg19", "gpt2"):
        prof = D.profile_from_dict(inputs["profiles"][name])
        t0 = time.perf_counter()
        sched = D.deft_schedule(prof, D.cluster_from_dict(cl_d), cfg, 200)
        t_gpu = time.perf_counter() - t0
        run = {"workload": f"deft_schedule {name}, dual link, 6.5M partition, 200 iterations",
               "gpu_s": round(t_gpu, 4)}
        if R:
            t0 = time.perf_counter()
            rs = R.deft_schedule(R.profile_from_dict(inputs["profiles"][name]),
                                 R.cluster_from_dict(cl_d),
                                 R.PartitionConfig(6_500_000, mu=1.65), 200)
            run["reference_cpu_s"] = round(time.perf_counter() - t0, 3)
            run["speedup"] = round(run["reference_cpu_s"] / t_gpu, 1)
            run["identical"] = text(rs.decisions) == text(sched.decisions)
        out["runs"].append(run)
    return out


def compute_only_step_ms(model, batch, loss_fn, steps, warmup, world, dist, device):
    """The compute roofline of SURVEY 8d: one GPU's fwd + bwd + fused SGD/momentum
    step with NO communication -- the faster of eager and CUDA-graphed execution
    (models differ: ResNet-101 gains from graphs, GPT-2 loses)."""
    import torch
    params = [p for p in model.parameters() if p.requires_grad]
    opt = torch.optim.SGD(params, lr=0.1, momentum=0.9, fused=True)
    s = torch.cuda.Stream(device)

    def step():
        opt.zero_grad(set_to_none=True)
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False,
                            enabled=next(model.parameters()).dtype == torch.float32):
            loss = loss_fn(model, batch)
        loss.backward()
        opt.step()
        return loss.detach()

    def timed(fn):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        if world > 1:
            t = torch.tensor([ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    s.synchronize()
    ms_eager = timed(step)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    ms_graph = timed(g.replay)
    del g, opt
    for p in params:
        p.grad = None
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return min(ms_eager, ms_graph), {"eager_ms": round(ms_eager, 3),
                                     "graph_ms": round(ms_graph, 3)}


def isolated_kernels(ddp, world, dist, device, reps=10):
    """Dominant native kernels timed alone (barrier-aligned across ranks, CUDA
    events on their own stream), over this model's real bucket layout."""
    import torch
    from paper_2503_16815_b200 import _native
    s = torch.cuda.Stream(device)
    out = {}
    esz = 4
    slot = 0

    def max_over_ranks(ms):
        if world > 1:
            t = torch.tensor([ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=device)   # 2x the L2

    def run(kind, fn, nbytes):
        """Every pass timed alone with CUDA events, the L2 flushed before it (cold,
        like ncu's default cache control: a back-to-back pass would find the tail
        of the previous one's writes in the 126 MB L2); then the same passes
        captured in ONE CUDA graph and replayed back to back -- the way the
        training step issues them (reported beside, warm L2)."""
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        with torch.cuda.stream(s):
            for a, b in evs:
                flush.zero_()
                a.record(s)
                fn()
                b.record(s)
        torch.cuda.synchronize()
        ms_eager = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / reps)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms_graph = None
        g = torch.cuda.CUDAGraph()
        ok = 1
        try:
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn()
        except Exception:   # reported as eager-only
            ok = 0
            torch.cuda.synchronize()
        if world > 1:       # replay only if every rank captured (barriers inside)
            t = torch.tensor([ok], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok = int(t.item())
        if ok:
            with torch.cuda.stream(s):
                g.replay()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a.record(s)
            with torch.cuda.stream(s):
                g.replay()
            b.record(s)
            torch.cuda.synchronize()
            ms_graph = max_over_ranks(a.elapsed_time(b) / reps)
        del g
        ms = ms_eager
        n = len(ddp.buckets)
        if kind == "update" and ddp.placement == "end":
            n = 1
        elif kind == "update" and ddp.placement == "start":
            n = len(ddp._start_groups())
        out[kind] = {"launches": n, "ms_per_pass": round(ms, 4),
                     "avg_launch_us": round(ms / n * 1e3, 2), "bytes_per_pass": nbytes,
                     "achieved_gbs": round(nbytes / (ms / 1e3) / 1e9, 1),
                     "timing": "each pass alone after an L2 flush, host-issued launches",
                     "graph_ms_per_pass": round(ms_graph, 4) if ms_graph else None,
                     "graph_achieved_gbs": round(nbytes / (ms_graph / 1e3) / 1e9, 1)
                     if ms_graph else None,
                     "graph_timing": "the passes replayed back to back as one CUDA graph "
                                     "(warm L2), as the step issues them"}

    saved_p = ddp.comm.params.clone()
    saved_m = ddp.mom.clone()
    if ddp.cfg.grad_dtype == torch.bfloat16:
        esz = 2
    if world == 1:      # HBM bytes: read g, v, p (master); write v, p (+ bf16 copy)
        upd_bytes = sum((b.hi - b.lo) * 20 for b in ddp.buckets)
    else:               # NVLink bytes: updated params stored to the W-1 peers
        upd_bytes = sum((b.hi - b.lo) * esz * (world - 1) // world for b in ddp.buckets)

    def updates():   # the step's own launch shape
        if ddp.placement == "end":
            ddp.comm.update_multi(slot, [(b.lo, b.hi) for b in ddp.buckets], 1.0, 0.0, 0.9,
                                  ddp.mom, s)
        elif ddp.placement == "start":   # first group on the full grid, as in the step
            for gi, g in enumerate(ddp._start_groups()):
                ddp.comm.set_update_blocks(0 if gi == 0 else ddp._update_blocks)
                ddp.comm.update_multi(slot, [(ddp.buckets[b].lo, ddp.buckets[b].hi) for b in g],
                                      1.0, 0.0, 0.9, ddp.mom, s)
            ddp.comm.set_update_blocks(ddp._update_blocks)
        else:                             # "bucket": one launch per bucket
            for b in ddp.buckets:
                ddp.comm.update_multi(slot, [(b.lo, b.hi)], 1.0, 0.0, 0.9, ddp.mom, s)
    with torch.cuda.stream(s):
        run("update", updates, upd_bytes)
        if world > 1:
            rs_bytes = sum((b.hi - b.lo) * esz * (world - 1) // world for b in ddp.buckets)

            def rss():
                for b in ddp.buckets:
                    ddp.comm.reduce_scatter(_native.CHANNEL_SM, slot, b.lo, b.hi - b.lo, s)
            run("reduce_scatter", rss, rs_bytes)
    torch.cuda.synchronize()
    ddp.comm.params.copy_(saved_p)
    ddp.mom.copy_(saved_m)
    torch.cuda.synchronize()
    return out


def ncu_traffic(kernel, model, world):
    """DRAM bytes per launch of `kernel` for this model / world size from a committed
    ncu --set full capture (profiles/ncu_traffic.json), or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get(f"{kernel}:{model}:w{world}")


def _native_channel(name):
    from paper_2503_16815_b200 import _native
    return _native.CHANNEL_SM if name == "sm" else _native.CHANNEL_CE


def init_quiet(dist, device):
    """NCCL prints its version banner on fd 1 when the communicator comes up;
    rank 0's stdout must carry exactly one JSON line, so point fd 1 at stderr
    while the process group (eagerly, device_id given) initialises."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        dist.init_process_group("nccl", device_id=device)
        dist.barrier()
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def ddp_baseline(args, world, rank, device, dist):
    """NCCL WFBP baseline: torch DistributedDataParallel (bucketed all-reduce
    overlapped with backward, every iteration) + fused SGD/momentum; eager, or
    with ``--ddp-graphs`` the whole step (static_graph=True) captured in one CUDA
    graph and replayed -- the same launch-overhead treatment DeFT's executor gets."""
    import torch
    model = build_model(args.model, device)
    loss_fn = loss_fn_for(args.model)
    batch = make_batch(args.model, args.batch, device, seed=1234 + rank)
    bucket_mb = args.bucket_mb or 25
    # graphed arm: DDP is built, warmed up and captured on ONE side stream (its
    # reducer keeps the AccumulateGrad nodes of the first iterations alive, and a
    # node created on another stream breaks the capture)
    s = torch.cuda.Stream(device) if args.ddp_graphs else torch.cuda.current_stream(device)
    s.wait_stream(torch.cuda.current_stream(device))
    net = model
    with torch.cuda.stream(s):
        if world > 1:
            net = torch.nn.parallel.DistributedDataParallel(
                model, device_ids=[device.index], bucket_cap_mb=bucket_mb,
                gradient_as_bucket_view=True, static_graph=args.ddp_graphs)
        opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9, fused=True)
    amp = next(model.parameters()).dtype == torch.float32

    def step():
        opt.zero_grad(set_to_none=False)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=amp,
                            cache_enabled=not args.ddp_graphs):
            loss = loss_fn(net, batch)
        loss.backward()
        opt.step()
        return loss

    clk = ClockSampler(device.index).__enter__()
    mode = "eager"
    run = step
    if args.ddp_graphs:
        with torch.cuda.stream(s):
            for _ in range(max(11, args.warmup)):   # DDP settles its buckets first
                loss = step()
        del loss
        torch.cuda.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                step()
            run, mode = g.replay, "cuda_graph"
        except Exception as e:   # reported, the eager step is timed instead
            mode = f"eager (capture failed: {type(e).__name__}: {str(e)[:120]})"
            torch.cuda.synchronize()
    for _ in range(args.warmup):
        run()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark(True)
    a.record()
    for _ in range(args.steps):
        run()
    b.record()
    torch.cuda.synchronize()
    clk.mark(False)
    pad_load(clk, run, a.elapsed_time(b) / args.steps, world, dist, device)
    clk.end_load()
    ms = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk.__exit__()
    if rank == 0:
        print(json.dumps({
            "impl": "ddp", "metric": METRIC, "value": round(args.batch * world * args.steps /
                                                          (ms / 1e3), 2),
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "dtype": "bf16",
            "config": {"workload": f"{args.model} torch DDP (NCCL all-reduce WFBP) + fused SGD, "
                                   f"batch {args.batch}/GPU", "bucket_cap_mb": bucket_mb,
                       "mode": mode},
            "clocks": clk.summary()}))
    if args.ddp_graphs:
        # a communicator captured into a CUDA graph hangs in its teardown (measured:
        # the line is printed, then destroy_process_group never returns)
        sys.stdout.flush()
        sys.stderr.flush()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        os._exit(0)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.batch is None:
        args.batch = 16 if args.model == "gpt2" else BATCH
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference_run(args.model, max(1, min(args.steps, 3)), 1, 4)
        line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "samples/s",
                "n_gpus": args.gpus, "steps": max(1, min(args.steps, 3)), "warmup": 1,
                "ms_per_step": 4 / r["value"] * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"{args.model} DeFT delayed-update DP (CPU path)",
                           "global_batch": 4, "note": "bounded CPU sample of configs[1]"},
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if args.impl == "ddp" and args.ddp_graphs:
            # no watchdog event queries against a capturing stream
            os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "0")
        init_quiet(dist, device)
    torch.backends.cudnn.benchmark = True
    if args.impl == "ddp":
        return ddp_baseline(args, world, rank, device, dist)
    import paper_2503_16815_b200 as D

    model = build_model(args.model, device)
    loss_fn = loss_fn_for(args.model)
    batch = make_batch(args.model, args.batch, device, seed=1234 + rank)

    # 1) compute roofline: no communication at all
    ms_compute, compute_modes = compute_only_step_ms(model, batch, loss_fn, args.steps,
                                                     args.warmup, world, dist, device)

    # 2) DeFT: profile on this GPU, plan (partition + feedback loop), run
    walk = D.WalkParams.from_dict(
        json.loads(Path(args.walk).read_text()) if args.walk else DEFAULT_WALK)
    psize = 6_500_000 if args.bucket_mb is None else int(args.bucket_mb * 2**20 / 4)
    cfg = D.DeftConfig(lr=0.1, momentum=0.9, walk=walk,
                       cuda_graphs=False if args.eager else "auto",
                       update_placement=args.update_placement,
                       update_blocks=args.update_blocks, scheme=args.scheme,
                       start_grouping=args.start_grouping,
                       defer_tail=False if args.defer == "none" else args.defer,
                       oneshot_max_bytes=None if args.oneshot_mb is None else
                       int(args.oneshot_mb * 2**20),
                       autocast_dtype=None if args.model == "gpt2" else torch.bfloat16,
                       partition=D.PartitionConfig(partition_size=psize, mu=1.0))
    ddp = D.DeftDataParallel(model, cfg)
    t_setup = time.perf_counter()
    prof = ddp.measure_profile(batch, loss_fn, iters=3, name=args.model, batch_size=args.batch)
    if args.dump_profile and rank == 0:
        Path(args.dump_profile).write_text(json.dumps(
            {"profile": D.profile_to_dict(prof), "cluster": D.cluster_to_dict(ddp.cluster)},
            indent=1, sort_keys=True))
    if args.comm_scale != 1.0:
        prof = prof.scaled_comm(args.comm_scale)
    cluster = ddp.cluster
    if args.links != "both" and world > 1:
        cluster = D.ClusterSpec(links=(D.LinkSpec(f"nvlink_{args.links}", 1.0),))
        ddp.channel_of_link = [_native_channel(args.links)]
        ddp.cluster = cluster
    part = ddp.plan(prof, cluster)
    t_setup = time.perf_counter() - t_setup

    def timed(step_fn, k):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            step_fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    clk = ClockSampler(local).__enter__()      # sampling from before the warm-up on
    warm = ddp.warm_up(batch, loss_fn, min_steps=args.warmup)  # until steady-state replay
    if ddp.static_batch is not None:
        batch = ddp.static_batch      # graphs read these; no per-step device copy
    n0 = ddp.native_launches()
    clk.mark(True)
    ms = timed(lambda: ddp.train_step(batch, loss_fn), args.steps)
    clk.mark(False)
    launches = ddp.native_launches() - n0
    ms_step = ms / args.steps
    value = args.batch * world * args.steps / (ms / 1e3)

    # 3) e2e: every step's inputs copied from pinned host memory (on a copy stream,
    #    double-buffered so the copy for step t+1 overlaps step t) and every step's
    #    loss read back to pinned host memory
    hx = batch[0].cpu().pin_memory()
    hy = batch[1].cpu().pin_memory()
    loss_host = torch.empty(1, dtype=torch.float32).pin_memory()
    copy_stream = torch.cuda.Stream(device)
    staging = [(torch.empty_like(batch[0]), torch.empty_like(batch[1])) for _ in range(2)]
    loaded = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    state = {"i": 0}

    n_chunks = max(1, min(args.h2d_chunks, hx.shape[0]))
    bounds = [hx.shape[0] * c // n_chunks for c in range(n_chunks + 1)]

    def h2d(k):
        copy_stream.wait_event(consumed[k])
        with torch.cuda.stream(copy_stream):
            # batch-dim slices are contiguous (NCHW and NHWC alike): several
            # shorter DMA copies let the copy-engine channel's transfers interleave
            for a, b in zip(bounds, bounds[1:]):
                staging[k][0][a:b].copy_(hx[a:b], non_blocking=True)
            staging[k][1].copy_(hy, non_blocking=True)
        loaded[k].record(copy_stream)

    for k in range(2):
        consumed[k].record()
    h2d(0)

    def e2e_step():
        i = state["i"]
        cur, nxt = i % 2, (i + 1) % 2
        h2d(nxt)                                   # next step's inputs, overlapped
        torch.cuda.current_stream().wait_event(loaded[cur])
        loss = ddp.train_step(staging[cur], loss_fn)
        consumed[cur].record()
        loss_host.copy_(loss.float().reshape(1), non_blocking=True)
        state["i"] = i + 1

    for _ in range(2):
        e2e_step()
    ms_e2e = timed(e2e_step, args.steps)
    # keep the GPU loaded until the clock sampler has seen >= 1 s (short steps)
    pad_load(clk, lambda: ddp.train_step(batch, loss_fn), ms_step, world, dist, device)
    clk.end_load()
    e2e_value = args.batch * world * args.steps / (ms_e2e / 1e3)
    h2d_bytes = hx.numel() * hx.element_size() + hy.numel() * hy.element_size()

    # 4) kernel roofline: (a) in-step -- an instrumented eager pass with CUDA events
    #    around every native launch on its own stream; (b) isolated, barrier-aligned
    ddp.cfg.instrument = True
    ddp.timing_summary()
    n_instr = max(3, args.steps // 2)
    timed(lambda: ddp.train_step(batch, loss_fn), n_instr)
    ks = ddp.timing_summary()
    ddp.cfg.instrument = False
    iso = isolated_kernels(ddp, world, dist, device)

    pk = peaks()
    kind = "update" if world == 1 else max(iso, key=lambda k: iso[k]["ms_per_pass"])
    hbm_bound = world == 1
    peak = pk["hbm_gbs"] if hbm_bound else 770.0
    r = ks.get(kind)
    in_step = None
    if r:
        avg_ms = r["ms"] / r["launches"]
        in_step = (r["bytes"] / r["launches"]) / (avg_ms / 1e3) / 1e9
    achieved = iso[kind]["achieved_gbs"]
    # the kernels the step launches (csrc/bucket_comm.cu; env overrides as there)
    tma_upd = os.environ.get("DEFT_UPDATE_IMPL", "tma")[:1] != "l"
    tma_rs = os.environ.get("DEFT_RS_IMPL", "tma")[:1] != "l"
    upd_name = "sgd_local_kernel" if world == 1 else (
        ("update_allgather_tma_kernel" if tma_upd else "update_allgather_multi_kernel")
        if ddp.placement in ("end", "start", "bucket") else "update_allgather_kernel")
    rs_name = "reduce_scatter_tma_kernel" if tma_rs else "reduce_scatter_kernel"
    traffic = ncu_traffic(upd_name if kind == "update" else rs_name, args.model, world)
    roof = {"kernel": {"update": upd_name, "reduce_scatter": rs_name}[kind],
            "bound": "hbm" if hbm_bound else "nvlink",
            "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_src": "profiles/ncu_traffic.json (dram__bytes_read.sum + "
                           "dram__bytes_write.sum of one ncu --set full capture, per launch)"
            if traffic else None,
            "measured": "isolated over this model's buckets in the step's launch shape, each pass after an L2 flush, CUDA events, max over ranks (back-to-back CUDA-graph replay in isolated.*.graph_*)",
            "in_step_achieved": round(in_step, 1) if in_step else None,
            "in_step_note": "same kernel inside the training step (overlapping backward "
                            "compute; at W>1 includes cross-rank barrier waits)",
            "algorithmic_bytes": "W=1 update: 20 B/param of HBM traffic (read g,v,p; write v,p). "
                                 "W>1: bytes crossing NVLink per rank = (W-1)/W x bucket "
                                 "bytes, for the reduce-scatter (peer loads) and for the "
                                 "update+all-gather (peer stores) alike",
            "peak_src": (pk["src"] + " MEASURED_PEAKS.json hbm_gbs") if hbm_bound
            else "B200_PROFILING.md measured peer copy 770 GB/s",
            "isolated": iso, "in_step": ks}

    solver = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            solver = solver_measurement(full=args.solver_full)
        except Exception as e:  # reported, never fatal
            solver = {"error": repr(e)}
    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu_base = cpu_reference_run(args.model, 2, 1, 4)
        except Exception as e:  # reported, never fatal
            cpu_base = {"error": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            # arithmetic of the DeFT path itself: gradient reduce + SGD/momentum update
            "dtype": "bf16" if ddp.cfg.grad_dtype == torch.bfloat16 else "f32",
            "data": "synthetic (random-init weights, randn images / random tokens)",
            "config": {"workload": f"{args.model} " + (
                           "DeFT delayed-update DP" if args.scheme == "deft" else
                           f"{args.scheme} synchronous DP (reference baseline schedule)") +
                       ", batch "
                                   f"{args.batch}/GPU" + (", 224x224" if args.model != "gpt2"
                                                           else ", seq 1024"),
                       "model": args.model, "global_batch": args.batch * world,
                       "parallelism": f"dp{world}", "l2": "working set (activations) >> L2 126 MB",
                       "grad_dtype": str(ddp.cfg.grad_dtype).replace("torch.", ""),
                       "compute": "bf16 autocast" if args.model != "gpt2" else "bf16 weights",
                       "scheme": args.scheme, "update_placement": ddp.placement,
                       "buckets": part.n_buckets, "links": [l.name for l in ddp.cluster.links],
                       "capacity_multiplier": ddp.capacity_multiplier,
                       "partition_size": psize, "comm_scale": args.comm_scale,
                       "merge_counts": sorted({u.merge_count for pair in ddp.decision_log
                                               for d in pair for u in d.update_events}),
                       "cuda_graphs": ddp.cfg.cuda_graphs, "graph_choice": ddp.graph_choice,
                       "graphs_captured": len(ddp._graphs),
                       "oneshot_buckets": sum(ddp._oneshot), "defer_tail": ddp.cfg.defer_tail,
                       "warmup_steps_run": warm, "setup_s": round(t_setup, 2)},
            "e2e": {"value": round(e2e_value, 2), "unit": "samples/s",
                    "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": 4,
                    "note": "H2D on a copy stream, double-buffered (copy of step t+1 "
                            f"overlaps step t) in {n_chunks} batch slice(s); loss D2H every "
                            "step"},
            "gpu_launches": int(launches),
            "compute_only_ms_per_step": round(ms_compute, 3),
            "compute_only_modes": compute_modes,
            "exposed_comm_ms": round(ms_step - ms_compute, 3),
            "frac_of_compute_roofline": round(ms_compute / ms_step, 4),
            "roofline": roof,
            "cpu_baseline": cpu_base,
            "solver": solver,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    clk.__exit__()
    ddp.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
