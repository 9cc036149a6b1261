"""Experiments on the B200 with the reference's report schema.

The reference plans and SIMULATES an experiment grid -- schemes x sweep points --
and writes ``summary.json`` / ``comparison.csv`` / ``plotdata/*.csv``
(cli.py:52-391).  This module reads the same experiment JSON, RUNS every
(scheme, point) on the GPUs through ``DeftDataParallel`` and writes the same
files from measured CUDA-event timings, so simulator-vs-hardware comparisons
line up column for column.

What the fields mean on hardware (``RunReport.from_measurement``):
  * ``total_time_us``          CUDA-event time of the ``iterations`` timed steps
                               (max over ranks);
  * ``mean_iteration_time_us`` total / iterations;
  * ``bubble_time_us``         time the steps exceed the compute-only step (one
                               GPU's forward + backward [+ local optimizer step],
                               no communication), i.e. exposed
                               communication -- the simulator's compute idle time
                               (simulator.py:250-256);
  * ``updates_performed``      update events applied inside the timed steps;
  * ``throughput_samples_per_s`` per-GPU samples/s (profile batch size, as
                               simulator.py:258).
Sweep axes: ``partition_size`` re-partitions the real buckets; ``bandwidth_scale``
scales the PLANNED communication times (the schedule DeFT computes), the
links themselves run at NVLink speed; ``gpu_count`` points other than the
launched world size are skipped.  ``nonsequential`` (scheduler.py:421-472)
runs its candidate search on the executor: the four candidates are scored by
a timed hardware probe on this batch instead of ``simulate()``.
"""
from __future__ import annotations

import csv
import hashlib
import json
from dataclasses import dataclass, field, replace
from pathlib import Path
from typing import Callable

from .errors import ComparisonError, SchemaError
from .partition import PartitionConfig
from .preserver import WalkParams, check_sequence, extract_batch_sequence
from .profiles import ClusterSpec, ModelProfile
from .scheduler import SCHEMES, Schedule

HW_SCHEMES = ("wfbp", "priority", "nonsequential", "deft", "deft_single_link")


# ----------------------------------------------------------------- config (cli.py:52-226)
#
# The experiment file's schema as data: which keys are required, the "partition"
# block's fields with their casts and defaults, and the sweep axes with the
# ExperimentConfig field each one fills.  Defaults, validation and messages follow
# cli.py:70-143 so a file the reference accepts (or rejects) behaves the same here;
# the reference's "sim" block configures its simulator and is ignored.

_REQUIRED_KEYS = ("profile", "schemes", "iterations")
_PARTITION_SCHEMA = (("partition_size", int, 6_500_000), ("mu", float, 1.0),
                     ("enable_fusion", bool, False), ("comm_startup_us", int, 0))
_SWEEP_SCHEMA = (("bandwidth_scale", "bandwidth_scales", float),
                 ("partition_size", "partition_sizes", int),
                 ("gpu_counts", "gpu_counts", int))


@dataclass(frozen=True)
class SweepPoint:
    """One grid point; every axis at its base value is the base point (cli.py:52-67)."""

    bandwidth_scale: float = 1.0
    partition_size: int | None = None
    gpu_count: int | None = None

    def label(self) -> str:
        tags = (f"bw{self.bandwidth_scale:g}" if self.bandwidth_scale != 1.0 else "",
                f"ps{self.partition_size}" if self.partition_size is not None else "",
                f"gpu{self.gpu_count}" if self.gpu_count is not None else "")
        return "_".join(t for t in tags if t) or "base"


@dataclass(frozen=True)
class ExperimentConfig:
    """The parsed experiment file (cli.py:70-97)."""

    profile_path: str
    cluster_path: str | None
    cluster_inline: dict | None
    schemes: tuple[str, ...]
    iterations: int
    partition: PartitionConfig
    walk: WalkParams | None
    bandwidth_scales: tuple[float, ...] = ()
    partition_sizes: tuple[int, ...] = ()
    gpu_counts: tuple[int, ...] = ()

    def __post_init__(self):
        checks = (
            (self.iterations >= 1, "iterations must be >= 1"),
            (bool(self.schemes), "schemes must be non-empty"),
            (all(s in SCHEMES for s in self.schemes),
             f"unknown schemes {[s for s in self.schemes if s not in SCHEMES]}; "
             f"valid: {list(SCHEMES)}"),
            (all(x > 0 for x in self.bandwidth_scales), "bandwidth_scale values must be > 0"),
            (all(x > 0 for x in self.partition_sizes), "partition_size values must be > 0"),
            (all(x >= 2 for x in self.gpu_counts), "gpu_counts values must be >= 2"),
        )
        for ok, msg in checks:
            if not ok:
                raise SchemaError(msg)


def experiment_config_from_dict(data: dict, base_dir: Path) -> ExperimentConfig:
    """cli.py:100-143: the file's dict -> ExperimentConfig, paths relative to base_dir."""
    if not isinstance(data, dict):
        raise SchemaError("experiment config must be a JSON object")
    for key in _REQUIRED_KEYS:
        if key not in data:
            raise SchemaError(f"experiment config: missing field {key!r}")
    block = data.get("partition", {})
    partition = PartitionConfig(**{name: cast(block.get(name, default))
                                   for name, cast, default in _PARTITION_SCHEMA})
    sweeps = data.get("sweeps", {})
    axes = {}
    for key, field_name, cast in _SWEEP_SCHEMA:
        values = sweeps.get(key, [])
        if key in sweeps and not values:
            raise SchemaError(f"sweep axis {key!r} must be non-empty when present")
        axes[field_name] = tuple(cast(v) for v in values)
    base = Path(base_dir)
    cluster = data.get("cluster")
    inline = cluster if isinstance(cluster, dict) else None
    return ExperimentConfig(
        profile_path=str(base / data["profile"]),
        cluster_path=None if cluster is None or inline is not None else str(base / cluster),
        cluster_inline=inline,
        schemes=tuple(data["schemes"]),
        iterations=int(data["iterations"]),
        partition=partition,
        walk=WalkParams.from_dict(data["walk"]) if "walk" in data else None,
        **axes)


def load_experiment_config(path) -> ExperimentConfig:
    """cli.py:146-152."""
    path = Path(path)
    try:
        raw = json.loads(path.read_text())
    except json.JSONDecodeError as e:
        raise SchemaError(f"{path}: invalid JSON ({e})") from e
    return experiment_config_from_dict(raw, path.parent)


def sweep_points(cfg: ExperimentConfig) -> list[SweepPoint]:
    """The base point, then every axis value away from its base on its own; with a
    gpu_counts axis its first entry is the reference size and is dropped
    (cli.py:160-175)."""
    grid = [SweepPoint()]
    grid += [SweepPoint(bandwidth_scale=x) for x in cfg.bandwidth_scales if x != 1.0]
    grid += [SweepPoint(partition_size=x) for x in cfg.partition_sizes
             if x != cfg.partition.partition_size]
    if not cfg.gpu_counts:
        return grid
    reference = cfg.gpu_counts[0]
    grid += [SweepPoint(gpu_count=g) for g in cfg.gpu_counts[1:]]
    return [p for p in grid if p.gpu_count != reference]


def point_profile(profile: ModelProfile, point: SweepPoint,
                  gpu_reference: int | None) -> ModelProfile:
    """The profile a grid point plans with: communication times scaled by
    1/bandwidth_scale and, for a gpu_count point, by the ring all-reduce volume
    2(p-1)/p relative to the reference size (cli.py:178-186)."""
    factor = 1.0 / point.bandwidth_scale
    if point.gpu_count is not None and gpu_reference:
        ring = lambda p: 2.0 * (p - 1) / p   # noqa: E731
        factor *= ring(point.gpu_count) / ring(gpu_reference)
    return profile if factor == 1.0 else profile.scaled_comm(factor, name_suffix="")


def config_hash(cfg: ExperimentConfig, seed: int) -> str:
    """First 16 hex digits of sha256 over the experiment's identity -- the same
    JSON document cli.py:211-226 hashes, so a hardware run and a simulated run of
    one experiment file carry the same hash."""
    identity = {
        "profile": Path(cfg.profile_path).name,
        "schemes": list(cfg.schemes),
        "iterations": cfg.iterations,
        "partition": dict(vars(cfg.partition)),
        "walk": dict(vars(cfg.walk)) if cfg.walk else None,
        "seed": seed,
    }
    identity.update({field_name: list(getattr(cfg, field_name))
                     for _, field_name, _ in _SWEEP_SCHEMA})
    return hashlib.sha256(json.dumps(identity, sort_keys=True).encode()).hexdigest()[:16]


# ------------------------------------------------------------ reports (simulator.py:64-300)

@dataclass(frozen=True)
class RunReport:
    """The fields of SimReport.summary_dict (simulator.py:75-86)."""

    scheme: str
    profile_name: str
    iterations: int
    total_time_us: int
    mean_iteration_time_us: float
    bubble_time_us: int
    bubble_ratio: float
    updates_performed: int
    throughput_samples_per_s: float

    @classmethod
    def from_measurement(cls, scheme: str, profile_name: str, iterations: int,
                         total_ms: float, compute_only_ms_per_step: float,
                         batch_size: int, updates_performed: int) -> "RunReport":
        total_us = int(round(total_ms * 1e3))
        bubble = max(0, total_us - int(round(compute_only_ms_per_step * 1e3 * iterations)))
        return cls(scheme, profile_name, iterations, total_us,
                   total_us / iterations if iterations else 0.0, bubble,
                   bubble / total_us if total_us > 0 else 0.0, updates_performed,
                   iterations * batch_size / (total_us / 1e6) if total_us > 0 else 0.0)

    # summary.json's "report" block: (key, attribute, digits kept or None) in the
    # reference's key set (simulator.py:262-273)
    _SUMMARY = (("scheme", "scheme", None), ("profile", "profile_name", None),
                ("iterations", "iterations", None), ("total_time_us", "total_time_us", None),
                ("mean_iteration_time_us", "mean_iteration_time_us", 3),
                ("bubble_time_us", "bubble_time_us", None), ("bubble_ratio", "bubble_ratio", 6),
                ("updates_performed", "updates_performed", None),
                ("throughput_samples_per_s", "throughput_samples_per_s", 3))

    def summary_dict(self) -> dict:
        return {key: getattr(self, attr) if digits is None else round(getattr(self, attr), digits)
                for key, attr, digits in self._SUMMARY}


def compare(reports: dict[str, RunReport], baseline: str = "wfbp") -> dict:
    """Every scheme's totals and its speedup over the named baseline, schemes in
    name order (simulator.py:276-300: same checks, rounding and keys)."""
    if not reports:
        raise ComparisonError("no reports to compare")
    iteration_counts = sorted({r.iterations for r in reports.values()})
    if len(iteration_counts) != 1:
        raise ComparisonError(f"iteration counts differ: {iteration_counts}")
    if baseline not in reports:
        raise ComparisonError(f"baseline {baseline!r} missing from reports")
    t_base = reports[baseline].total_time_us

    def row(name: str, r: RunReport) -> dict:
        speedup = round(t_base / r.total_time_us, 4) if r.total_time_us else 0.0
        return {"scheme": name, "profile": r.profile_name, "total_time_us": r.total_time_us,
                "mean_iteration_time_us": round(r.mean_iteration_time_us, 3),
                "bubble_ratio": round(r.bubble_ratio, 6),
                "updates_performed": r.updates_performed, f"speedup_vs_{baseline}": speedup}
    return {"baseline": baseline,
            "profiles": sorted({r.profile_name for r in reports.values()}),
            "rows": [row(name, reports[name]) for name in sorted(reports)]}


@dataclass
class RunRecord:
    """One (scheme, sweep point) run of an experiment and its report (cli.py:189-199)."""

    scheme: str
    point: SweepPoint
    report: RunReport
    schedule_scheme: str
    verdict: dict | None
    hardware: dict | None = None     # measured extras (world size, compute-only step, ...)

    @property
    def run_id(self) -> str:
        return f"{self.scheme}__{self.point.label()}"


@dataclass
class ReportBundle:
    """Every run of an experiment plus its identity (cli.py:202-208)."""

    config_hash: str
    runs: list[RunRecord]
    iterations: int
    skipped: list[dict] = field(default_factory=list)

    def by_point(self) -> dict[str, dict[str, RunRecord]]:
        """sweep-point label -> scheme -> run."""
        grid: dict[str, dict[str, RunRecord]] = {}
        for run in self.runs:
            grid.setdefault(run.point.label(), {})[run.scheme] = run
        return grid


def _write_csv(path: Path, header: list[str], rows: list[list]) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(header)
        w.writerows(rows)


_COMPARISON_HEADER = ["sweep_point", "scheme", "total_time_us", "mean_iteration_time_us",
                      "bubble_ratio", "updates_performed", "speedup_vs_baseline"]


def _run_doc(r: RunRecord) -> dict:
    """One run of summary.json: the reference's keys (cli.py:299-316), plus the
    hardware block of a GPU run."""
    p = r.point
    doc = {"run_id": r.run_id, "scheme": r.scheme, "report": r.report.summary_dict(),
           "preserver": r.verdict,
           "sweep_point": {"bandwidth_scale": p.bandwidth_scale,
                           "partition_size": p.partition_size, "gpu_count": p.gpu_count}}
    if r.hardware is not None:
        doc["hardware"] = r.hardware
    return doc


def _comparison_rows(bundle: ReportBundle) -> list[list]:
    """comparison.csv: every scheme against wfbp (else the first scheme by name) at
    every sweep point (cli.py:325-343)."""
    out = []
    for label, by_scheme in sorted(bundle.by_point().items()):
        base = "wfbp" if "wfbp" in by_scheme else min(by_scheme)
        table = compare({name: run.report for name, run in by_scheme.items()}, base)
        out += [[label] + [row[k] for k in ("scheme", "total_time_us", "mean_iteration_time_us",
                                            "bubble_ratio", "updates_performed")]
                + [row["speedup_vs_" + base]] for row in table["rows"]]
    return out


def _speedup_curves(bundle: ReportBundle):
    """plotdata/: speedup vs wfbp along the bandwidth and the partition-size axes
    (cli.py:354-389) -> (file name, header, rows), empty curves left out."""
    by_point = bundle.by_point()
    scales = sorted({r.point.bandwidth_scale for r in bundle.runs} - {1.0})
    sizes = sorted({r.point.partition_size for r in bundle.runs if r.point.partition_size})
    axes = (("speedup_vs_bandwidth.csv", "bandwidth_scale",
             [("base", 1.0)] + [(SweepPoint(bandwidth_scale=x).label(), x) for x in scales]),
            ("speedup_vs_partition_size.csv", "partition_size",
             [(SweepPoint(partition_size=x).label(), x) for x in sizes]))
    for fname, axis, points in axes:
        rows = []
        for label, x in points:
            runs = by_point.get(label, {})
            if "wfbp" in runs:
                t_base = runs["wfbp"].report.total_time_us
                rows += [[x, name, round(t_base / runs[name].report.total_time_us, 4)
                          if runs[name].report.total_time_us else 0.0]
                         for name in sorted(runs)]
        if rows:
            yield fname, [axis, "scheme", "speedup_vs_wfbp"], rows


def emit_reports(bundle: ReportBundle, out_dir) -> list[Path]:
    """summary.json, comparison.csv and plotdata/ in the schema of cli.py:294-391
    (timeline / Chrome-trace files are simulator output and not written)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    summary = {"config_hash": bundle.config_hash, "iterations": bundle.iterations,
               "runs": [_run_doc(r) for r in sorted(bundle.runs, key=lambda r: r.run_id)]}
    if bundle.skipped:
        summary["skipped"] = bundle.skipped
    files = [out / "summary.json"]
    files[0].write_text(json.dumps(summary, indent=2, sort_keys=True) + "\n")
    if not bundle.runs:
        return files
    files.append(out / "comparison.csv")
    _write_csv(files[-1], _COMPARISON_HEADER, _comparison_rows(bundle))
    (out / "plotdata").mkdir(exist_ok=True)
    for fname, header, rows in _speedup_curves(bundle):
        files.append(out / "plotdata" / fname)
        _write_csv(files[-1], header, rows)
    return files


# ------------------------------------------------------------------- running on GPUs

def preserver_verdict(schedule: Schedule, walk: WalkParams) -> dict:
    """The verdict block of cli.py:255-266."""
    seq = extract_batch_sequence(schedule)
    preserved, ratio, merged, base = check_sequence(seq, walk)
    return {"preserved": preserved, "ratio": round(ratio, 6),
            "expected_state": round(merged, 9), "baseline_state": round(base, 9),
            "k_values": list(seq.k_values)}


def run_hw_experiment(cfg: ExperimentConfig, make_model: Callable, batch, loss_fn: Callable,
                      seed: int = 0, warmup: int = 3, executor_kwargs: dict | None = None,
                      process_group=None, log: Callable | None = None,
                      compute_only_ms: Callable | None = None) -> ReportBundle:
    """Run every (scheme, sweep point) of ``cfg`` on this process's GPU (one
    process per GPU, all ranks call it).  ``make_model()`` builds a fresh
    random-init model on the device for each run; the B200 profile is measured
    once (CUDA events) and shared by every run, as the reference shares its
    fixture profile.  ``compute_only_ms(model)`` times one forward+backward step
    without communication or update (default: eager, under the executor's
    autocast).  Returns the bundle (``emit_reports`` writes it)."""
    import torch

    from .executor import DeftConfig, DeftDataParallel

    import contextlib
    import gc

    dist = torch.distributed
    ac_dtype = (executor_kwargs or {}).get("autocast_dtype", torch.bfloat16)

    def autocast():
        if ac_dtype is None:
            return contextlib.nullcontext()
        return torch.autocast("cuda", dtype=ac_dtype)

    world = dist.get_world_size(process_group) if dist.is_initialized() else 1
    kw = dict(executor_kwargs or {})

    def executor(scheme, partition):
        model = make_model()
        dcfg = DeftConfig(scheme="deft" if scheme.startswith("deft") else scheme,
                          partition=partition, **kw)
        return model, DeftDataParallel(model, dcfg, process_group=process_group)

    def timed_steps(ddp, model, n):
        if world > 1:
            dist.barrier(group=process_group)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            if ddp is None:
                model.zero_grad(set_to_none=True)
                with autocast():
                    loss = loss_fn(model, batch)
                loss.backward()
            else:
                ddp.train_step(batch, loss_fn)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([ms], device=torch.device("cuda", torch.cuda.current_device()))
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=process_group)
            ms = float(t.item())
        return ms

    # the profile of THIS hardware, measured once
    model, ddp = executor("deft", cfg.partition)
    profile = ddp.measure_profile(batch, loss_fn, iters=3,
                                  name=Path(cfg.profile_path).stem,
                                  batch_size=int(batch[0].shape[0]))
    cluster = ddp.cluster
    ddp.close()
    # compute-only step (forward + backward, no communication, no update)
    model = make_model()
    if compute_only_ms is not None:
        compute_ms = compute_only_ms(model)
    else:
        timed_steps(None, model, warmup)
        compute_ms = timed_steps(None, model, cfg.iterations) / cfg.iterations
    del model

    gpu_ref = cfg.gpu_counts[0] if cfg.gpu_counts else None
    runs, skipped = [], []
    for point in sweep_points(cfg):
        if point.gpu_count is not None and point.gpu_count != world:
            skipped.append({"sweep_point": point.label(),
                            "reason": f"launched on {world} GPU(s)"})
            continue
        p_profile = point_profile(profile, point, gpu_ref)
        p_partition = cfg.partition
        if point.partition_size is not None:
            p_partition = replace(cfg.partition, partition_size=point.partition_size)
        for scheme in cfg.schemes:
            if scheme not in HW_SCHEMES:
                skipped.append({"sweep_point": point.label(), "scheme": scheme,
                                "reason": "simulator-scored baseline, not an executor "
                                          "schedule (DESIGN.md §7)"})
                continue
            model, ddp = executor(scheme, p_partition)
            links = (ClusterSpec(links=(cluster.fast_link,))
                     if scheme == "deft_single_link" else cluster)
            # nonsequential: the candidates are timed on this hardware, not simulated
            probe = (batch, loss_fn) if scheme == "nonsequential" else None
            part = ddp.plan(p_profile, links, probe=probe)
            ddp.warm_up(batch, loss_fn, min_steps=warmup)
            u0 = ddp.updates_applied
            total_ms = timed_steps(ddp, model, cfg.iterations)
            updates = ddp.updates_applied - u0
            verdict = None
            if scheme.startswith("deft") and cfg.walk is not None:
                decisions = [d for pair in ddp.decision_log[:cfg.iterations] for d in pair]
                verdict = preserver_verdict(
                    Schedule(scheme, part, links, decisions, True, cfg.iterations), cfg.walk)
            report = RunReport.from_measurement(
                scheme, profile.name, cfg.iterations, total_ms, compute_ms,
                profile.batch_size, updates)
            runs.append(RunRecord(scheme, point, report, scheme, verdict, hardware={
                "world": world, "buckets": part.n_buckets,
                "links": [l.name for l in links.links],
                "compute_only_ms_per_step": round(compute_ms, 4),
                "global_samples_per_s": round(report.throughput_samples_per_s * world, 2),
                "update_placement": ddp.placement,
                "graph_choice": ddp.graph_choice}))
            if log is not None:
                log(runs[-1])
            ddp.close()
            del model, ddp
            gc.collect()                  # captured graphs and their pools
            torch.cuda.empty_cache()
    return ReportBundle(config_hash(cfg, seed), runs, cfg.iterations, skipped)
