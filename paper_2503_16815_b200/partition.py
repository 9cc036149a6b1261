"""Bucket partitioning (mirrors deftsim/partition.py:21-199).

Host-only input preparation.  It must be bit-exact with the reference
because it fixes the bucket ids, the solver weights and -- on B200 -- the
element ranges of the flat gradient buffer each bucket owns.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import InfeasiblePartitionError, check_rules
from .profiles import BucketProfile, ModelProfile

DEFAULT_PARTITION_SIZE = 6_500_000


@dataclass(frozen=True)
class PartitionConfig:
    """partition.py:21-34."""

    partition_size: int = DEFAULT_PARTITION_SIZE
    mu: float = 1.0
    enable_fusion: bool = False
    comm_startup_us: int = 0

    def __post_init__(self):
        check_rules(((self.partition_size > 0, "partition_size must be > 0"),
                     (self.mu >= 1.0, "mu must be >= 1"),
                     (self.comm_startup_us >= 0, "comm_startup_us must be >= 0")),
                    InfeasiblePartitionError)


def split_evenly(total: int, parts: int) -> list[int]:
    """``parts`` integers summing to ``total``; the first ``total % parts``
    pieces carry the extra unit (partition.py:37-40)."""
    q, r = divmod(total, parts)
    return [q + 1] * r + [q] * (parts - r)


def comm_capacity_bound_us(profile: ModelProfile, cfg: PartitionConfig) -> float:
    """Strict per-bucket comm bound: total forward time / mu (partition.py:43-45)."""
    return profile.total_forward_us / cfg.mu


def _pieces(b: BucketProfile, parts: int) -> list[BucketProfile]:
    # a piece keeps >= 1 parameter and >= 1 us of comm (partition.py:48-64)
    parts = max(1, min(parts, b.param_count, b.comm_fast_us))
    cols = [split_evenly(v, parts) for v in
            (b.param_count, b.forward_us, b.backward_us, b.comm_fast_us)]
    return [BucketProfile(0, p, f, w, c) for p, f, w, c in zip(*cols)]


def _parts_needed(b: BucketProfile, cfg: PartitionConfig, bound: float) -> int:
    parts = 1
    if b.param_count > cfg.partition_size:
        parts = math.ceil(b.param_count / cfg.partition_size)
    if b.comm_fast_us / parts >= bound:
        parts = max(parts, math.ceil(b.comm_fast_us / bound))
    # integer pieces round up, so keep splitting until the largest clears the bound
    while parts <= b.param_count and math.ceil(b.comm_fast_us / parts) >= bound:
        parts += 1
    return parts


def _renumber(profile: ModelProfile, pieces: list[BucketProfile]) -> ModelProfile:
    return ModelProfile(
        name=profile.name,
        buckets=tuple(BucketProfile(i, b.param_count, b.forward_us, b.backward_us,
                                    b.comm_fast_us) for i, b in enumerate(pieces, 1)),
        batch_size=profile.batch_size,
        learning_rate=profile.learning_rate,
        notes=dict(profile.notes),
    )


def partition_buckets(profile: ModelProfile, cfg: PartitionConfig) -> ModelProfile:
    """Split until the size and the strict capacity constraints hold
    (partition.py:67-120)."""
    bound = comm_capacity_bound_us(profile, cfg)
    pieces: list[BucketProfile] = []
    for b in profile.buckets:
        parts = _parts_needed(b, cfg, bound)
        if parts > b.param_count:
            raise InfeasiblePartitionError(
                f"bucket {b.id}: comm time {b.comm_fast_us}us cannot be split "
                f"below the capacity bound {bound:.1f}us", bucket_id=b.id)
        pieces.extend([b] if parts == 1 else _pieces(b, parts))
    for i, b in enumerate(pieces, 1):
        if b.comm_fast_us >= bound:
            raise InfeasiblePartitionError(
                f"bucket piece {i}: comm {b.comm_fast_us}us >= bound {bound:.1f}us",
                bucket_id=i)
    return _renumber(profile, pieces)


def partition_by_size(profile: ModelProfile, partition_size: int) -> ModelProfile:
    """Size-only split used by the baselines (partition.py:123-151)."""
    if partition_size <= 0:
        raise InfeasiblePartitionError("partition_size must be > 0")
    pieces: list[BucketProfile] = []
    for b in profile.buckets:
        parts = math.ceil(b.param_count / partition_size)
        pieces.extend([b] if parts == 1 else _pieces(b, parts))
    return _renumber(profile, pieces)


def fuse_buckets(profile: ModelProfile, comm_startup_us: int,
                 cfg: PartitionConfig) -> ModelProfile:
    """Merge adjacent buckets while the merged payload stays under the bound
    and a startup cost exists (partition.py:154-199)."""
    if comm_startup_us < 0:
        raise InfeasiblePartitionError("comm_startup_us must be >= 0")
    bound = comm_capacity_bound_us(profile, cfg)
    out: list[BucketProfile] = []
    for b in profile.buckets:
        if out and comm_startup_us > 0 and out[-1].comm_fast_us + b.comm_fast_us < bound:
            a = out[-1]
            out[-1] = BucketProfile(a.id, a.param_count + b.param_count,
                                    a.forward_us + b.forward_us,
                                    a.backward_us + b.backward_us,
                                    a.comm_fast_us + b.comm_fast_us)
        else:
            out.append(b)
    return _renumber(profile, out)


def element_ranges(profile: ModelProfile, original: ModelProfile | None = None
                   ) -> list[tuple[int, int]]:
    """[start, end) element offsets of every bucket in the flat, output-side-first
    gradient buffer.  Bucket b occupies param_count elements right after b-1,
    which is how the reference's proportional splits (partition.py:48-64) map
    onto a real parameter buffer."""
    out, start = [], 0
    for b in profile.buckets:
        out.append((start, start + b.param_count))
        start += b.param_count
    if original is not None and start != original.total_param_count:
        raise InfeasiblePartitionError("partition does not conserve the parameter count")
    return out
