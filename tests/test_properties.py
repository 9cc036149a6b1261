"""Property tests (hypothesis) of the product's host logic, mirroring the
reference's own property tests (test_knapsack.py:81-91, 176-187; test_partition.py:88-107;
test_profiles.py:115-128) plus the executor planner's invariants on random
schedules.  The DP runs through the CPU oracle backend here (no GPU); the same
wrappers run the sm_100a kernel in the GPU tests."""
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2503_16815_b200 as D
from paper_2503_16815_b200 import knapsack as K
from paper_2503_16815_b200.planner import (ExecutionPlanner, release_runs, start_groups,
                                           start_groups_timed)
from oracle import deft_oracle as O
from test_planner import check_invariants


@pytest.fixture(autouse=True)
def oracle_dp():
    with K.subset_sum_backend(O.subset_sum_c_batch):
        yield


def items_of(ws):
    return [D.Item(i + 1, w) for i, w in enumerate(ws)]


@given(st.lists(st.integers(1, 200), min_size=1, max_size=12), st.integers(0, 1500))
@settings(max_examples=150, deadline=None)
def test_naive_selection_partitions_items(weights, cap):
    with K.subset_sum_backend(O.subset_sum_c_batch):
        asn = D.naive_knapsack(items_of(weights), cap)
    sel = set(asn.selections[0])
    assert sel | set(asn.leftovers) == set(range(1, len(weights) + 1))
    assert not sel & set(asn.leftovers)
    assert sum(weights[i - 1] for i in sel) == asn.total_value <= cap


@given(st.lists(st.integers(1, 50), min_size=1, max_size=7), st.integers(0, 200))
@settings(max_examples=100, deadline=None)
def test_recursive_with_zero_backward_is_the_optimum(weights, remain):
    with K.subset_sum_backend(O.subset_sum_c_batch):
        order = D.recursive_knapsack(items_of(weights), remain, [0] * len(weights))
        want = D.naive_knapsack(items_of(weights), remain).total_value
    assert sum(weights[i - 1] for i in order) == want


@given(st.lists(st.integers(1, 400), max_size=18),
       st.lists(st.integers(0, 900), min_size=1, max_size=4))
@settings(max_examples=200, deadline=None)
def test_greedy_feasible(weights, caps):
    asn = D.greedy_multi_knapsack(items_of(weights), caps)
    seen = []
    for k, sel in enumerate(asn.selections):
        assert sum(weights[i - 1] for i in sel) <= caps[k]
        seen.extend(sel)
    assert len(seen) == len(set(seen))
    assert set(seen) | set(asn.leftovers) == set(range(1, len(weights) + 1))


rows_st = st.lists(st.tuples(st.integers(1, 10**6), st.integers(1, 10**4),
                             st.integers(1, 10**4), st.integers(1, 10**4)),
                   min_size=1, max_size=8)


def profile_of(rows):
    return D.ModelProfile(name="p", buckets=tuple(
        D.BucketProfile(i + 1, p, f, b, c) for i, (p, f, b, c) in enumerate(rows)),
        batch_size=32)


@given(rows_st, st.integers(1, 10**5))
@settings(max_examples=120, deadline=None)
def test_partition_by_size_conserves(rows, size):
    p = profile_of(rows)
    out = D.partition_by_size(p, size)
    assert out.total_param_count == p.total_param_count
    assert out.total_forward_us == p.total_forward_us
    assert out.total_backward_us == p.total_backward_us
    assert out.total_comm_fast_us == p.total_comm_fast_us
    assert [b.id for b in out.buckets] == list(range(1, out.n_buckets + 1))


@given(rows_st, st.integers(1, 10**6), st.floats(1.0, 3.0))
@settings(max_examples=120, deadline=None)
def test_partition_buckets_bound_and_conservation(rows, size, mu):
    p = profile_of(rows)
    cfg = D.PartitionConfig(partition_size=size, mu=mu)
    try:
        out = D.partition_buckets(p, cfg)
    except D.InfeasiblePartitionError:
        return
    assert out.total_param_count == p.total_param_count
    bound = D.comm_capacity_bound_us(p, cfg)
    assert all(b.comm_fast_us < bound for b in out.buckets)
    # the flat-buffer ranges tile [0, total) in bucket order
    ranges = D.partition.element_ranges(out, None)
    assert ranges[0][0] == 0 and ranges[-1][1] == out.total_param_count
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


@given(rows_st)
@settings(max_examples=80, deadline=None)
def test_profile_round_trip(rows):
    p = profile_of(rows)
    assert D.profile_from_dict(D.profile_to_dict(p)) == p


@given(rows_st, st.floats(1.0, 10.0))
@settings(max_examples=80, deadline=None)
def test_comm_time_monotone_in_ratio(rows, ratio):
    p = profile_of(rows)
    fast, slow = D.LinkSpec("f"), D.LinkSpec("s", speed_ratio_to_fast=ratio)
    for b in p.buckets:
        assert D.comm_time_on_link(b, slow) >= D.comm_time_on_link(b, fast)


@given(st.integers(4, 24), st.integers(100, 3000), st.sampled_from([0, 1, 2]),
       st.floats(1.0, 1.5))
@settings(max_examples=40, deadline=None)
def test_planner_invariants_random_schedules(n, comm_us, lag, mult):
    """Uniform profiles with random comm times (k = 1 .. several merges) through
    the DeFT state machine: slot lifetimes, transfer coverage and update timing
    hold for every lag the executor uses."""
    fwd, bwd = 3600, 7200
    prof = D.ModelProfile(name="u", buckets=tuple(
        D.BucketProfile(i + 1, 1000, fwd // n, bwd // n, comm_us) for i in range(n)),
        batch_size=32)
    cluster = D.ClusterSpec(links=(D.LinkSpec("fast"), D.LinkSpec("slow", 1.65)))
    sched = D.DeftScheduler(prof, cluster, mult)
    check_invariants(ExecutionPlanner(sched, 8, lag=lag), n, 40)


@given(st.lists(st.integers(1, 10**7), min_size=1, max_size=40), st.integers(1, 10))
@settings(max_examples=150, deadline=None)
def test_start_groups_partition_in_forward_order(sizes, max_groups):
    for groups in (start_groups(sizes, max_groups),
                   start_groups_timed(sizes, [float(s % 997) for s in sizes], 1e-5, 20.0,
                                      max_groups)):
        assert [b for g in groups for b in g] == list(range(len(sizes) - 1, -1, -1))
        assert 1 <= len(groups) <= max(1, min(max_groups, len(sizes)))
        assert all(g for g in groups)


@given(st.lists(st.tuples(st.integers(0, 2), st.integers(0, 3), st.integers(0, 50)),
                max_size=30))
@settings(max_examples=150, deadline=None)
def test_release_runs_preserve_per_link_order(transfers):
    runs = release_runs(transfers)
    for link in {l for l, _, _ in transfers}:
        assert [b for l, _, bl in runs if l == link for b in bl] == \
            [b for l, _, b in transfers if l == link]
    assert sum(len(bl) for _, _, bl in runs) == len(transfers)
    assert all(bl for _, _, bl in runs)
    # no two adjacent runs of one link share a slot (they would have merged)
    for link in {l for l, _, _ in transfers}:
        slots = [s for l, s, _ in runs if l == link]
        assert all(a != b for a, b in zip(slots, slots[1:]))


@given(st.integers(1, 4096), st.integers(1, 4096))
@settings(max_examples=60, deadline=None)
def test_larger_batch_never_worse(b1, b2):
    """preserver.py:97-112 via the product's restatement: the expected next state
    is monotone non-increasing in the batch size (reference
    test_preserver.py:66-75), and never below the optimum."""
    p = D.WalkParams(s0=0.3, s_star=0.0, eta=0.01, mu_t=1.0, sigma_t=30.0)
    lo, hi = sorted((b1, b2))
    assert D.expected_next_state(0.3, hi, p) <= D.expected_next_state(0.3, lo, p) + 1e-12
    q = D.WalkParams(s0=0.2, s_star=0.05, eta=0.1, mu_t=5.0, sigma_t=2.0)
    assert D.expected_next_state(0.2, lo, q) >= q.s_star


@given(st.integers(4, 24), st.integers(100, 3000), st.floats(1.0, 1.5))
@settings(max_examples=30, deadline=None)
def test_sequence_from_merge_counts_equals_extract(n, comm_us, mult):
    """The lazy K5 path builds the preserver's batch sequence from the update
    events' merge counts alone; it must equal extract_batch_sequence of the full
    decision stream (preserver.py:137-168)."""
    from paper_2503_16815_b200.preserver import sequence_from_merge_counts
    prof = D.ModelProfile(name="u", buckets=tuple(
        D.BucketProfile(i + 1, 1000, 3600 // n, 7200 // n, comm_us) for i in range(n)),
        batch_size=32)
    cluster = D.ClusterSpec(links=(D.LinkSpec("fast"), D.LinkSpec("slow", 1.65)))
    iters = 120
    decisions = D.DeftScheduler(prof, cluster, mult).run(iters)
    sched = D.Schedule("deft", prof, cluster, decisions, True, iters)
    ks = [u.merge_count for d in decisions for u in d.update_events]
    try:
        want = D.extract_batch_sequence(sched)
    except D.DeftError as e:
        with pytest.raises(type(e)):
            sequence_from_merge_counts(ks, prof.batch_size, iters)
        return
    got = sequence_from_merge_counts(ks, prof.batch_size, iters)
    assert got == want
