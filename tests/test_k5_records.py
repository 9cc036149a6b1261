"""K5's record layout (csrc/scheduler_kernel.cu) round-trips through the host
decoder into the exact ScheduleDecision objects (and exec notes) the host state
machine produces -- checked on CPU over the golden streams by encoding the
host decisions in the kernel's layout."""
import numpy as np
import pytest

from oracle import deft_oracle as O
import paper_2503_16815_b200 as D
from paper_2503_16815_b200 import gpu_scheduler as G
from paper_2503_16815_b200 import knapsack as K
from test_host_logic import build_product_inputs


def encode(decisions):
    """The kernel's layout: header (stage, case, n_transfers, n_events, merged,
    grad_group, grad_merge), transfers (link, id, group, fresh), events
    (uid, first_origin, merge_count)."""
    out = []
    for d in decisions:
        ex = d.exec
        if d.stage == "forward":
            out += [0, 1, len(ex.transfers), 0, 0, -1, 0]
        else:
            out += [1, d.case_taken.value, len(ex.transfers), len(ex.updates),
                    int(bool(d.merged)), ex.grad_group, int(ex.grad_merge)]
        for t in ex.transfers:
            out += [t.link, t.bucket_id, t.group, int(t.fresh)]
        if d.stage == "backward":
            for uid, k, origins in ex.updates:
                assert list(origins) == list(range(origins[0], origins[0] + k))
                out += [uid, origins[0], k]
    return np.array(out, dtype=np.int32)


@pytest.fixture(autouse=True)
def oracle_dp():
    with K.subset_sum_backend(O.subset_sum_c_batch):
        yield


def test_record_round_trip(golden_index, golden_inputs):
    n_checked = 0
    for e in golden_index:
        if len(e["partitioned"]) > 60:
            continue
        prof, cluster, cfg, mult, iters = build_product_inputs(e, golden_inputs)
        part = D.partition_buckets(prof, cfg) if cfg is not None else prof
        iters = min(iters, 80)
        want = D.DeftScheduler(part, cluster, mult).run(iters)
        rec = encode(want)
        ks = G.KernelSchedule(rec, len(rec), [l.name for l in cluster.links],
                              tuple(b.id for b in part.buckets), iters)
        got = ks.decisions()
        assert got == want
        assert [a.exec for a in got] == [b.exec for b in want]
        assert ks.merge_counts() == [u.merge_count for d in want for u in d.update_events]
        n_checked += 1
    assert n_checked >= 45
