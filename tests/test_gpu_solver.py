"""K1 parity on the B200: the product solver path (C-ABI -> sm_100a kernel)
against the reference's golden vectors and against the C oracle on random
instances.  Bit-exact everywhere (integer work)."""
import hashlib
import random

import pytest

from conftest import golden_schedule_text, read_jsonl_gz
from oracle import deft_oracle as O
import paper_2503_16815_b200 as D
from paper_2503_16815_b200 import _native

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_naive_golden_on_gpu():
    before = _native.launch_count()
    for r in read_jsonl_gz("naive.jsonl.gz"):
        items = [D.Item(i, w) for i, w in zip(r["ids"], r["weights"])]
        asn = D.naive_knapsack(items, r["cap"])
        assert asn.selections == (tuple(r["selection"]),), r
        assert asn.total_value == r["value"]
        assert asn.leftovers == tuple(r["leftovers"])
    assert _native.launch_count() > before  # the kernel really ran


def test_recursive_golden_on_gpu():
    for r in read_jsonl_gz("recursive.jsonl.gz"):
        items = [D.Item(i, w) for i, w in zip(r["ids"], r["weights"])]
        assert D.recursive_knapsack(items, r["remain"], r["backward"]) == r["order"], r


def _random_problems(rng, count, n_lo, n_hi, cap_lo, cap_hi):
    out = []
    for _ in range(count):
        n = rng.randint(n_lo, n_hi)
        cap = rng.randint(cap_lo, cap_hi)
        style = rng.random()
        if style < 0.3:
            ws = [rng.randint(1, max(1, 3 * cap // n)) for _ in range(n)]
        elif style < 0.6:
            ws = [rng.randint(1, max(1, cap // 2)) for _ in range(n)]
        elif style < 0.8:
            base = rng.randint(1, 64)
            ws = [base * rng.randint(1, 40) for _ in range(n)]  # many ties
        else:
            ws = [rng.randint(max(1, cap // (n + 1)), max(2, 2 * cap // (n + 1))) for _ in range(n)]
        out.append((ws, cap))
    return out


@pytest.mark.parametrize("seed,count,n_lo,n_hi,cap_lo,cap_hi", [
    (1, 6000, 1, 16, 1, 3000),              # tiny
    (2, 3000, 10, 60, 50_000, 400_000),     # fixture-sized windows (VGG/ResNet)
    (3, 600, 20, 80, 900_000, 1_800_000),   # GPT-2-sized windows, largest shared-memory rows
    (4, 120, 5, 40, 1_900_000, 9_000_000),  # global-memory row path, exact mode
    (5, 60, 2, 30, 10_000_001, 90_000_000),  # scaled mode
    (6, 40, 300, 600, 100_000, 300_000),    # 1 MB buckets: hundreds of items
])
def test_random_vs_oracle(seed, count, n_lo, n_hi, cap_lo, cap_hi):
    rng = random.Random(seed)
    probs = _random_problems(rng, count, n_lo, n_hi, cap_lo, cap_hi)
    solver = _native.subset_sum_solver()
    for s in range(0, len(probs), 256):
        batch = probs[s:s + 256]
        got = solver.solve(batch)
        want = O.subset_sum_c_batch(batch)
        assert got == want


def test_schedules_golden_on_gpu(golden_index, golden_inputs):
    from test_host_logic import product_stream
    for e in golden_index:
        text = product_stream(e, golden_inputs)
        assert hashlib.sha256(text.encode()).hexdigest() == e["sha256"], e["key"]
        assert text == golden_schedule_text(e)


def test_feedback_loop_golden_on_gpu(golden_index, golden_inputs):
    from test_host_logic import build_product_inputs
    walk = D.WalkParams.from_dict(golden_inputs["walk"])
    for e in golden_index:
        v = e.get("verdict")
        if v is None:
            continue
        prof, cluster, cfg, _, iters = build_product_inputs(e, golden_inputs)
        sched, got = D.feedback_loop(prof, cluster, cfg, walk, iterations=iters)
        text = "".join(l + "\n" for l in sched.jsonl_lines())
        assert hashlib.sha256(text.encode()).hexdigest() == v["final_sha256"], e["key"]
        assert (got.preserved, got.retries, got.ratio, list(got.sequence.k_values)) == \
            (v["preserved"], v["retries"], v["ratio"], v["k_values"])


@pytest.mark.parametrize("engine", ["kernel", "host"])
def test_schedule_engines_golden(golden_index, golden_inputs, engine):
    """K5 (one persistent kernel per schedule) and the host state machine over
    GPU knapsacks both reproduce every golden decision stream."""
    from test_host_logic import build_product_inputs
    from paper_2503_16815_b200 import gpu_scheduler
    used_kernel = 0
    for e in golden_index:
        prof, cluster, cfg, mult, iters = build_product_inputs(e, golden_inputs)
        if cfg is None:
            part, links = prof, cluster
        else:
            part = D.partition_buckets(prof, cfg)
            links = (D.ClusterSpec(links=(cluster.fast_link,))
                     if e["spec"].get("single_link") else cluster)
        if engine == "kernel":
            decisions = gpu_scheduler.run_schedules(part, links, [mult], iters)[0]
            if decisions is None:      # scaled mode: not covered by K5
                continue
            used_kernel += 1
        else:
            decisions = D.DeftScheduler(part, links, mult).run(iters)
        text = "".join(d.to_json() + "\n" for d in decisions)
        assert hashlib.sha256(text.encode()).hexdigest() == e["sha256"], e["key"]
    if engine == "kernel":
        assert used_kernel >= 50


def test_kernel_exec_notes_match_host(golden_index, golden_inputs):
    from test_host_logic import build_product_inputs
    from paper_2503_16815_b200 import gpu_scheduler
    for e in golden_index:
        prof, cluster, cfg, mult, iters = build_product_inputs(e, golden_inputs)
        part = D.partition_buckets(prof, cfg) if cfg is not None else prof
        got = gpu_scheduler.run_schedules(part, cluster, [mult], min(iters, 60))[0]
        if got is None:
            continue
        want = D.DeftScheduler(part, cluster, mult).run(min(iters, 60))
        for a, b in zip(got, want):
            assert a == b and a.exec == b.exec, (e["key"], a.iteration, a.stage)


def test_feedback_loop_kernel_engine(golden_index, golden_inputs):
    from test_host_logic import build_product_inputs
    walk = D.WalkParams.from_dict(golden_inputs["walk"])
    for e in golden_index:
        v = e.get("verdict")
        if v is None:
            continue
        prof, cluster, cfg, _, iters = build_product_inputs(e, golden_inputs)
        for engine in ("kernel", "host"):
            sched, got = D.feedback_loop(prof, cluster, cfg, walk, iterations=iters,
                                         engine=engine)
            text = "".join(l + "\n" for l in sched.jsonl_lines())
            assert hashlib.sha256(text.encode()).hexdigest() == v["final_sha256"], e["key"]
            assert (got.preserved, got.retries, got.ratio) == \
                (v["preserved"], v["retries"], v["ratio"])


@pytest.mark.parametrize("chunk", [1, 7, 64])
def test_kernel_scheduler_chunks_match_host(golden_index, golden_inputs, chunk):
    """K5 in chunks with carried state == the host state machine, across chunk
    boundaries that fall inside merged groups."""
    from test_host_logic import build_product_inputs
    from paper_2503_16815_b200.gpu_scheduler import KernelScheduler
    keys = ("uniform48__equal_dual__raw", "uniform36__equal_dual__raw__m1",
            "vgg19__dual__bw0.25", "gpt2__fast__bw0.25", "resnet101__fast__bw0.25",
            "measured_vgg19_w4__x200")
    n = 0
    for e in golden_index:
        if e["key"] not in keys:
            continue
        prof, cluster, cfg, mult, _ = build_product_inputs(e, golden_inputs)
        part = D.partition_buckets(prof, cfg) if cfg is not None else prof
        if not KernelScheduler.supported(part, cluster, mult):
            continue
        iters = 70
        got = KernelScheduler(part, cluster, mult, chunk=chunk).run(iters)
        want = D.DeftScheduler(part, cluster, mult).run(iters)
        for a, b in zip(got, want):
            assert a == b and a.exec == b.exec, (e["key"], chunk, a.iteration, a.stage)
        n += 1
    assert n >= 5
