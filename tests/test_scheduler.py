"""NEXT-4: the DP batch scheduler (§5, Algorithm 2, Eq. 2) in libtt.so,
against an exhaustive-partition oracle and the paper's five-request example.
Host code only: runs on CPU."""
import itertools

import numpy as np
import pytest

import oracle


def _table(max_len, max_batch, fn):
    c = np.full((max_len + 1, max_batch + 1), np.nan)
    for L in range(1, max_len + 1):
        for k in range(1, max_batch + 1):
            c[L, k] = fn(L, k)
    return c


def _gpu_like(L, k):
    # per-request cost of a batch of k padded to L: a fixed launch/latency part
    # amortised over the batch, plus work proportional to the padded length
    return 30.0 / k + 0.05 * L + 0.0004 * L * L


def test_paper_five_request_example(ttlib):
    """Lengths 17, 18, 52, 63, 77 (fig:batch-example): with
    a strong padding penalty, three batches beat one batch and no batching."""
    lens = [17, 18, 52, 63, 77]
    cost = _table(80, 5, lambda L, k: 4.0 / k + 0.02 * L * L / 10)
    plans, total = ttlib.dp_schedule(lens, cost)
    assert [sorted(lens[i] for i in b) for b in plans] == [[17, 18], [52, 63], [77]]
    one = oracle.plan_cost(lens, cost, [list(range(5))])
    none = oracle.plan_cost(lens, cost, [[i] for i in range(5)])
    assert total < one and total < none
    bf, _ = oracle.schedule_bruteforce(lens, cost, 5)
    assert abs(total - bf) < 1e-9


@pytest.mark.parametrize("seed", range(25))
def test_dp_equals_exhaustive_minimum(ttlib, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    n = int(rng.integers(1, 12))
    max_batch = int(rng.integers(1, n + 1))
    lens = rng.integers(1, 60, size=n).tolist()
    cost = _table(60, max_batch, lambda L, k: float(rng.uniform(0.5, 2.0)) * _gpu_like(L, k))
    plans, total = ttlib.dp_schedule(lens, cost)
    bf, _ = oracle.schedule_bruteforce(lens, cost, max_batch)
    assert abs(total - bf) <= 1e-9 * max(1.0, bf)
    # the returned plan is valid and its own cost is the reported optimum
    assert sorted(i for b in plans for i in b) == list(range(n))
    assert all(1 <= len(b) <= max_batch for b in plans)
    assert abs(oracle.plan_cost(lens, cost, plans) - total) <= 1e-9 * max(1.0, total)
    assert abs(ttlib.schedule_cost(lens, cost, plans) - total) <= 1e-9 * max(1.0, total)
    # batches are contiguous runs of the length-sorted order
    pad = [max(lens[i] for i in b) for b in plans]
    assert pad == sorted(pad)
    for b, nxt in zip(plans, plans[1:]):
        assert max(lens[i] for i in b) <= min(lens[i] for i in nxt)


def test_dominates_naive_and_no_batching(ttlib):
    rng = np.random.Generator(np.random.PCG64(7))
    for _ in range(20):
        n = int(rng.integers(1, 40))
        lens = rng.integers(1, 200, size=n).tolist()
        cost = _table(200, n, _gpu_like)
        plans, total = ttlib.dp_schedule(lens, cost)
        assert total <= ttlib.schedule_cost(lens, cost, [list(range(n))]) + 1e-9
        assert total <= ttlib.schedule_cost(lens, cost, [[i] for i in range(n)]) + 1e-9


def test_equal_lengths_keep_queue_order_and_determinism(ttlib):
    lens = [5, 3, 5, 3, 5]
    cost = _table(5, 5, lambda L, k: 1.0)
    a = ttlib.dp_schedule(lens, cost)
    b = ttlib.dp_schedule(lens, cost)
    assert a == b
    flat = [i for bt in a[0] for i in bt]
    assert flat == [1, 3, 0, 2, 4]   # stable sort: FIFO within a length class


def test_single_request_and_empty(ttlib):
    cost = _table(10, 4, _gpu_like)
    plans, total = ttlib.dp_schedule([7], cost)
    assert plans == [[0]] and abs(total - cost[7, 1]) < 1e-12
    assert ttlib.dp_schedule([], cost) == ([], 0.0)


def test_invalid_inputs_are_rejected(ttlib):
    cost = _table(10, 4, _gpu_like)
    with pytest.raises(ttlib.TTError):
        ttlib.dp_schedule([11], cost)             # length beyond the table
    with pytest.raises(ttlib.TTError):
        ttlib.dp_schedule([0, 3], cost)           # length < 1
    bad = cost.copy()
    bad[5, 2] = np.nan
    with pytest.raises(ttlib.TTError):
        ttlib.dp_schedule([5, 5, 5], bad)         # the recursion reads a missing entry
    with pytest.raises(ttlib.TTError):
        ttlib.schedule_cost([1, 2], cost, [[0, 0]])   # request twice
    with pytest.raises(ttlib.TTError):
        ttlib.schedule_cost([1, 2, 3, 4, 5], cost, [[0, 1, 2, 3, 4]])  # batch > max_batch


def test_max_batch_is_respected(ttlib):
    lens = [10] * 9
    cost = _table(10, 4, lambda L, k: 10.0 / k)   # bigger batches always cheaper
    plans, _ = ttlib.dp_schedule(lens, cost)
    assert all(len(b) <= 4 for b in plans) and sum(len(b) for b in plans) == 9


def test_oracle_bruteforce_itself_on_a_hand_case():
    """Pin for the oracle: two requests, batching cost 1.5 per request vs 1
    alone -> no batching; vs 0.4 -> one batch."""
    lens = [2, 2]
    c1 = _table(2, 2, lambda L, k: 1.0 if k == 1 else 1.5)
    c2 = _table(2, 2, lambda L, k: 1.0 if k == 1 else 0.4)
    assert oracle.schedule_bruteforce(lens, c1, 2) == (2.0, [[0], [1]])
    assert oracle.schedule_bruteforce(lens, c2, 2) == (0.8, [[0, 1]])
    assert len(list(itertools.product([0, 1], repeat=3))) == 8


# ---- set-partition oracle (independent of Alg. 2's contiguity premise) ----
def test_set_partitions_count_is_bell():
    """Pin: the enumerator yields each partition of {0..n-1} once; the counts
    are the Bell numbers 1, 1, 2, 5, 15, 52, 203, 877, 4140 (OEIS A000110)."""
    bell = [1, 1, 2, 5, 15, 52, 203, 877, 4140]
    for n, b in enumerate(bell):
        parts = list(oracle.set_partitions(n))
        assert len(parts) == b
        canon = {tuple(sorted(tuple(sorted(blk)) for blk in p)) for p in parts}
        assert len(canon) == b
        for p in parts:
            assert sorted(i for blk in p for i in blk) == list(range(n))
            assert all(blk for blk in p)


def test_setpartition_oracle_hand_cases():
    """Pins by hand: (i) lengths 1, 9, 1 with a cost linear in the padded
    length: batching the two 1s together (and 9 alone) is optimal, a plan that
    is non-contiguous in queue order; (ii) a non-monotone table (padding to 2
    is cheaper than to 1) makes a non-contiguous batch strictly better than any
    contiguous run of the sorted list, so the two oracles differ."""
    lens = [1, 9, 1]
    c = _table(9, 3, lambda L, k: float(L) + 3.0 / k)
    best, plan = oracle.schedule_setpartition_bruteforce(lens, c, 3)
    assert sorted(sorted(b) for b in plan) == [[0, 2], [1]]
    assert best == 2 * (1 + 1.5) + (9 + 3)
    # (ii) sorted order 1, 2, 3; cost per request: L=1 -> 5, L=2 -> 1, L=3 -> 4 (any k)
    lens = [1, 2, 3]
    c = _table(3, 3, lambda L, k: {1: 5.0, 2: 1.0, 3: 4.0}[L])
    sp, plan = oracle.schedule_setpartition_bruteforce(lens, c, 2)
    assert sp == 2 * 1.0 + 4.0 and sorted(sorted(b) for b in plan) == [[0, 1], [2]]
    ct, _ = oracle.schedule_bruteforce(lens, c, 2)
    assert ct == sp                                # {1,2} is also a sorted run here
    lens = [1, 3, 2]                               # same multiset, other queue order
    assert oracle.schedule_setpartition_bruteforce(lens, c, 2)[0] == 6.0
    # (iii) a table where padding to 2 is cheaper than to 1 alone (non-monotone):
    # the optimum batches the shortest with the longest request, {1, 3}, which is
    # not a contiguous run of the sorted list, so Alg. 2's search space misses it
    lens = [1, 2, 3]
    tab = {(1, 1): 5.0, (2, 1): 1.0, (3, 1): 10.0, (1, 2): 9.0, (2, 2): 10.0, (3, 2): 1.0}
    c = _table(3, 2, lambda L, k: tab[(L, k)])
    sp, plan = oracle.schedule_setpartition_bruteforce(lens, c, 2)
    ct, _ = oracle.schedule_bruteforce(lens, c, 2)
    assert sorted(sorted(b) for b in plan) == [[0, 2], [1]] and sp == 2 * 1.0 + 1.0
    assert ct == 2 * 1.0 + 5.0 and sp < ct


def _monotone_table(rng, max_len, max_batch):
    """cached_cost[L][k] nondecreasing in L for every k (positive increments)."""
    c = np.full((max_len + 1, max_batch + 1), np.nan)
    for k in range(1, max_batch + 1):
        base = float(rng.uniform(0.1, 5.0))
        inc = rng.uniform(0.0, 1.0, size=max_len) * (rng.uniform(size=max_len) < 0.6)
        c[1:, k] = base + np.cumsum(inc)
    return c


@pytest.mark.parametrize("seed", range(30))
def test_dp_equals_setpartition_minimum_when_cost_monotone_in_length(ttlib, seed):
    """When cached_cost is nondecreasing in the padded length, restricting the
    search to contiguous runs of the sorted list (Alg. 2's premise, PAPER.md
    l.619-648) loses nothing: re-assigning any partition's batch sizes to the
    sorted list in order never raises a batch's max length.  So the DP optimum
    must equal the minimum over ALL set partitions."""
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    n = int(rng.integers(1, 10))
    max_batch = int(rng.integers(1, n + 1))
    lens = rng.integers(1, 30, size=n).tolist()
    cost = _monotone_table(rng, 30, max_batch)
    plans, total = ttlib.dp_schedule(lens, cost)
    sp, _ = oracle.schedule_setpartition_bruteforce(lens, cost, max_batch)
    assert abs(total - sp) <= 1e-9 * max(1.0, sp)


def test_setpartition_never_above_contiguous():
    rng = np.random.Generator(np.random.PCG64(77))
    for _ in range(20):
        n = int(rng.integers(1, 8))
        mb = int(rng.integers(1, n + 1))
        lens = rng.integers(1, 20, size=n).tolist()
        cost = _table(20, mb, lambda L, k: float(rng.uniform(0.1, 3.0)))
        sp, _ = oracle.schedule_setpartition_bruteforce(lens, cost, mb)
        ct, _ = oracle.schedule_bruteforce(lens, cost, mb)
        assert sp <= ct + 1e-12
