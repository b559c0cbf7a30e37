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
