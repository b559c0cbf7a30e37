"""Host-side multi-GPU logic on CPU: batch partitioning, per-rank records and
their gather over torch.distributed (gloo, world size 2).

The data path has no collective; what must hold is that every
batch is processed exactly once, the work is balanced, and the gathered
per-rank records reproduce the single-rank digests bit for bit (sharding
invariance).  The per-batch "compute" here is the oracle on tiny shapes (the
GPU path is exercised by the gpu tests and bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_2010_05680_b200 import sharding


def test_lpt_partition_covers_each_batch_once_and_balances():
    costs = [int(c) for c in np.random.Generator(np.random.PCG64(1)).integers(1, 1000, 64)]
    for world in (1, 2, 3, 4, 8):
        parts = sharding.lpt_partition(costs, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(64))
        loads = [sum(costs[i] for i in p) for p in parts]
        # LPT bound: max load <= mean + max job
        assert max(loads) <= sum(costs) / world + max(costs)
        assert parts == sharding.lpt_partition(costs, world)  # deterministic


def test_lpt_ties_go_to_lower_rank_and_lower_index():
    parts = sharding.lpt_partition([5, 5, 5, 5], 2)
    assert parts == [[0, 2], [1, 3]]
    with pytest.raises(ValueError):
        sharding.lpt_partition([1], 0)


def test_contiguous_ranges():
    for n, w in ((10, 3), (0, 4), (7, 7), (5, 8)):
        rs = sharding.contiguous_ranges(n, w)
        assert len(rs) == w and rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_c5_stream_partition_by_bytes():
    batches = W.c5_stream()
    assert len(batches) == 64 and all(len(b) == 64 for b in batches)
    costs = [W.softmax_bytes_alg(b, 12, int(b.max()), int(b.max()), 2) +
             W.ln_bytes_alg(64 * int(b.max()), 768, 2) for b in batches]
    parts = sharding.lpt_partition(costs, 8)
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) / (sum(loads) / 8) < 1.1   # near-linear scaling is possible


def test_record_roundtrip_and_digest():
    d = (1 << 63) + 12345
    rec = sharding.make_record(d, 3.5, 1000, 10, 12.5, 2, 1)
    assert rec.numel() * rec.element_size() == 64
    assert sharding.record_digest(rec.tolist()) == d
    t = torch.arange(10, dtype=torch.float16)
    assert sharding.tensor_digest(t) == sharding.tensor_digest(t.clone())
    assert sharding.tensor_digest(t) != sharding.tensor_digest(t + 1)
    assert sharding.combine_digests([1, 2]) != sharding.combine_digests([2, 1])


def _tiny_batches():
    # 6 tiny variable-length batches (same recipe as C5, smaller)
    lens = W.lengths_uniform(24, 1, 9, seed_offset=5, salt=7)
    return [lens[i:i + 4] for i in range(0, 24, 4)]


def _batch_digest(bi, lens):
    S = int(lens.max())
    x = W.scores(len(lens), 2, S, S, torch.float16, seed=W.SEED + bi)
    y = oracle.softmax_masked(x, lens, W.SCALE_BERT).to(torch.float16)
    return sharding.tensor_digest(y), float(y.double().sum())


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batches = _tiny_batches()
        costs = [W.softmax_bytes_alg(b, 2, int(b.max()), int(b.max()), 2) for b in batches]
        mine = sharding.lpt_partition(costs, world)[rank]
        digests, checksum = {}, 0.0
        for bi in mine:
            d, c = _batch_digest(bi, batches[bi])
            digests[bi] = d
            checksum += c
        rec = sharding.make_record(sharding.combine_digests([digests[i] for i in mine]),
                                   checksum, sum(costs[i] for i in mine), len(mine), 10.0 + rank,
                                   len(mine), rank)
        recs = sharding.gather_records(rec)
        t = sharding.max_over_ranks(10.0 + rank, torch.device("cpu"))
        if rank == 0:
            q.put((recs.tolist(), t, {k: v for k, v in digests.items()}))
        else:
            q.put((None, t, {k: v for k, v in digests.items()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_records_match_single_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    recs = next(o[0] for o in outs if o[0] is not None)
    assert all(o[1] == 11.0 for o in outs)          # max over ranks
    per_batch = {}
    for o in outs:
        per_batch.update(o[2])
    batches = _tiny_batches()
    assert sorted(per_batch) == list(range(len(batches)))   # each batch exactly once
    # sharding invariance: every batch digest equals the single-rank computation
    for bi, lens in enumerate(batches):
        assert per_batch[bi] == _batch_digest(bi, lens)[0]
    # gathered records: ranks in order, all work accounted for
    assert [int(r[7]) for r in recs] == [0, 1]
    costs = [W.softmax_bytes_alg(b, 2, int(b.max()), int(b.max()), 2) for b in batches]
    assert sum(r[3] for r in recs) == sum(costs)
    assert sum(int(r[6]) for r in recs) == len(batches)

