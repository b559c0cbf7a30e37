"""Request-batch sharding across the GPUs of one node.

Rows and requests are independent and neither operation reduces across rows,
so the multi-GPU path has no data-path collective: every rank derives the same
batch list from the seed, takes its share, and runs the kernels on its own
GPU.  NCCL (torch.distributed) carries only per-rank records (checksums,
byte counts, timings) and the timing barriers.
"""
from __future__ import annotations

import hashlib
import struct
from typing import Sequence

import torch


def lpt_partition(costs: Sequence[int], world: int) -> list:
    """Greedy longest-processing-time bin packing of batch costs onto `world`
    ranks.  Deterministic: ties in cost keep the lower batch index first, ties
    in load go to the lower rank.  Returns, per rank, its batch indices in
    ascending order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-int(costs[i]), i))
    load = [0] * world
    parts = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        parts[r].append(i)
        load[r] += int(costs[i])
    return [sorted(p) for p in parts]


def contiguous_ranges(nrows: int, world: int) -> list:
    """Split [0, nrows) into `world` contiguous row ranges, sizes differing by <= 1."""
    base, extra = divmod(nrows, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((start, start + n))
        start += n
    return out


RECORD_FIELDS = ("digest_lo", "digest_hi", "checksum", "bytes_alg", "rows", "elapsed_us",
                 "batches", "rank")


def tensor_digest(t: torch.Tensor) -> int:
    """64-bit digest of a tensor's bytes (blake2b over the host copy)."""
    b = t.detach().contiguous().view(torch.uint8).cpu().numpy().tobytes()
    return int.from_bytes(hashlib.blake2b(b, digest_size=8).digest(), "little")


_M64 = (1 << 64) - 1
_K1 = 0x9E3779B97F4A7C15 - (1 << 64)   # as signed int64
_K2 = 0xBF58476D1CE4E5B9 - (1 << 64)


def device_digest(t: torch.Tensor, chunk: int = 1 << 24) -> int:
    """64-bit positional digest of a tensor's bytes computed where the tensor
    lives (no host copy of multi-GB outputs): sum over 32-bit words w_i of
    mix(w_i, i) modulo 2^64.  Integer addition modulo 2^64 is associative and
    commutative, so the value does not depend on the reduction order -- the
    same bytes give the same digest on any device and at any world size."""
    b = t.detach().contiguous().view(-1).view(torch.uint8)
    if b.numel() % 4:
        b = torch.cat([b, b.new_zeros(4 - b.numel() % 4)])
    w = b.view(torch.int32)
    acc = 0
    for off in range(0, w.numel(), chunk):
        v = w[off:off + chunk].to(torch.int64) & 0xFFFFFFFF
        idx = torch.arange(off, off + v.numel(), device=v.device, dtype=torch.int64)
        h = (v ^ (idx * _K1)) * _K2
        h = h ^ (h >> 31)
        acc = (acc + int(h.sum().item())) & _M64
    return acc ^ (t.numel() * 0x100000001B3 & _M64)


def gather_objects(obj, group=None) -> list:
    """all_gather_object over the default group (nccl or gloo)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def stream_digest(batch_digests: dict) -> int:
    """Digest of a whole request stream from {batch_id: digest}: independent
    of which rank processed which batch (sharding invariance)."""
    return combine_digests([batch_digests[k] for k in sorted(batch_digests)])


def combine_digests(digests: Sequence[int]) -> int:
    h = hashlib.blake2b(digest_size=8)
    for d in digests:
        h.update(struct.pack("<Q", d & 0xFFFFFFFFFFFFFFFF))
    return int.from_bytes(h.digest(), "little")


def make_record(digest: int, checksum: float, bytes_alg: int, rows: int, elapsed_us: float,
                batches: int, rank: int) -> torch.Tensor:
    """Fixed 64-byte per-rank record (8 float64 slots; the 64-bit digest is
    split into two exact 32-bit halves)."""
    return torch.tensor([float(digest & 0xFFFFFFFF), float(digest >> 32), float(checksum),
                         float(bytes_alg), float(rows), float(elapsed_us), float(batches),
                         float(rank)], dtype=torch.float64)


def record_digest(rec) -> int:
    return int(rec[0]) | (int(rec[1]) << 32)


def gather_records(rec: torch.Tensor, group=None) -> torch.Tensor:
    """all_gather of the 64-byte records -> [world, 8] on every rank."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty((world, rec.numel()), dtype=rec.dtype, device=rec.device)
    dist.all_gather_into_tensor(out, rec.reshape(1, -1).contiguous(), group=group)
    return out


def max_over_ranks(value: float, device) -> float:
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
