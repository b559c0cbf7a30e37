"""Seeded synthetic workloads shared by the tests and bench.py.

This module holds NO arithmetic of the method (no softmax, no LayerNorm): only
shapes, seeds, value distributions and the algorithmic-byte counts used for
reporting.  Both sides of every parity check (the CUDA path and ``oracle/``)
consume the same tensors generated here; neither side imports the other.

Configurations follow BASELINE.json ``configs`` in order:

* C1  BERT-base b=1 s=40, heads 12, hidden 768, fp32
* C2  BERT-base b=20, seq sweep 10..500, fp16/fp32
* C3  64 requests, lengths U{5..500}
* C4  BERT-large heads 16, hidden 1024, b=64 s=512, bf16        (long-row, bandwidth-bound)
* C5  4096 requests U{5..500} in 64 batches of 64, sharded over GPUs

Value recipe: raw attention logits q.k with d_head = 64 and unit
entries have std 8, hence x ~ N(0, 8^2) and scale = 1/sqrt(64) = 0.125 (exact in
binary).  LayerNorm activations x, residual ~ N(0, 1); bias, beta ~ U(-0.1, 0.1);
gamma ~ 1 + U(-0.1, 0.1); eps = 1e-12 (BERT's value).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

SEED = 201005680
SCALE_BERT = 0.125
EPS_BERT = 1e-12
LOGIT_STD = 8.0

ELEM_BYTES = {torch.float32: 4, torch.float16: 2, torch.bfloat16: 2}
DTYPES = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}
DTYPE_NAMES = {v: k for k, v in DTYPES.items()}


@dataclass(frozen=True)
class Config:
    name: str
    heads: int
    hidden: int
    dtypes: tuple
    description: str
    seed_offset: int
    extra: dict = field(default_factory=dict)


C1 = Config("C1", 12, 768, ("f32",), "BERT-base batch=1 seq=40 fp32", 1, {"batch": 1, "seq": 40})
C2 = Config("C2", 12, 768, ("f16", "f32"), "BERT-base batch=20 seq sweep 10-500", 2,
            {"batch": 20, "seqs": (10, 20, 37, 40, 64, 100, 128, 200, 256, 300, 400, 500)})
C3 = Config("C3", 12, 768, ("f16", "f32"), "64 requests, lengths U{5..500}", 3,
            {"batch": 64, "lo": 5, "hi": 500})
C4 = Config("C4", 16, 1024, ("bf16",), "BERT-large batch=64 seq=512 bf16", 4,
            {"batch": 64, "seq": 512})
C5 = Config("C5", 12, 768, ("f16", "bf16"), "4096-request stream U{5..500}, 64 batches of 64", 5,
            {"requests": 4096, "per_batch": 64, "lo": 5, "hi": 500})
CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}


def rng(seed_offset: int, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED + seed_offset + 1000003 * salt))


# ----------------------------------------------------------------------------- lengths
def lengths_full(batch: int, seq: int) -> np.ndarray:
    return np.full(batch, seq, dtype=np.int32)


def lengths_ragged(batch: int, seq: int, seed_offset: int = 2, salt: int = 0) -> np.ndarray:
    """C2 ragged variant: lengths[0] = S (so Smax = S), the rest U{1..S}."""
    g = rng(seed_offset, salt + seq)
    lens = g.integers(1, seq, size=batch, endpoint=True).astype(np.int32)
    if batch:
        lens[0] = seq
    return lens


def lengths_uniform(n: int, lo: int, hi: int, seed_offset: int, salt: int = 0) -> np.ndarray:
    """n request lengths drawn uniformly from {lo..hi}."""
    return rng(seed_offset, salt).integers(lo, hi, size=n, endpoint=True).astype(np.int32)


def c3_lengths(salt: int = 0) -> np.ndarray:
    return lengths_uniform(C3.extra["batch"], C3.extra["lo"], C3.extra["hi"], C3.seed_offset, salt)


def c5_stream() -> list:
    """The C5 request stream in arrival order, cut into 64 batches of 64
    consecutive requests; each batch is padded to its own Smax (batch
    scheduling is out of scope)."""
    lens = lengths_uniform(C5.extra["requests"], C5.extra["lo"], C5.extra["hi"], C5.seed_offset)
    pb = C5.extra["per_batch"]
    return [lens[i:i + pb].copy() for i in range(0, len(lens), pb)]


# ----------------------------------------------------------------------------- tensors
def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def scores(B: int, H: int, Sq: int, Sk: int, dtype, device="cpu", seed: int = SEED,
           std: float = LOGIT_STD) -> torch.Tensor:
    """Attention logits [B,H,Sq,Sk] ~ N(0, std^2), stored in `dtype`."""
    g = _gen(device, seed)
    t = torch.randn((B, H, Sq, Sk), generator=g, device=device, dtype=torch.float32)
    t.mul_(std)
    return t.to(dtype)


def poison_masked(scores_t: torch.Tensor, lengths) -> torch.Tensor:
    """Fill padded key columns with NaN / +Inf / -Inf (cycling) -- the masked
    bytes must never influence a valid output (DESIGN R1)."""
    lens = torch.as_tensor(np.asarray(lengths), dtype=torch.int64)
    B, H, Sq, Sk = scores_t.shape
    cols = torch.arange(Sk)
    mask = cols[None, :] >= lens.clamp(0, Sk)[:, None]           # [B, Sk]
    poison = torch.tensor([float("nan"), float("inf"), float("-inf")])[cols % 3]
    full = poison.to(scores_t.dtype).to(scores_t.device)
    m = mask[:, None, None, :].to(scores_t.device).expand(B, H, Sq, Sk)
    return torch.where(m, full.expand(B, H, Sq, Sk), scores_t)


def ln_inputs(rows: int, hidden: int, dtype, device="cpu", seed: int = SEED,
              offset: float = 0.0) -> dict:
    """x, residual ~ N(0,1) (+offset on x); bias, beta ~ U(-.1,.1); gamma ~ 1+U(-.1,.1)."""
    g = _gen(device, seed)
    f = dict(device=device, dtype=torch.float32)
    x = torch.randn((rows, hidden), generator=g, **f)
    if offset:
        x.add_(offset)
    res = torch.randn((rows, hidden), generator=g, **f)
    bias = (torch.rand((hidden,), generator=g, **f) - 0.5) * 0.2
    gamma = 1.0 + (torch.rand((hidden,), generator=g, **f) - 0.5) * 0.2
    beta = (torch.rand((hidden,), generator=g, **f) - 0.5) * 0.2
    return {k: v.to(dtype) for k, v in
            dict(x=x, residual=res, bias=bias, gamma=gamma, beta=beta).items()}


# ----------------------------------------------------------------------------- accounting
def softmax_bytes_alg(lengths, H: int, Sq: int, Sk: int, elem_bytes: int) -> int:
    """sum over rows of (L_b*e read + Sk*e write) + 4*B (lengths)."""
    lens = np.clip(np.asarray(lengths, dtype=np.int64), 0, Sk)
    B = len(lens)
    return int(H * Sq * (int(lens.sum()) * elem_bytes + B * Sk * elem_bytes) + 4 * B)


def ln_bytes_alg(rows: int, hidden: int, elem_bytes: int) -> int:
    """x + residual read, out written, + bias/gamma/beta once."""
    return int(3 * rows * hidden * elem_bytes + 3 * hidden * elem_bytes)
