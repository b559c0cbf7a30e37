"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A plain double-precision C implementation (``oracle/oracle.c``) of the two
batch-reduction operations of TurboTransformers (arXiv 2010.05680, PAPER.md
§4.1.2 l.313-317, Eq. 1 l.406-409, kernel names l.765), loaded with ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2010_05680_b200/`` and imports nothing from it.

Parity: every function here is pinned by ``tests/test_oracle_pins.py``
(closed forms, invariants, exhaustive decoder checks, brute force against
mpmath, independent library routines); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

DTYPE_CODE = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no fast-math) into liboracle.so."""
    stale = (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)
    if force or stale:
        tmp = _LIB_PATH + f".{os.getpid()}.tmp"
        subprocess.check_call(
            ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c11", "-fPIC",
             "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.tto_widen.argtypes = [_vp, ctypes.c_int, _i64, _vp]
            lib.tto_softmax_masked.argtypes = [_vp, ctypes.c_int, _vp, _i64, _i64, _i64, _i64,
                                               ctypes.c_float, _vp]
            lib.tto_add_bias_layernorm.argtypes = [_vp, _vp, _vp, _vp, _vp, ctypes.c_int, _i64,
                                                   _i64, ctypes.c_float, _vp]
            lib.tto_layernorm_onepass_eq1.argtypes = [_vp, _vp, _vp, ctypes.c_int, _i64, _i64,
                                                      ctypes.c_float, _vp]
            lib.tto_add_bias_gelu.argtypes = [_vp, _vp, ctypes.c_int, _i64, _i64, ctypes.c_int,
                                              _vp]
            lib.tto_split_qkv_add_bias.argtypes = [_vp, _vp, ctypes.c_int, _i64, _i64, _i64,
                                                   _i64, _vp]
            lib.tto_merge_heads.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _i64, _vp]
            lib.tto_attention.argtypes = [_vp, _vp, _vp, ctypes.c_int, _vp, _i64, _i64, _i64,
                                          _i64, ctypes.c_float, _vp]
            for f in (lib.tto_widen, lib.tto_softmax_masked, lib.tto_add_bias_layernorm,
                      lib.tto_layernorm_onepass_eq1, lib.tto_add_bias_gelu,
                      lib.tto_split_qkv_add_bias, lib.tto_merge_heads, lib.tto_attention):
                f.restype = ctypes.c_int
            _lib = lib
    return _lib


def _host(t: torch.Tensor) -> torch.Tensor:
    if t.dtype not in DTYPE_CODE:
        raise TypeError(f"oracle: unsupported dtype {t.dtype}")
    return t.detach().to("cpu").contiguous()


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def widen(t: torch.Tensor) -> torch.Tensor:
    """Exact storage-dtype -> float64 widening by the oracle's own bit decoders."""
    src = _host(t)
    out = torch.empty(src.shape, dtype=torch.float64)
    rc = _load().tto_widen(_ptr(src), DTYPE_CODE[src.dtype], src.numel(), _ptr(out))
    assert rc == 0
    return out


def softmax_masked(scores: torch.Tensor, lengths, scale: float) -> torch.Tensor:
    """Masked softmax over the last dim of [B,H,Sq,Sk]; returns float64.

    Key columns j >= clamp(lengths[b], 0, Sk) are +0.0 (DESIGN R1-R3)."""
    if scores.dim() != 4:
        raise ValueError("scores must be [B,H,Sq,Sk]")
    src = _host(scores)
    B, H, Sq, Sk = src.shape
    lens = torch.as_tensor(np.asarray(lengths, dtype=np.int32) if not torch.is_tensor(lengths)
                           else lengths.detach().to("cpu", torch.int32)).contiguous()
    if lens.numel() != B:
        raise ValueError("lengths must have B entries")
    out = torch.empty((B, H, Sq, Sk), dtype=torch.float64)
    rc = _load().tto_softmax_masked(_ptr(src), DTYPE_CODE[src.dtype], _ptr(lens), B, H, Sq, Sk,
                                    ctypes.c_float(scale), _ptr(out))
    assert rc == 0
    return out


def softmax_rows(rows: torch.Tensor, row_lengths, scale: float) -> torch.Tensor:
    """Masked softmax of R independent rows [R, Sk], each with its own valid
    length (B=R, H=Sq=1).  Used to check sampled rows of full-size runs."""
    R, Sk = rows.shape
    return softmax_masked(rows.reshape(R, 1, 1, Sk), row_lengths, scale).reshape(R, Sk)


def add_bias_layernorm(x, residual, bias, gamma, beta, eps: float) -> torch.Tensor:
    """LayerNorm((x + bias) + residual) * gamma + beta over the last dim; float64."""
    xs, rs, bs, gs, be = (_host(t) for t in (x, residual, bias, gamma, beta))
    if not (xs.dtype == rs.dtype == bs.dtype == gs.dtype == be.dtype):
        raise TypeError("all LayerNorm operands share one dtype (DESIGN R11)")
    hidden = xs.shape[-1]
    rows = xs.numel() // hidden if hidden else 0
    if rs.shape != xs.shape or bs.numel() != hidden or gs.numel() != hidden or be.numel() != hidden:
        raise ValueError("shape mismatch")
    out = torch.empty(xs.shape, dtype=torch.float64)
    rc = _load().tto_add_bias_layernorm(_ptr(xs), _ptr(rs), _ptr(bs), _ptr(gs), _ptr(be),
                                        DTYPE_CODE[xs.dtype], rows, hidden, ctypes.c_float(eps),
                                        _ptr(out))
    assert rc == 0
    return out


def layernorm_onepass_eq1(x, gamma, beta, eps: float) -> torch.Tensor:
    """The paper's one-pass variance form (Eq. 1 RHS), plain LN, float64."""
    xs, gs, be = (_host(t) for t in (x, gamma, beta))
    hidden = xs.shape[-1]
    rows = xs.numel() // hidden if hidden else 0
    out = torch.empty(xs.shape, dtype=torch.float64)
    rc = _load().tto_layernorm_onepass_eq1(_ptr(xs), _ptr(gs), _ptr(be), DTYPE_CODE[xs.dtype],
                                           rows, hidden, ctypes.c_float(eps), _ptr(out))
    assert rc == 0
    return out


def softmax_packed(flat: torch.Tensor, lengths, H: int, scale: float) -> torch.Tensor:
    """Packed (padding-free) softmax: request r is a dense [H, L_r, L_r] block,
    blocks concatenated in request order; each block is the masked softmax with
    every key valid.  Returns float64 of flat's shape."""
    src = _host(flat).reshape(-1)
    lens = [int(v) for v in np.asarray(lengths).reshape(-1)]
    if sum(H * L * L for L in lens) != src.numel():
        raise ValueError("flat size does not match the lengths")
    out = torch.empty(src.shape, dtype=torch.float64)
    off = 0
    for L in lens:
        n = H * L * L
        if n:
            out[off:off + n] = softmax_masked(src[off:off + n].reshape(1, H, L, L), [L],
                                              scale).reshape(-1)
        off += n
    if off != src.numel():
        raise ValueError("flat size does not match the lengths")
    return out


# ---------------------------------------------------------------- NEXT-2 ops
def add_bias_gelu(x, bias, approximate: bool = False) -> torch.Tensor:
    """gelu(x + bias) over the last dim, float64 (exact erf form, or tanh form)."""
    xs, bs = _host(x), _host(bias)
    if xs.dtype != bs.dtype:
        raise TypeError("x and bias share one dtype")
    n = xs.shape[-1]
    rows = xs.numel() // n if n else 0
    if bs.numel() != n:
        raise ValueError("bias must have n elements")
    out = torch.empty(xs.shape, dtype=torch.float64)
    rc = _load().tto_add_bias_gelu(_ptr(xs), _ptr(bs), DTYPE_CODE[xs.dtype], rows, n,
                                   int(bool(approximate)), _ptr(out))
    assert rc == 0
    return out


def split_qkv_add_bias(qkv, bias, B: int, S: int, H: int, D: int):
    """qkv [B*S, 3*H*D] + bias [3*H*D] -> (q, k, v), each float64 [B, H, S, D]."""
    qs, bs = _host(qkv), _host(bias)
    if qs.numel() != B * S * 3 * H * D or bs.numel() != 3 * H * D:
        raise ValueError("shape mismatch")
    out = torch.empty((3, B, H, S, D), dtype=torch.float64)
    rc = _load().tto_split_qkv_add_bias(_ptr(qs), _ptr(bs), DTYPE_CODE[qs.dtype], B, S, H, D,
                                        _ptr(out))
    assert rc == 0
    return out[0], out[1], out[2]


def merge_heads(x, B: int, S: int, H: int, D: int) -> torch.Tensor:
    """[B, H, S, D] -> [B*S, H*D] float64 (exact)."""
    xs = _host(x)
    if xs.numel() != B * H * S * D:
        raise ValueError("shape mismatch")
    out = torch.empty((B * S, H * D), dtype=torch.float64)
    rc = _load().tto_merge_heads(_ptr(xs), DTYPE_CODE[xs.dtype], B, S, H, D, _ptr(out))
    assert rc == 0
    return out


def attention(q, k, v, lengths, scale: float) -> torch.Tensor:
    """NEXT-3: o = softmax_masked(scale * q k^T) v per (b, h), [B, H, S, D] float64;
    keys j >= clamp(lengths[b], 0, S) masked, o = 0 for an empty request."""
    qs, ks, vs = _host(q), _host(k), _host(v)
    if not (qs.shape == ks.shape == vs.shape) or qs.dim() != 4:
        raise ValueError("q, k, v must share one [B, H, S, D] shape")
    if not (qs.dtype == ks.dtype == vs.dtype):
        raise TypeError("q, k, v share one dtype")
    B, H, S, D = qs.shape
    lens = torch.as_tensor(np.asarray(lengths, dtype=np.int32)).contiguous()
    if lens.numel() != B:
        raise ValueError("lengths must have B entries")
    out = torch.empty((B, H, S, D), dtype=torch.float64)
    rc = _load().tto_attention(_ptr(qs), _ptr(ks), _ptr(vs), DTYPE_CODE[qs.dtype], _ptr(lens),
                               B, H, S, D, ctypes.c_float(scale), _ptr(out))
    assert rc == 0
    return out


# ------------------------------------------------------ NEXT-4 (Alg. 2) oracle
def plan_cost(lengths, cost, batches) -> float:
    """Alg. 2's objective: sum over batches of
    cached_cost[max length][count] * count (plain Python)."""
    total = 0.0
    for b in batches:
        L = max(int(lengths[i]) for i in b)
        total += float(cost[L][len(b)]) * len(b)
    return total


def schedule_bruteforce(lengths, cost, max_batch: int):
    """Exhaustive minimum of Alg. 2's objective over every contiguous partition
    of the length-sorted request list (2^(n-1) plans; small n only).  Returns
    (min_cost, one optimal plan as lists of request indices)."""
    n = len(lengths)
    order = sorted(range(n), key=lambda i: (int(lengths[i]), i))
    best, best_plan = float("inf"), None
    for mask in range(1 << max(n - 1, 0)):
        plan, cur = [], [order[0]] if n else []
        for k in range(1, n):
            if mask >> (k - 1) & 1:
                plan.append(cur)
                cur = []
            cur.append(order[k])
        if cur:
            plan.append(cur)
        if any(len(b) > max_batch for b in plan):
            continue
        c = plan_cost(lengths, cost, plan)
        if c < best:
            best, best_plan = c, plan
    return best, best_plan


def set_partitions(n: int):
    """Every partition of {0..n-1} into non-empty blocks, as lists of index
    lists, by restricted growth strings a[0] = 0, a[i] <= 1 + max(a[:i])
    (each partition exactly once; there are Bell(n) of them)."""
    if n == 0:
        yield []
        return
    a = [0] * n

    def rec(i, m):
        if i == n:
            blocks = [[] for _ in range(m + 1)]
            for idx, b in enumerate(a):
                blocks[b].append(idx)
            yield blocks
            return
        for b in range(m + 2):
            a[i] = b
            yield from rec(i + 1, max(m, b))

    yield from rec(1, 0)


def schedule_setpartition_bruteforce(lengths, cost, max_batch: int):
    """Exhaustive minimum of Alg. 2's objective (Eq. 2, l.609-615)
    over EVERY partition of the requests into batches of at most max_batch --
    not only the contiguous runs of the length-sorted list that Alg. 2 itself
    searches (l.619-648).  Bell(n) plans: n <= 10 only.  Returns (min_cost,
    one optimal plan as lists of request indices)."""
    n = len(lengths)
    best, best_plan = float("inf"), None
    for plan in set_partitions(n):
        if any(len(b) > max_batch for b in plan):
            continue
        c = plan_cost(lengths, cost, plan)
        if c < best:
            best, best_plan = c, plan
    return best, best_plan
