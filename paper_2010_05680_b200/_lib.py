"""ctypes binding of libtt.so (contract: include/tt.h).

Argument marshalling only: every step of both operations runs in the CUDA
kernels behind the C ABI.  There is no fallback of any kind -- if libtt.so is
missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TT_LIB_PATH") or os.path.join(_HERE, "libtt.so")  # override: experiments only

TT_SUCCESS = 0
TT_ERROR_INVALID_VALUE = 1
TT_ERROR_NOT_SUPPORTED = 2
TT_ERROR_CUDA = 3
TT_MAX_SOFTMAX_COLS = 1073741824
TT_MAX_LN_HIDDEN = 32768

DTYPE_CODE = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}
_SUFFIX = {torch.float32: "f32", torch.float16: "f16", torch.bfloat16: "bf16"}

# Every symbol include/tt.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "tt_softmax_masked_f32", "tt_softmax_masked_f16", "tt_softmax_masked_bf16",
    "tt_add_bias_layernorm_f32", "tt_add_bias_layernorm_f16", "tt_add_bias_layernorm_bf16",
    "tt_softmax_packed_f32", "tt_softmax_packed_f16", "tt_softmax_packed_bf16",
    "tt_softmax_masked_staged", "tt_add_bias_layernorm_staged",
    "tt_softmax_masked_staged_overlap", "tt_add_bias_layernorm_staged_overlap",
    "tt_status_string", "tt_last_cuda_error", "tt_version",
    "tt_softmax_masked_plan", "tt_add_bias_layernorm_plan", "tt_softmax_packed_plan",
    "ttx_tier_count", "ttx_tier_name", "ttx_force_tier",
    "tt_add_bias_gelu", "tt_split_qkv_add_bias", "tt_merge_heads",
    "tt_dp_schedule", "tt_schedule_cost", "tt_attention_fwd", "ttx_attention_variant",
    "ttx_attention_variant_count", "ttx_attention_variant_ok", "ttx_tuning_build", "ttx_set_pdl", "ttx_get_pdl",
)


class TTError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)}"
                         + (f" (cudaError {lib().tt_last_cuda_error()})" if status == TT_ERROR_CUDA
                            else ""))


_i64, _vp, _f, _i = ctypes.c_int64, ctypes.c_void_p, ctypes.c_float, ctypes.c_int
_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load libtt.so once.  Raises if the CUDA library is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libtt.so not found at {LIB_PATH}: build it with "
                    "`python -m paper_2010_05680_b200.build` (there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            sm = [_vp, _vp, _i64, _i64, _i64, _i64, _f, _vp]
            ln = [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f, _vp]
            for s in ("f32", "f16", "bf16"):
                getattr(L, f"tt_softmax_masked_{s}").argtypes = sm
                getattr(L, f"tt_add_bias_layernorm_{s}").argtypes = ln
            pk = [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _f, _vp]
            for s in ("f32", "f16", "bf16"):
                getattr(L, f"tt_softmax_packed_{s}").argtypes = pk
            L.tt_softmax_packed_plan.argtypes = [_i, _i64, ctypes.c_char_p, _i]
            L.tt_softmax_masked_staged.argtypes = [_i, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64,
                                                   _f, _vp]
            L.tt_add_bias_layernorm_staged.argtypes = [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                                       _vp, _i64, _i64, _f, _vp]
            L.tt_softmax_masked_staged_overlap.argtypes = [_i, _vp, _vp, _vp, _vp, _i64, _i64,
                                                           _i64, _i64, _f, _i64, _vp, _vp]
            L.tt_add_bias_layernorm_staged_overlap.argtypes = [_i, _vp, _vp, _vp, _vp, _vp, _vp,
                                                               _vp, _vp, _vp, _i64, _i64, _f,
                                                               _i64, _vp, _vp]
            L.tt_softmax_masked_plan.argtypes = [_i, _i64, _i64, _i64, _i64, ctypes.c_char_p, _i]
            L.tt_add_bias_layernorm_plan.argtypes = [_i, _i64, _i64, ctypes.c_char_p, _i]
            L.tt_add_bias_gelu.argtypes = [_i, _vp, _vp, _vp, _i64, _i64, _i, _vp]
            L.tt_split_qkv_add_bias.argtypes = [_i, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                                                _i64, _vp]
            L.tt_merge_heads.argtypes = [_i, _vp, _vp, _i64, _i64, _i64, _i64, _vp]
            L.tt_attention_fwd.argtypes = [_i, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64,
                                           _f, _vp]
            L.ttx_attention_variant.argtypes = [_i]
            L.ttx_attention_variant_count.argtypes = []
            L.ttx_attention_variant_ok.argtypes = [_i]
            L.ttx_tuning_build.argtypes = []
            L.ttx_set_pdl.argtypes = [_i]
            L.ttx_get_pdl.argtypes = []
            L.tt_dp_schedule.argtypes = [_vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp]
            L.tt_schedule_cost.argtypes = [_vp, _i64, _vp, _i64, _i64, _vp, _vp, _i64, _vp]
            L.ttx_tier_count.argtypes = [_i]
            L.ttx_tier_name.argtypes = [_i, _i, _i]
            L.ttx_tier_name.restype = ctypes.c_char_p
            L.ttx_force_tier.argtypes = [_i, _i, _i]
            L.tt_status_string.argtypes = [_i]
            L.tt_status_string.restype = ctypes.c_char_p
            for name in EXPORTS:
                if name not in ("tt_status_string", "ttx_tier_name"):
                    getattr(L, name).restype = _i
            _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().tt_status_string(int(s)).decode()


def version() -> int:
    return lib().tt_version()


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _check(status: int, what: str):
    if status != TT_SUCCESS:
        raise TTError(status, what)


def _dev(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _host(t: torch.Tensor, name: str):
    if t.is_cuda:
        raise ValueError(f"{name} must be a host tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _pair(h: torch.Tensor, d: torch.Tensor, name: str):
    """host/device counterparts: same shape and dtype (the copies move
    numel * element_size bytes between them)."""
    _host(h, f"host_{name}")
    _dev(d, f"dev_{name}")
    if h.shape != d.shape or h.dtype != d.dtype:
        raise ValueError(f"host_{name} / dev_{name} differ in shape or dtype")


def _staged_softmax_args(host_scores, host_lengths, dev_scores, dev_lengths):
    _pair(host_scores, dev_scores, "scores")
    _pair(host_lengths, dev_lengths, "lengths")
    if dev_scores.dim() != 4:
        raise ValueError("scores must be [B, H, Sq, Sk]")
    if dev_lengths.dtype != torch.int32 or dev_lengths.numel() != dev_scores.shape[0]:
        raise ValueError("lengths must be int32[B]")


def _staged_ln_args(host_out, host_x, host_residual, dev_out, dev_x, dev_residual, bias, gamma,
                    beta):
    for h, d, n in ((host_out, dev_out, "out"), (host_x, dev_x, "x"),
                    (host_residual, dev_residual, "residual")):
        _pair(h, d, n)
        if d.shape != dev_x.shape or d.dtype != dev_x.dtype:
            raise ValueError("out, x, residual must share one shape and dtype")
    hidden = dev_x.shape[-1] if dev_x.dim() else 0
    for t, n in ((bias, "bias"), (gamma, "gamma"), (beta, "beta")):
        _dev(t, n)
        if t.dtype != dev_x.dtype or t.numel() != hidden:
            raise ValueError(f"{n} must have `hidden` elements of the operands' dtype")


# --------------------------------------------------------------------- softmax
def tt_softmax_masked(scores: torch.Tensor, lengths: torch.Tensor, scale: float, stream=None):
    """In place: scores[b,h,i,:] <- masked softmax (tt_softmax_masked_{f32,f16,bf16})."""
    _dev(scores, "scores")
    _dev(lengths, "lengths")
    if scores.dim() != 4:
        raise ValueError("scores must be [B, H, Sq, Sk]")
    if lengths.dtype != torch.int32 or lengths.numel() != scores.shape[0]:
        raise ValueError("lengths must be int32[B]")
    B, H, Sq, Sk = scores.shape
    fn = getattr(lib(), f"tt_softmax_masked_{_SUFFIX[scores.dtype]}")
    _check(fn(scores.data_ptr(), lengths.data_ptr(), B, H, Sq, Sk, float(scale),
              _stream_ptr(stream)), fn.__name__)
    return scores


def tt_softmax_masked_raw(dtype: torch.dtype, scores_ptr: int, lengths_ptr: int, B: int, H: int,
                          Sq: int, Sk: int, scale: float, stream_ptr: int = 0) -> int:
    """Pointer-level call; returns the tt_status (used by the ABI tests)."""
    fn = getattr(lib(), f"tt_softmax_masked_{_SUFFIX[dtype]}")
    return fn(scores_ptr, lengths_ptr, B, H, Sq, Sk, float(scale), stream_ptr)


def tt_softmax_masked_staged(host_scores: torch.Tensor, host_lengths: torch.Tensor,
                             dev_scores: torch.Tensor, dev_lengths: torch.Tensor, scale: float,
                             stream=None):
    """H2D copy, kernel, D2H copy on one stream (host buffers pinned)."""
    _staged_softmax_args(host_scores, host_lengths, dev_scores, dev_lengths)
    B, H, Sq, Sk = dev_scores.shape
    _check(lib().tt_softmax_masked_staged(DTYPE_CODE[dev_scores.dtype], host_scores.data_ptr(),
                                          host_lengths.data_ptr(), dev_scores.data_ptr(),
                                          dev_lengths.data_ptr(), B, H, Sq, Sk, float(scale),
                                          _stream_ptr(stream)), "tt_softmax_masked_staged")
    return host_scores


def tt_softmax_masked_staged_overlap(host_scores: torch.Tensor, host_lengths: torch.Tensor,
                                     dev_scores: torch.Tensor, dev_lengths: torch.Tensor,
                                     scale: float, chunks: int, stream=None, copy_stream=None):
    """As tt_softmax_masked_staged, cut into `chunks` pieces whose D2H copies run
    on `copy_stream` under the next piece's H2D copy (include/tt.h)."""
    _staged_softmax_args(host_scores, host_lengths, dev_scores, dev_lengths)
    B, H, Sq, Sk = dev_scores.shape
    _check(lib().tt_softmax_masked_staged_overlap(
        DTYPE_CODE[dev_scores.dtype], host_scores.data_ptr(), host_lengths.data_ptr(),
        dev_scores.data_ptr(), dev_lengths.data_ptr(), B, H, Sq, Sk, float(scale), int(chunks),
        _stream_ptr(stream), _stream_ptr(copy_stream) if copy_stream is not None else None),
        "tt_softmax_masked_staged_overlap")
    return host_scores


def softmax_plan(dtype: torch.dtype, B: int, H: int, Sq: int, Sk: int) -> str:
    buf = ctypes.create_string_buffer(128)
    _check(lib().tt_softmax_masked_plan(DTYPE_CODE[dtype], B, H, Sq, Sk, buf, 128),
           "tt_softmax_masked_plan")
    return buf.value.decode()


# ---------------------------------------------------------------------- packed
def packed_offsets(lengths, H: int, device="cuda"):
    """cu_seqlens (int32[n+1]) and dense block offsets cu_blocks (int64[n],
    H * sum_{i<r} L_i^2) for requests of the given lengths (host plumbing)."""
    lens = torch.as_tensor(lengths, dtype=torch.int64).cpu()
    cu = torch.zeros(lens.numel() + 1, dtype=torch.int64)
    cu[1:] = torch.cumsum(lens, 0)
    blocks = torch.zeros(lens.numel(), dtype=torch.int64)
    if lens.numel() > 1:
        blocks[1:] = torch.cumsum(H * lens * lens, 0)[:-1]
    return cu.to(torch.int32).to(device), blocks.to(device), int(cu[-1]), int(
        (H * lens * lens).sum())


def tt_softmax_packed(scores: torch.Tensor, cu_seqlens: torch.Tensor, cu_blocks: torch.Tensor,
                      H: int, total_tokens: int, max_seqlen: int, scale: float, stream=None):
    """In place: every [H, L_r, L_r] block of the packed `scores` buffer
    (tt_softmax_packed_{f32,f16,bf16})."""
    _dev(scores, "scores")
    _dev(cu_seqlens, "cu_seqlens")
    _dev(cu_blocks, "cu_blocks")
    if cu_seqlens.dtype != torch.int32 or cu_blocks.dtype != torch.int64:
        raise ValueError("cu_seqlens must be int32, cu_blocks int64")
    n = cu_blocks.numel()
    if cu_seqlens.numel() != n + 1:
        raise ValueError("cu_seqlens must have num_req + 1 entries")
    fn = getattr(lib(), f"tt_softmax_packed_{_SUFFIX[scores.dtype]}")
    _check(fn(scores.data_ptr(), cu_seqlens.data_ptr(), cu_blocks.data_ptr(), n, H, total_tokens,
              max_seqlen, float(scale), _stream_ptr(stream)), fn.__name__)
    return scores


def softmax_packed_plan(dtype: torch.dtype, max_seqlen: int) -> str:
    buf = ctypes.create_string_buffer(128)
    _check(lib().tt_softmax_packed_plan(DTYPE_CODE[dtype], max_seqlen, buf, 128),
           "tt_softmax_packed_plan")
    return buf.value.decode()


# ------------------------------------------------------------------- layernorm
def tt_add_bias_layernorm(out: torch.Tensor, x: torch.Tensor, residual: torch.Tensor,
                          bias: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor,
                          eps: float, stream=None):
    """out <- LayerNorm((x + bias) + residual) * gamma + beta (tt_add_bias_layernorm_*)."""
    for t, n in ((out, "out"), (x, "x"), (residual, "residual"), (bias, "bias"),
                 (gamma, "gamma"), (beta, "beta")):
        _dev(t, n)
        if t.dtype != x.dtype:
            raise ValueError("all operands share one dtype")
    hidden = x.shape[-1]
    rows = x.numel() // hidden if hidden else 0
    if out.shape != x.shape or residual.shape != x.shape:
        raise ValueError("out, x, residual must have the same shape")
    if bias.numel() != hidden or gamma.numel() != hidden or beta.numel() != hidden:
        raise ValueError("bias, gamma, beta must have `hidden` elements")
    fn = getattr(lib(), f"tt_add_bias_layernorm_{_SUFFIX[x.dtype]}")
    _check(fn(out.data_ptr(), x.data_ptr(), residual.data_ptr(), bias.data_ptr(),
              gamma.data_ptr(), beta.data_ptr(), rows, hidden, float(eps), _stream_ptr(stream)),
           fn.__name__)
    return out


def tt_add_bias_layernorm_raw(dtype: torch.dtype, out: int, x: int, residual: int, bias: int,
                              gamma: int, beta: int, rows: int, hidden: int, eps: float,
                              stream_ptr: int = 0) -> int:
    fn = getattr(lib(), f"tt_add_bias_layernorm_{_SUFFIX[dtype]}")
    return fn(out, x, residual, bias, gamma, beta, rows, hidden, float(eps), stream_ptr)


def tt_add_bias_layernorm_staged(host_out, host_x, host_residual, dev_out, dev_x, dev_residual,
                                 bias, gamma, beta, eps: float, stream=None):
    _staged_ln_args(host_out, host_x, host_residual, dev_out, dev_x, dev_residual, bias, gamma,
                    beta)
    hidden = dev_x.shape[-1]
    rows = dev_x.numel() // hidden if hidden else 0
    _check(lib().tt_add_bias_layernorm_staged(
        DTYPE_CODE[dev_x.dtype], host_out.data_ptr(), host_x.data_ptr(), host_residual.data_ptr(),
        dev_out.data_ptr(), dev_x.data_ptr(), dev_residual.data_ptr(), bias.data_ptr(),
        gamma.data_ptr(), beta.data_ptr(), rows, hidden, float(eps), _stream_ptr(stream)),
        "tt_add_bias_layernorm_staged")
    return host_out


def tt_add_bias_layernorm_staged_overlap(host_out, host_x, host_residual, dev_out, dev_x,
                                         dev_residual, bias, gamma, beta, eps: float, chunks: int,
                                         stream=None, copy_stream=None):
    """As tt_add_bias_layernorm_staged, cut into `chunks` row ranges whose D2H
    copies run on `copy_stream` (include/tt.h)."""
    _staged_ln_args(host_out, host_x, host_residual, dev_out, dev_x, dev_residual, bias, gamma,
                    beta)
    hidden = dev_x.shape[-1]
    rows = dev_x.numel() // hidden if hidden else 0
    _check(lib().tt_add_bias_layernorm_staged_overlap(
        DTYPE_CODE[dev_x.dtype], host_out.data_ptr(), host_x.data_ptr(), host_residual.data_ptr(),
        dev_out.data_ptr(), dev_x.data_ptr(), dev_residual.data_ptr(), bias.data_ptr(),
        gamma.data_ptr(), beta.data_ptr(), rows, hidden, float(eps), int(chunks),
        _stream_ptr(stream), _stream_ptr(copy_stream) if copy_stream is not None else None),
        "tt_add_bias_layernorm_staged_overlap")
    return host_out


def layernorm_plan(dtype: torch.dtype, rows: int, hidden: int) -> str:
    buf = ctypes.create_string_buffer(128)
    _check(lib().tt_add_bias_layernorm_plan(DTYPE_CODE[dtype], rows, hidden, buf, 128),
           "tt_add_bias_layernorm_plan")
    return buf.value.decode()


# --------------------------------------------------------------------- NEXT-2
def tt_add_bias_gelu(out: torch.Tensor, x: torch.Tensor, bias: torch.Tensor,
                     approximate: bool = False, stream=None):
    """out <- gelu(x + bias) over the last dim (tt_add_bias_gelu)."""
    for t, nm in ((out, "out"), (x, "x"), (bias, "bias")):
        _dev(t, nm)
        if t.dtype != x.dtype:
            raise ValueError("all operands share one dtype")
    n = x.shape[-1]
    rows = x.numel() // n if n else 0
    if out.shape != x.shape or bias.numel() != n:
        raise ValueError("shape mismatch")
    _check(lib().tt_add_bias_gelu(DTYPE_CODE[x.dtype], out.data_ptr(), x.data_ptr(),
                                  bias.data_ptr(), rows, n, int(bool(approximate)),
                                  _stream_ptr(stream)), "tt_add_bias_gelu")
    return out


def tt_split_qkv_add_bias(q, k, v, qkv, bias, B: int, S: int, H: int, D: int, stream=None):
    """qkv [B*S, 3*H*D] + bias -> q, k, v [B, H, S, D] (tt_split_qkv_add_bias)."""
    for t, nm in ((q, "q"), (k, "k"), (v, "v"), (qkv, "qkv"), (bias, "bias")):
        _dev(t, nm)
        if t.dtype != qkv.dtype:
            raise ValueError("all operands share one dtype")
    if qkv.numel() != B * S * 3 * H * D or bias.numel() != 3 * H * D or \
            any(t.numel() != B * H * S * D for t in (q, k, v)):
        raise ValueError("shape mismatch")
    _check(lib().tt_split_qkv_add_bias(DTYPE_CODE[qkv.dtype], q.data_ptr(), k.data_ptr(),
                                       v.data_ptr(), qkv.data_ptr(), bias.data_ptr(), B, S, H, D,
                                       _stream_ptr(stream)), "tt_split_qkv_add_bias")
    return q, k, v


def tt_merge_heads(out, x, B: int, S: int, H: int, D: int, stream=None):
    """[B, H, S, D] -> [B*S, H*D] (tt_merge_heads)."""
    _dev(out, "out")
    _dev(x, "in")
    if out.dtype != x.dtype or out.numel() != x.numel() or x.numel() != B * H * S * D:
        raise ValueError("shape mismatch")
    _check(lib().tt_merge_heads(DTYPE_CODE[x.dtype], out.data_ptr(), x.data_ptr(), B, S, H, D,
                                _stream_ptr(stream)), "tt_merge_heads")
    return out


# ------------------------------------------------------------------ attention
def tt_attention_fwd(out, q, k, v, lengths, scale: float, stream=None):
    """NEXT-3: out <- softmax_masked(scale * q k^T) v on tcgen05 (tt_attention_fwd);
    q, k, v, out [B, H, S, 64] fp16/bf16, lengths int32[B] on the device."""
    for t, nm in ((out, "out"), (q, "q"), (k, "k"), (v, "v"), (lengths, "lengths")):
        _dev(t, nm)
    if not (q.shape == k.shape == v.shape == out.shape) or q.dim() != 4:
        raise ValueError("q, k, v, out must share one [B, H, S, D] shape")
    if not (q.dtype == k.dtype == v.dtype == out.dtype) or lengths.dtype != torch.int32:
        raise ValueError("dtype mismatch")
    B, H, S, D = q.shape
    _check(lib().tt_attention_fwd(DTYPE_CODE[q.dtype], out.data_ptr(), q.data_ptr(),
                                  k.data_ptr(), v.data_ptr(), lengths.data_ptr(), B, H, S, D,
                                  float(scale), _stream_ptr(stream)), "tt_attention_fwd")
    return out


def attention_variant(v: int):
    """0 = automatic, 1 = 128-key tiles single-buffered (2 CTAs/SM), 2 = 128-key
    tiles double-buffered, pipelined (1 CTA/SM), 3 = 64-key tiles (4 CTAs/SM),
    4 = 64-key tiles double-buffered, pipelined (3 CTAs/SM), 5 = warp-specialised
    (producer / MMA / softmax warps, mbarrier hand-offs, 2 CTAs/SM), 6 / 7 = variant 4
    with two threads per query row (2 / 3 CTAs/SM), 8 = variant 4 with the previous
    P.V waited for after the exponentials, 9 / 10 = warp-specialised TMA schedules
    with 128- / 64-key tiles (1..10: tuning build only)."""
    _check(lib().ttx_attention_variant(int(v)), "ttx_attention_variant")


def attention_variants() -> list:
    """Attention variants compiled into the loaded library besides 0 (automatic)."""
    L = lib()
    return [v for v in range(1, L.ttx_attention_variant_count()) if L.ttx_attention_variant_ok(v)]


def tuning_build() -> bool:
    return bool(lib().ttx_tuning_build())


def set_pdl(enable: bool):
    """Programmatic dependent launch on (default) or off for every kernel of the
    library (include/tt_tune.h ttx_set_pdl)."""
    _check(lib().ttx_set_pdl(1 if enable else 0), "ttx_set_pdl")


def get_pdl() -> bool:
    return bool(lib().ttx_get_pdl())


# ------------------------------------------------------------------ scheduler
def _cost_array(cost):
    import numpy as np
    c = np.ascontiguousarray(np.asarray(cost, dtype=np.float64))
    if c.ndim != 2 or c.shape[0] < 2 or c.shape[1] < 2:
        raise ValueError("cost table must be [max_len + 1, max_batch + 1]")
    return c


def dp_schedule(lengths, cost):
    """Alg. 2 (tt_dp_schedule): returns (batches, total_cost), each batch a list
    of request indices (queue order), batches in increasing padded length."""
    import numpy as np
    lens = np.ascontiguousarray(np.asarray(lengths, dtype=np.int32))
    c = _cost_array(cost)
    n = lens.size
    order = np.zeros(max(n, 1), dtype=np.int32)
    starts = np.zeros(n + 1, dtype=np.int32)
    nb = ctypes.c_int64(0)
    tot = ctypes.c_double(0.0)
    _check(lib().tt_dp_schedule(lens.ctypes.data, n, c.ctypes.data, c.shape[0] - 1,
                                c.shape[1] - 1, order.ctypes.data, starts.ctypes.data,
                                ctypes.addressof(nb), ctypes.addressof(tot)), "tt_dp_schedule")
    batches = [order[starts[b]:starts[b + 1]].tolist() for b in range(nb.value)]
    return batches, tot.value


def schedule_cost(lengths, cost, batches) -> float:
    """Cost of a given plan under Alg. 2's model (tt_schedule_cost)."""
    import numpy as np
    lens = np.ascontiguousarray(np.asarray(lengths, dtype=np.int32))
    c = _cost_array(cost)
    idx = np.ascontiguousarray(np.asarray([i for b in batches for i in b] or [0],
                                          dtype=np.int32))
    starts = np.ascontiguousarray(np.cumsum([0] + [len(b) for b in batches]).astype(np.int32))
    tot = ctypes.c_double(0.0)
    _check(lib().tt_schedule_cost(lens.ctypes.data, lens.size, c.ctypes.data, c.shape[0] - 1,
                                  c.shape[1] - 1, idx.ctypes.data, starts.ctypes.data,
                                  len(batches), ctypes.addressof(tot)), "tt_schedule_cost")
    return tot.value


# --------------------------------------------------------------------- tuning
OPS = {"softmax": 0, "layernorm": 1}


def tiers(op: str, dtype: torch.dtype) -> list:
    """Names of every compiled tier of `op` for `dtype` (include/tt_tune.h)."""
    L = lib()
    o = OPS[op]
    return [L.ttx_tier_name(o, DTYPE_CODE[dtype], i).decode() for i in range(L.ttx_tier_count(o))]


def force_tier(op: str, dtype: torch.dtype, index: int):
    """Force tier `index` (-1 = automatic) for subsequent calls in this process."""
    _check(lib().ttx_force_tier(OPS[op], DTYPE_CODE[dtype], int(index)), "ttx_force_tier")
