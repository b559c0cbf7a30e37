"""Tolerances for GPU-vs-oracle parity (north_star; R14).

g = GPU output widened to float64, ref = oracle (float64).
  fp32 softmax   |g - ref| <= 1e-5
  fp32 LN        |g - ref| <= 1e-4 * max(1, |ref|)
  fp16 (both)    |g - ref| <= 2e-3 * max(1, |ref|)
  bf16 softmax   |g - ref| <= 2e-3
  bf16 LN        |g - ref| <= max(2e-3 * max(1, |ref|), ulp_bf16(ref))
                 (the literal 2e-3 is below bf16's own rounding of LN outputs
                 of magnitude > 0.5; DESIGN R14(v))
  masked softmax positions: bit pattern exactly 0 (+0.0) in every dtype.
"""
import torch


def ulp_bf16(ref: torch.Tensor) -> torch.Tensor:
    a = ref.abs().clamp_min(2.0 ** -126)
    return torch.exp2(torch.floor(torch.log2(a)) - 7)


def bound(op: str, dtype, ref: torch.Tensor) -> torch.Tensor:
    one = torch.ones_like(ref)
    mag = torch.maximum(one, ref.abs())
    if op == "gelu":   # NEXT-2 element-wise: fp32 1e-5 relative, 16-bit as LayerNorm
        if dtype == torch.float32:
            return 1e-5 * mag
        op = "layernorm"
    if op == "softmax":
        if dtype == torch.float32:
            return torch.full_like(ref, 1e-5)
        if dtype == torch.float16:
            return 2e-3 * mag
        return torch.full_like(ref, 2e-3)
    if dtype == torch.float32:
        return 1e-4 * mag
    if dtype == torch.float16:
        return 2e-3 * mag
    return torch.maximum(2e-3 * mag, ulp_bf16(ref))


def assert_close(op: str, dtype, got: torch.Tensor, ref: torch.Tensor, what: str = ""):
    g = got.detach().to("cpu").to(torch.float64)
    r = ref.to(torch.float64)
    assert g.shape == r.shape, (g.shape, r.shape)
    err = (g - r).abs()
    b = bound(op, dtype, r)
    bad = ~(err <= b)  # NaN counts as bad
    if bad.any():
        idx = bad.nonzero()[0].tolist()
        raise AssertionError(
            f"{what} {op} {dtype}: {int(bad.sum())} of {g.numel()} outside tolerance; first at "
            f"{idx}: got {g[tuple(idx)].item()!r} ref {r[tuple(idx)].item()!r}; max err "
            f"{err.nan_to_num(float('inf')).max().item():.3e}")
    return err.max().item() if err.numel() else 0.0


def masked_bits_zero(y: torch.Tensor, lengths) -> bool:
    """Every padding key column (j >= clamp(L_b, 0, Sk)) holds bit pattern 0."""
    B, H, Sq, Sk = y.shape
    lens = torch.as_tensor(lengths, dtype=torch.int64, device=y.device).clamp(0, Sk)
    cols = torch.arange(Sk, device=y.device)
    mask = (cols[None, :] >= lens[:, None])[:, None, None, :].expand(B, H, Sq, Sk)
    ib = torch.int32 if y.dtype == torch.float32 else torch.int16
    bits = y.view(ib)
    return bool((bits[mask] == 0).all().item())


# ------------------------------------------------------------ every-row checks
# Full-size configs (C3, C4, C5 batches) are compared with the fp64 oracle on
# EVERY row: the oracle runs over row chunks on all host threads (its ctypes
# calls release the GIL) and each chunk is compared as soon as it is done, so
# no full-size float64 tensor is ever materialised.
def _pool():
    import concurrent.futures as cf
    import os
    return cf.ThreadPoolExecutor(max_workers=max(1, min(32, os.cpu_count() or 1)))


def softmax_all_rows(x_before: torch.Tensor, y: torch.Tensor, lengths, scale: float,
                     what: str = "") -> float:
    """x_before, y: [B, H, Sq, Sk] (CPU input snapshot, GPU or CPU output).
    Checks every row of every request against oracle.softmax_masked and every
    padding key for +0.0 bits.  Returns the max abs error."""
    import numpy as np
    import oracle
    B, H, Sq, Sk = x_before.shape
    lens = np.asarray(lengths, dtype=np.int32)
    yc = y.detach().to("cpu")
    dtype = x_before.dtype

    def one(b):
        ref = oracle.softmax_masked(x_before[b:b + 1], lens[b:b + 1], scale)
        err = assert_close("softmax", dtype, yc[b:b + 1], ref, f"{what} request {b}")
        assert masked_bits_zero(yc[b:b + 1], lens[b:b + 1]), f"{what} request {b}"
        return err

    with _pool() as ex:
        return max(ex.map(one, range(B)), default=0.0)


def layernorm_all_rows(d: dict, y: torch.Tensor, eps: float, what: str = "",
                       chunk: int = 2048) -> float:
    """d: CPU inputs (x, residual, bias, gamma, beta); y: [rows, hidden] output.
    Every row against oracle.add_bias_layernorm.  Returns the max abs error."""
    import oracle
    rows = d["x"].shape[0]
    yc = y.detach().to("cpu")
    dtype = d["x"].dtype

    def one(lo):
        hi = min(rows, lo + chunk)
        ref = oracle.add_bias_layernorm(d["x"][lo:hi], d["residual"][lo:hi], d["bias"],
                                        d["gamma"], d["beta"], eps)
        return assert_close("layernorm", dtype, yc[lo:hi], ref, f"{what} rows {lo}..{hi}")

    with _pool() as ex:
        return max(ex.map(one, range(0, rows, chunk)), default=0.0)
