"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Each test checks the oracle against something the paper or mathematics fixes:
closed forms (tests/golden/*), invariants, exhaustive decoder checks against an
independent library, brute force against 50-digit mpmath, and independent
library routines (torch float64).  A plausible mistake anywhere in the oracle
(a dropped term, a wrong sign or index, a transposed operand, N-1 instead of N,
eps outside the sqrt, a missed max subtraction, a masked key leaking into the
max or the sum) fails at least one of them.  CPU only.
"""
import itertools
import math

import mpmath
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import workloads as W
from conftest import read_golden

DT = [torch.float32, torch.float16, torch.bfloat16]


def _vals(s):
    return [float(v) for v in s.split()]


def _exact_in(dtype, vals):
    t = torch.tensor(vals, dtype=torch.float64)
    return bool(torch.equal(t.to(dtype).to(torch.float64), t))


# ----------------------------------------------------------------- decoders
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_widen_exhaustive_16bit(dtype):
    """Every one of the 65536 bit patterns decodes as torch's own widening."""
    bits = torch.arange(-32768, 32768, dtype=torch.int32).to(torch.int16)
    t = bits.view(dtype)
    got = oracle.widen(t)
    ref = t.to(torch.float64)
    nan = torch.isnan(ref)
    assert torch.equal(torch.isnan(got), nan)
    assert torch.equal(got[~nan], ref[~nan])
    # signed zeros keep their sign
    assert torch.equal(torch.signbit(got[~nan]), torch.signbit(ref[~nan]))


def test_widen_f32_exact():
    g = torch.Generator().manual_seed(1)
    t = torch.randn(4096, generator=g) * 1e3
    t[:4] = torch.tensor([0.0, -0.0, float("inf"), 1e-45])
    assert torch.equal(oracle.widen(t), t.double())


# ----------------------------------------------------------------- softmax
@pytest.mark.parametrize("dtype", DT)
def test_softmax_golden(dtype):
    rows = read_golden("softmax_closed_forms.txt")
    assert len(rows) >= 10
    ran = 0
    for name, scale, L, xs, ys, _ in rows:
        x, y = _vals(xs), _vals(ys)
        if not _exact_in(dtype, x):
            continue
        t = torch.tensor(x, dtype=dtype).reshape(1, 1, 1, -1)
        got = oracle.softmax_masked(t, [int(L)], float(scale)).reshape(-1)
        assert torch.allclose(got, torch.tensor(y, dtype=torch.float64), rtol=0, atol=2e-16), name
        # masked columns are +0.0 exactly (sign bit clear)
        Lc = min(max(int(L), 0), len(x))
        assert not torch.signbit(got[Lc:]).any(), name
        ran += 1
    assert ran >= 8


def _random_scores(B, H, Sq, Sk, dtype, seed, std=8.0):
    return W.scores(B, H, Sq, Sk, dtype, seed=seed, std=std)


@pytest.mark.parametrize("dtype", DT)
def test_softmax_rows_sum_to_one_and_masking(dtype):
    B, H, Sq, Sk = 5, 3, 7, 37
    x = _random_scores(B, H, Sq, Sk, dtype, 11)
    lens = [37, 1, 0, 20, 50]
    y = oracle.softmax_masked(x, lens, 0.125)
    for b, L in enumerate(lens):
        Lc = min(max(L, 0), Sk)
        if Lc:
            s = y[b, :, :, :Lc].sum(-1)
            assert torch.allclose(s, torch.ones_like(s), rtol=0, atol=1e-12)
            assert (y[b, :, :, :Lc] > 0).all() and (y[b, :, :, :Lc] <= 1).all()
        tail = y[b, :, :, Lc:]
        assert torch.equal(tail, torch.zeros_like(tail)) and not torch.signbit(tail).any()


def test_softmax_vs_torch_float64():
    """Independent library: torch.softmax over the valid prefix, zeros after."""
    for dtype in DT:
        B, H, Sq, Sk = 4, 2, 5, 64
        x = _random_scores(B, H, Sq, Sk, dtype, 21, std=40.0)  # peaky
        lens = [64, 33, 1, 9]
        y = oracle.softmax_masked(x, lens, 0.125)
        for b, L in enumerate(lens):
            ref = torch.softmax(x[b, ..., :L].double() * 0.125, dim=-1)
            assert torch.allclose(y[b, ..., :L], ref, rtol=0, atol=1e-15)
            assert torch.equal(y[b, ..., L:], torch.zeros_like(y[b, ..., L:]))


def test_softmax_shift_invariance_exact_shifts():
    """softmax(x + c) == softmax(x) for exactly representable shifts."""
    g = np.random.Generator(np.random.PCG64(5))
    x = torch.tensor(g.integers(-64, 65, size=(3, 2, 4, 24)) / 8.0, dtype=torch.float32)
    lens = [24, 13, 2]
    y0 = oracle.softmax_masked(x, lens, 1.0)
    for c in (1000.0, -1000.0, 3.5, -3.5):
        y = oracle.softmax_masked(x + c, lens, 1.0)
        assert torch.allclose(y, y0, rtol=0, atol=1e-13), c


def test_softmax_scale_closed_form():
    """softmax_masked(x, s) == softmax_masked(s*x, 1) for s = 0.125 (exact)."""
    x = _random_scores(2, 2, 3, 40, torch.float32, 31)
    lens = [40, 17]
    assert torch.allclose(oracle.softmax_masked(x, lens, 0.125),
                          oracle.softmax_masked(x * 0.125, lens, 1.0), rtol=0, atol=1e-15)


def test_softmax_poison_in_masked_columns():
    """NaN/+-Inf in padded keys change no output bit (DESIGN R1)."""
    for dtype in DT:
        x = _random_scores(4, 2, 3, 29, dtype, 41)
        lens = [29, 10, 1, 0]
        clean = oracle.softmax_masked(x, lens, 0.125)
        dirty = oracle.softmax_masked(W.poison_masked(x, lens), lens, 0.125)
        assert torch.equal(clean.view(torch.int64), dirty.view(torch.int64))


def test_softmax_bruteforce_mpmath():
    """All rows of length 1..5 over {-2..2} vs 50-digit mpmath (<= 1e-15)."""
    mpmath.mp.dps = 50
    rows = []
    for L in range(1, 6):
        for combo in itertools.product(range(-2, 3), repeat=L):
            rows.append(list(combo) + [0] * (5 - L))
    lens = []
    for L in range(1, 6):
        lens += [L] * (5 ** L)
    x = torch.tensor(rows, dtype=torch.float32)
    y = oracle.softmax_rows(x, lens, 1.0)
    exp_cache = {k: mpmath.exp(k) for k in range(-4, 5)}
    worst = 0.0
    for r, (row, L) in enumerate(zip(rows, lens)):
        m = max(row[:L])
        s = mpmath.fsum(exp_cache[v - m] for v in row[:L])
        for j in range(L):
            ref = exp_cache[row[j] - m] / s
            worst = max(worst, abs(float(ref) - y[r, j].item()))
        assert (y[r, L:] == 0).all()
    assert worst <= 1e-15, worst


# ----------------------------------------------------------------- layernorm
@pytest.mark.parametrize("dtype", DT)
def test_layernorm_golden(dtype):
    rows = read_golden("layernorm_closed_forms.txt")
    assert len(rows) >= 6
    for name, eps, xs, rs, bs, gs, bes, ys, _ in rows:
        ops = [torch.tensor(_vals(s), dtype=dtype) for s in (xs, rs, bs, gs, bes)]
        assert all(_exact_in(dtype, _vals(s)) for s in (xs, rs, bs, gs, bes))
        x, r, b, g, be = ops
        got = oracle.add_bias_layernorm(x[None], r[None], b, g, be, float(eps))[0]
        ref = torch.tensor(_vals(ys), dtype=torch.float64)
        # eps is passed as fp32; 1e-5 vs (float)1e-5 moves results by < 1e-12
        assert torch.allclose(got, ref, rtol=0, atol=1e-13), (name, got, ref)


@pytest.mark.parametrize("eps", [1e-12, 1e-5])
def test_layernorm_standardisation(eps):
    """gamma=1, beta=0: row mean 0, row variance var/(var+eps)."""
    d = W.ln_inputs(64, 768, torch.float32, seed=7)
    one, zero = torch.ones(768), torch.zeros(768)
    y = oracle.add_bias_layernorm(d["x"], d["residual"], d["bias"], one, zero, eps)
    v = d["x"].double() + d["bias"].double() + d["residual"].double()
    var = v.var(dim=-1, unbiased=False)
    assert torch.allclose(y.mean(-1), torch.zeros(64, dtype=torch.float64), atol=1e-12)
    assert torch.allclose(y.var(-1, unbiased=False), var / (var + float(np.float32(eps))),
                          rtol=0, atol=1e-12)


def test_layernorm_vs_torch_float64():
    """Independent library: F.layer_norm on the double sum (x + bias) + residual."""
    for dtype in DT:
        for hidden in (16, 37, 768, 1024):
            d = W.ln_inputs(33, hidden, dtype, seed=hidden)
            y = oracle.add_bias_layernorm(d["x"], d["residual"], d["bias"], d["gamma"], d["beta"],
                                          1e-5)
            v = d["x"].double() + d["bias"].double() + d["residual"].double()
            ref = F.layer_norm(v, (hidden,), d["gamma"].double(), d["beta"].double(),
                               float(np.float32(1e-5)))
            assert torch.allclose(y, ref, rtol=0, atol=1e-13), (dtype, hidden)


def test_layernorm_fused_adds_special_case():
    """add_bias_ln(x, res, bias) == ln(x + bias + res, bias=0, res=0) with the
    sum formed exactly (x on a dyadic grid)."""
    g = np.random.Generator(np.random.PCG64(3))
    x = torch.tensor(g.integers(-512, 512, size=(9, 40)) / 64.0, dtype=torch.float32)
    r = torch.tensor(g.integers(-512, 512, size=(9, 40)) / 64.0, dtype=torch.float32)
    b = torch.tensor(g.integers(-64, 64, size=40) / 64.0, dtype=torch.float32)
    gam = torch.tensor(1 + g.integers(-8, 8, size=40) / 64.0, dtype=torch.float32)
    bet = torch.tensor(g.integers(-8, 8, size=40) / 64.0, dtype=torch.float32)
    z = torch.zeros(40)
    a = oracle.add_bias_layernorm(x, r, b, gam, bet, 1e-5)
    c = oracle.add_bias_layernorm(x + b + r, torch.zeros_like(x), z, gam, bet, 1e-5)
    assert torch.allclose(a, c, rtol=0, atol=1e-14)


def test_layernorm_equivariance():
    """LN(alpha*v + c) == LN(v) for alpha > 0, eps = 0; alpha < 0 flips x_hat."""
    g = np.random.Generator(np.random.PCG64(9))
    v = torch.tensor(g.integers(-256, 256, size=(7, 64)) / 16.0, dtype=torch.float32)
    one, zero = torch.ones(64), torch.zeros(64)
    base = oracle.add_bias_layernorm(v, torch.zeros_like(v), zero, one, zero, 0.0)
    for alpha, c in ((2.0, 3.0), (0.5, -7.0), (4.0, 100.0)):
        y = oracle.add_bias_layernorm(alpha * v + c, torch.zeros_like(v), zero, one, zero, 0.0)
        assert torch.allclose(y, base, rtol=0, atol=1e-13)
    flip = oracle.add_bias_layernorm(-v, torch.zeros_like(v), zero, one, zero, 0.0)
    assert torch.allclose(flip, -base, rtol=0, atol=1e-13)


def test_layernorm_population_variance_not_bessel():
    """[1,2,3,4]: population var 1.25 (Eq. 1); Bessel's 5/3 would give 1.1619..."""
    x = torch.tensor([[1.0, 2, 3, 4]])
    z = torch.zeros(4)
    y = oracle.add_bias_layernorm(x, torch.zeros_like(x), z, torch.ones(4), z, 0.0)
    assert abs(y[0, 3].item() - 1.5 / math.sqrt(1.25)) < 1e-15
    assert abs(y[0, 3].item() - 1.5 / math.sqrt(5 / 3)) > 0.1


def test_eq1_onepass_matches_twopass_in_double():
    """Eq. 1: E(x-Ex)^2 == E(x^2) - E^2(x); in double the two agree to 1e-10
    relative (10^4 rows, |x| <= 100, N in 16..1024)."""
    g = np.random.Generator(np.random.PCG64(13))
    worst = 0.0
    for N in (16, 37, 64, 100, 256, 768, 1024):
        rows = 10000 // 7
        x = torch.tensor(g.uniform(-100, 100, size=(rows, N)), dtype=torch.float32)
        gam = torch.ones(N)
        bet = torch.zeros(N)
        one = oracle.layernorm_onepass_eq1(x, gam, bet, 1e-5)
        two = oracle.add_bias_layernorm(x, torch.zeros_like(x), bet, gam, bet, 1e-5)
        worst = max(worst, ((one - two).abs() / two.abs().clamp_min(1.0)).max().item())
    assert worst < 1e-10, worst


def test_eq1_onepass_cancellation_documented():
    """Eq. 1's RHS loses digits when mean >> std even in double; documented,
    not asserted beyond sanity.  The two forms still agree in
    double at offset 64, which is why the offset test targets fp32 kernels."""
    d = W.ln_inputs(16, 768, torch.float32, seed=3, offset=64.0)
    one = oracle.layernorm_onepass_eq1(d["x"], d["gamma"], d["beta"], 1e-12)
    two = oracle.add_bias_layernorm(d["x"], torch.zeros_like(d["x"]), torch.zeros(768),
                                    d["gamma"], d["beta"], 1e-12)
    assert (one - two).abs().max().item() < 1e-9


def test_oracle_argument_errors():
    with pytest.raises(ValueError):
        oracle.softmax_masked(torch.zeros(2, 3), [1], 1.0)
    with pytest.raises(ValueError):
        oracle.softmax_masked(torch.zeros(2, 1, 1, 3), [1], 1.0)
    with pytest.raises(TypeError):
        oracle.widen(torch.zeros(3, dtype=torch.int32))
    # empty shapes are no-ops
    assert oracle.softmax_masked(torch.zeros(0, 2, 2, 2), [], 1.0).numel() == 0


def test_packed_equals_padded_valid_blocks():
    """The packed layout holds exactly the valid
    [H, L_r, L_r] blocks of the padded masked softmax (P:l.576 padding)."""
    lens = [5, 1, 0, 9, 3, 9]
    H, S = 2, 9
    x = W.scores(len(lens), H, S, S, torch.float32, seed=17)
    padded = oracle.softmax_masked(W.poison_masked(x, lens), lens, 0.125)
    flat = torch.cat([x[b, :, :L, :L].reshape(-1) for b, L in enumerate(lens)])
    packed = oracle.softmax_packed(flat, lens, H, 0.125)
    ref = torch.cat([padded[b, :, :L, :L].reshape(-1) for b, L in enumerate(lens)])
    assert torch.equal(packed, ref)
    with pytest.raises(ValueError):
        oracle.softmax_packed(flat[:-1], lens, H, 0.125)
