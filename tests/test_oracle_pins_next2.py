"""Pins for the NEXT-2 oracle functions (the other fused
non-GEMM kernels): add-bias + GELU and the QKV split /
head merge transposes.  CPU only."""
import math

import mpmath
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle

DT = [torch.float32, torch.float16, torch.bfloat16]


def test_gelu_closed_forms_and_identity():
    """gelu(0) = 0; gelu(v) - gelu(-v) = v exactly (Phi(v) + Phi(-v) = 1);
    gelu(1) = Phi(1) to 50 digits."""
    v = torch.tensor([[0.0, 1.0, -1.0, 2.5, -2.5, 8.0, -8.0, 0.5]])
    z = torch.zeros(8)
    y = oracle.add_bias_gelu(v, z)
    assert y[0, 0].item() == 0.0
    for i, j in ((1, 2), (3, 4), (5, 6)):
        assert abs((y[0, i] - y[0, j]).item() - v[0, i].item()) < 1e-15
    mpmath.mp.dps = 50
    phi1 = float(mpmath.ncdf(1))
    assert abs(y[0, 1].item() - phi1) < 1e-16
    # large |v|: gelu(v) -> v, gelu(-v) -> 0
    assert abs(y[0, 5].item() - 8.0) < 1e-14 and abs(y[0, 6].item()) < 1e-14


def test_gelu_bias_is_added_before_activation():
    x = torch.tensor([[0.5, -1.0]])
    b = torch.tensor([0.5, 1.0])
    y = oracle.add_bias_gelu(x, b)
    assert abs(y[0, 0].item() - float(mpmath.ncdf(1))) < 1e-16   # gelu(1)
    assert y[0, 1].item() == 0.0                                 # gelu(0)


@pytest.mark.parametrize("dtype", DT)
def test_gelu_vs_torch_float64(dtype):
    g = torch.Generator().manual_seed(3)
    x = (torch.randn(17, 96, generator=g) * 3).to(dtype)
    b = (torch.randn(96, generator=g) * 0.1).to(dtype)
    v = x.double() + b.double()
    assert torch.allclose(oracle.add_bias_gelu(x, b), F.gelu(v), rtol=0, atol=1e-14)
    assert torch.allclose(oracle.add_bias_gelu(x, b, approximate=True),
                          F.gelu(v, approximate="tanh"), rtol=0, atol=1e-14)


def test_gelu_tanh_form_closed_value():
    """tanh form at v = 1: 0.5 (1 + tanh(sqrt(2/pi) * 1.044715))."""
    y = oracle.add_bias_gelu(torch.tensor([[1.0]]), torch.zeros(1), approximate=True)
    ref = 0.5 * (1 + math.tanh(math.sqrt(2 / math.pi) * 1.044715))
    assert abs(y.item() - ref) < 1e-15


@pytest.mark.parametrize("dtype", DT)
def test_split_qkv_is_the_stated_permutation(dtype):
    """Index-exact check with unique values (no two elements equal)."""
    B, S, H, D = 2, 3, 4, 5
    n = B * S * 3 * H * D
    qkv = torch.arange(n, dtype=torch.float32).reshape(B * S, 3 * H * D)
    if dtype != torch.float32:
        qkv = (qkv % 64).to(dtype)   # exactly representable in 16-bit
    bias = torch.zeros(3 * H * D, dtype=dtype)
    q, k, v = oracle.split_qkv_add_bias(qkv, bias, B, S, H, D)
    ref = qkv.double().reshape(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
    assert torch.equal(q, ref[0]) and torch.equal(k, ref[1]) and torch.equal(v, ref[2])


def test_split_qkv_bias_per_part_and_head():
    B, S, H, D = 1, 2, 2, 3
    qkv = torch.zeros(B * S, 3 * H * D)
    bias = torch.arange(3 * H * D, dtype=torch.float32)
    q, k, v = oracle.split_qkv_add_bias(qkv, bias, B, S, H, D)
    for t, out in enumerate((q, k, v)):
        for h in range(H):
            assert torch.equal(out[0, h, 1], bias[(t * H + h) * D:(t * H + h + 1) * D].double())


@pytest.mark.parametrize("dtype", DT)
def test_merge_heads_inverts_the_head_split(dtype):
    B, S, H, D = 3, 5, 4, 8
    g = torch.Generator().manual_seed(1)
    x = torch.randn(B, H, S, D, generator=g).to(dtype)
    m = oracle.merge_heads(x, B, S, H, D)
    assert torch.equal(m, x.double().permute(0, 2, 1, 3).reshape(B * S, H * D))
    # merge(split(qkv)) restores each third of the token-major input
    qkv = torch.randn(B * S, 3 * H * D, generator=g).to(dtype)
    q, k, v = oracle.split_qkv_add_bias(qkv, torch.zeros(3 * H * D, dtype=dtype), B, S, H, D)
    for t, part in enumerate((q, k, v)):
        back = oracle.merge_heads(part.to(dtype), B, S, H, D)
        assert torch.equal(back, qkv.double()[:, t * H * D:(t + 1) * H * D])


def test_next2_argument_errors():
    with pytest.raises(ValueError):
        oracle.add_bias_gelu(torch.zeros(2, 3), torch.zeros(4))
    with pytest.raises(ValueError):
        oracle.split_qkv_add_bias(torch.zeros(2, 10), torch.zeros(10), 1, 2, 1, 3)
    with pytest.raises(ValueError):
        oracle.merge_heads(torch.zeros(7), 1, 2, 2, 2)
    assert oracle.add_bias_gelu(torch.zeros(0, 4), torch.zeros(4)).numel() == 0
