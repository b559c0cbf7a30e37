"""Pins for the NEXT-3 attention oracle:
o = softmax_masked(scale * q k^T) v.  CPU only."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle

DT = [torch.float32, torch.float16, torch.bfloat16]


def _qkv(B, H, S, D, dtype, seed, std=1.0):
    g = torch.Generator().manual_seed(seed)
    return [(torch.randn(B, H, S, D, generator=g) * std).to(dtype) for _ in range(3)]


@pytest.mark.parametrize("dtype", DT)
def test_attention_vs_torch_sdpa_float64(dtype):
    B, H, S, D = 3, 2, 19, 16
    q, k, v = _qkv(B, H, S, D, dtype, 1, std=2.0)
    lens = [19, 7, 1]
    o = oracle.attention(q, k, v, lens, 0.25)
    for b, L in enumerate(lens):
        ref = F.scaled_dot_product_attention(q[b:b + 1].double(), k[b:b + 1, :, :L].double(),
                                             v[b:b + 1, :, :L].double(), scale=0.25)
        assert torch.allclose(o[b:b + 1], ref, rtol=0, atol=1e-13)


def test_attention_closed_forms():
    B, H, S, D = 1, 1, 6, 4
    q, k, v = _qkv(B, H, S, D, torch.float32, 2)
    # constant values -> output is that constant for every query
    vc = torch.full_like(v, 0.75)
    assert torch.allclose(oracle.attention(q, k, vc, [6], 1.0), torch.full((1, 1, 6, 4), 0.75,
                                                                        dtype=torch.float64),
                          rtol=0, atol=1e-15)
    # a single valid key -> every output row is that key's value
    o = oracle.attention(q, k, v, [1], 1.0)
    assert torch.equal(o, v[:, :, :1].double().expand(1, 1, 6, 4))
    # zero queries -> uniform weights -> the mean of the valid values
    o = oracle.attention(torch.zeros_like(q), k, v, [4], 1.0)
    assert torch.allclose(o[0, 0], v[0, 0, :4].double().mean(0).expand(6, 4), rtol=0, atol=1e-15)
    # empty request -> zeros
    assert torch.equal(oracle.attention(q, k, v, [0], 1.0), torch.zeros(1, 1, 6, 4,
                                                                        dtype=torch.float64))


def test_attention_masked_keys_never_matter():
    q, k, v = _qkv(2, 2, 9, 8, torch.float32, 3)
    lens = [5, 9]
    a = oracle.attention(q, k, v, lens, 0.5)
    k2, v2 = k.clone(), v.clone()
    k2[0, :, 5:] = float("nan")
    v2[0, :, 5:] = float("inf")
    assert torch.equal(oracle.attention(q, k2, v2, lens, 0.5), a)


def test_attention_is_softmax_times_v():
    """Composition pin: attention == (the pinned masked softmax of the logits) @ v."""
    B, H, S, D = 2, 3, 11, 8
    q, k, v = _qkv(B, H, S, D, torch.float32, 4)
    lens = np.array([11, 6], dtype=np.int32)
    logits = (q.double() @ k.double().transpose(-1, -2)).float()
    p = oracle.softmax_masked(logits, lens, 0.125)
    o = oracle.attention(q, k, v, lens, 0.125)
    # logits rounded to fp32 before the softmax oracle: agreement to ~1e-6
    assert torch.allclose(o, p @ v.double(), rtol=0, atol=1e-5)
