"""GPU parity for the NEXT-2 element-wise kernels (PAPER.md
l.304-308): add-bias + GELU, QKV split with bias, head merge -- through the C
ABI, against the fp64 oracle."""
import pytest
import torch

import oracle
import workloads as W
from _parity import assert_close

pytestmark = pytest.mark.gpu
DT = [torch.float32, torch.float16, torch.bfloat16]


def _gen(shape, dtype, seed, std=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(shape, generator=g) * std).to(dtype)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("approx", [False, True])
@pytest.mark.parametrize("rows,n", [(40, 3072), (37, 3000), (5, 4096), (3, 17), (128, 1024),
                                    (1, 8)])
def test_add_bias_gelu(ttlib, dtype, approx, rows, n):
    x = _gen((rows, n), dtype, rows + n, std=3.0)
    b = _gen((n,), dtype, n, std=0.5)
    out = torch.empty_like(x, device="cuda")
    ttlib.tt_add_bias_gelu(out, x.cuda(), b.cuda(), approximate=approx)
    torch.cuda.synchronize()
    assert_close("gelu", dtype, out, oracle.add_bias_gelu(x, b, approximate=approx),
                 f"gelu {rows}x{n}")


@pytest.mark.parametrize("dtype", DT)
def test_add_bias_gelu_in_place_and_bert_ffn_shape(ttlib, dtype):
    rows, n = 20 * 128, 3072          # BERT-base FFN-up output, batch 20 seq 128
    x = W.scores(1, 1, rows, n, dtype, device="cuda", seed=7, std=2.0).reshape(rows, n)
    b = _gen((n,), dtype, 1, std=0.1).cuda()
    ref_in = x[:: 97].cpu()
    ttlib.tt_add_bias_gelu(x, x, b)   # in place
    torch.cuda.synchronize()
    assert_close("gelu", dtype, x[:: 97], oracle.add_bias_gelu(ref_in, b.cpu()), "in place")


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("rows,n", [(32771, 1024), (4099, 4100)])
def test_add_bias_gelu_large_calls(ttlib, dtype, rows, n):
    """Calls of >= 4 M vectors take the 4-vectors-per-thread kernel (elementwise.cu
    kGeluBigVecs): a row count that leaves a partial last CTA span, and a width whose
    pitch is not a multiple of the 16-byte vector (element-size vectors); every 61st
    row and the last row against the oracle."""
    x = W.scores(1, 1, rows, n, dtype, device="cuda", seed=rows, std=2.0).reshape(rows, n)
    b = _gen((n,), dtype, 3, std=0.3).cuda()
    out = torch.empty_like(x)
    ttlib.tt_add_bias_gelu(out, x, b)
    torch.cuda.synchronize()
    idx = torch.cat([torch.arange(0, rows, 61), torch.tensor([rows - 1])]).cuda()
    assert_close("gelu", dtype, out[idx], oracle.add_bias_gelu(x[idx].cpu(), b.cpu()),
                 f"gelu {rows}x{n}")


def _split_ref(qkv, bias, B, S, H, D, dtype):
    return [t.to(dtype) for t in oracle.split_qkv_add_bias(qkv, bias, B, S, H, D)]


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("B,S,H,D", [(1, 40, 12, 64), (20, 37, 12, 64), (3, 5, 16, 64),
                                     (2, 7, 3, 20), (1, 1, 1, 8), (4, 9, 2, 3)])
def test_split_qkv_add_bias_bit_exact(ttlib, dtype, B, S, H, D):
    """The sum of two stored values is exact in fp32 here, so one RNE rounding
    on each side: the GPU result equals the oracle rounded to the storage dtype."""
    qkv = _gen((B * S, 3 * H * D), dtype, B * S + H)
    bias = _gen((3 * H * D,), dtype, D, std=0.1)
    q, k, v = (torch.empty(B, H, S, D, dtype=dtype, device="cuda") for _ in range(3))
    ttlib.tt_split_qkv_add_bias(q, k, v, qkv.cuda(), bias.cuda(), B, S, H, D)
    torch.cuda.synchronize()
    for got, ref in zip((q, k, v), _split_ref(qkv, bias, B, S, H, D, dtype)):
        assert torch.equal(got.cpu(), ref)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("B,S,H,D", [(1, 40, 12, 64), (20, 37, 12, 64), (2, 7, 3, 20),
                                     (4, 9, 2, 3), (64, 16, 16, 64)])
def test_merge_heads_exact(ttlib, dtype, B, S, H, D):
    x = _gen((B, H, S, D), dtype, S + H)
    out = torch.empty(B * S, H * D, dtype=dtype, device="cuda")
    ttlib.tt_merge_heads(out, x.cuda(), B, S, H, D)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), oracle.merge_heads(x, B, S, H, D).to(dtype))


def test_next2_rejects_bad_arguments(ttlib):
    x = torch.zeros(4, 8, device="cuda")
    with pytest.raises(ttlib.TTError):          # out partially overlapping x
        ttlib.lib()  # noqa
        st = ttlib.lib().tt_add_bias_gelu(0, x.data_ptr() + 4, x.data_ptr(),
                                          torch.zeros(8, device="cuda").data_ptr(), 3, 8, 0, 0)
        ttlib._lib._check(st, "gelu")
    q = torch.zeros(1, 1, 2, 8, device="cuda")
    with pytest.raises(ttlib.TTError):          # q == k
        st = ttlib.lib().tt_split_qkv_add_bias(0, q.data_ptr(), q.data_ptr(),
                                               torch.zeros_like(q).data_ptr(),
                                               torch.zeros(2, 24, device="cuda").data_ptr(),
                                               torch.zeros(24, device="cuda").data_ptr(),
                                               1, 2, 1, 8, 0)
        ttlib._lib._check(st, "split")
