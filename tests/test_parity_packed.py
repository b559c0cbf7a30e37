"""GPU parity: tt_softmax_packed_* (padding-free softmax)
vs the fp64 oracle.  Request r is a dense [H, L_r, L_r] block; every key valid."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from _parity import assert_close

pytestmark = pytest.mark.gpu
DT = [torch.float32, torch.float16, torch.bfloat16]


def _packed_input(lens, H, dtype, seed, device="cpu"):
    n = int(sum(H * L * L for L in lens))
    g = torch.Generator(device=device).manual_seed(seed)
    x = torch.randn(max(n, 1), generator=g, device=device) * W.LOGIT_STD
    return x[:n].to(dtype)


def _run(tt, flat_cpu, lens, H, scale, max_seqlen=None):
    cu, blocks, total, n = tt.packed_offsets(lens, H)
    assert n == flat_cpu.numel()
    y = flat_cpu.cuda()
    tt.tt_softmax_packed(y, cu, blocks, H, total, max_seqlen or max(1, int(max(lens))), scale)
    torch.cuda.synchronize()
    return y


@pytest.mark.parametrize("dtype", DT)
def test_c3_lengths_packed(ttlib, dtype):
    lens = W.c3_lengths()
    H = 12
    x = _packed_input(lens, H, dtype, seed=3)
    y = _run(ttlib, x, lens, H, W.SCALE_BERT)
    assert_close("softmax", dtype, y, oracle.softmax_packed(x, lens, H, W.SCALE_BERT), "C3 packed")


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_c5_batches_packed(ttlib, dtype):
    for bi in (0, 31, 63):
        lens = W.c5_stream()[bi]
        x = _packed_input(lens, 12, dtype, seed=bi)
        y = _run(ttlib, x, lens, 12, W.SCALE_BERT)
        assert_close("softmax", dtype, y, oracle.softmax_packed(x, lens, 12, W.SCALE_BERT),
                     f"C5 b{bi} packed")


@pytest.mark.parametrize("dtype", DT)
def test_many_tiny_requests_straddle_ctas(ttlib, dtype):
    """Requests with fewer rows than a CTA chunk: CTAs straddle requests."""
    lens = list(range(0, 23)) + [1, 0, 2, 0, 3]
    x = _packed_input(lens, 2, dtype, seed=5)
    y = _run(ttlib, x, lens, 2, W.SCALE_BERT)
    assert_close("softmax", dtype, y, oracle.softmax_packed(x, lens, 2, W.SCALE_BERT), "tiny")


@pytest.mark.parametrize("num_req", [33, 1025, 40000])
def test_many_requests_search_rounds(ttlib, num_req):
    """The warp-parallel request search (32 probes per round, softmax_packed.cu
    find_req_warp) over 2, 3 and 4 rounds: many short requests with empty ones
    (equal cu_seqlens entries) mixed in, CTAs inside and across requests."""
    rng = np.random.default_rng(num_req)
    lens = rng.integers(0, 24, size=num_req)
    lens[rng.choice(num_req, num_req // 7, replace=False)] = 0
    lens[-1] = 17
    x = _packed_input(lens, 2, torch.float16, seed=num_req)
    y = _run(ttlib, x, lens, 2, W.SCALE_BERT)
    assert_close("softmax", torch.float16, y, oracle.softmax_packed(x, lens, 2, W.SCALE_BERT),
                 f"{num_req} requests")


@pytest.mark.parametrize("dtype", DT)
def test_length_boundaries_and_max(ttlib, dtype):
    cap = 1024 if dtype == torch.float32 else 2048
    lens = [1, 31, 32, 33, 64, 65, 127, 128, 129, 255, 256, 257, 511, 512, 513, 1000, cap]
    x = _packed_input(lens, 1, dtype, seed=9)
    y = _run(ttlib, x, lens, 1, -0.5, max_seqlen=cap)
    assert_close("softmax", dtype, y, oracle.softmax_packed(x, lens, 1, -0.5), "boundaries")


@pytest.mark.parametrize("dtype", DT)
def test_packed_matches_padded_kernel_bitwise_where_same_tier(ttlib, dtype):
    """Packed and padded kernels share the row body: for a full-length request
    (no padding) both produce identical bits."""
    L, H = 384, 4
    x = _packed_input([L, L], H, dtype, seed=11)
    y = _run(ttlib, x, [L, L], H, W.SCALE_BERT)
    pad = x.reshape(2, H, L, L).cuda()
    ttlib.tt_softmax_masked(pad, torch.tensor([L, L], dtype=torch.int32).cuda(), W.SCALE_BERT)
    torch.cuda.synchronize()
    assert_close("softmax", dtype, y, oracle.softmax_packed(x, [L, L], H, W.SCALE_BERT))
    assert_close("softmax", dtype, pad.reshape(-1), oracle.softmax_packed(x, [L, L], H,
                                                                          W.SCALE_BERT))


def test_packed_deterministic_and_empty(ttlib):
    lens = W.c3_lengths(salt=2)
    x = _packed_input(lens, 12, torch.bfloat16, seed=1)
    a = _run(ttlib, x, lens, 12, W.SCALE_BERT)
    b = _run(ttlib, x, lens, 12, W.SCALE_BERT)
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    # all-empty requests: no-op
    e = torch.empty(0, dtype=torch.float16, device="cuda")
    cu, blocks, total, n = ttlib.packed_offsets([0, 0], 12)
    ttlib.tt_softmax_packed(e, cu, blocks, 12, total, 0, 1.0)
