"""Programmatic dependent launch (include/tt_tune.h ttx_set_pdl).

Every kernel starts with griddepcontrol.wait before any global access, so a
chain of DEPENDENT calls (each reading what the previous one wrote) must give
the same bytes with PDL on and off, and match the oracle applied in sequence.
The chains below are launch-bound on purpose (C1-sized calls back to back,
also inside a CUDA graph), which is where the next kernel actually launches
early.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from _parity import assert_close


def test_set_pdl_validates(ttlib):
    L = ttlib.lib()
    assert L.ttx_set_pdl(2) == ttlib.TT_ERROR_INVALID_VALUE
    assert L.ttx_set_pdl(-1) == ttlib.TT_ERROR_INVALID_VALUE
    old = ttlib.get_pdl()
    try:
        ttlib.set_pdl(False)
        assert ttlib.get_pdl() is False
        ttlib.set_pdl(True)
        assert ttlib.get_pdl() is True
    finally:
        ttlib.set_pdl(old)


def _ln_chain(tt, d, n, eps):
    """x_{i+1} = LN(x_i + bias + residual) n times, each call reading the last output."""
    cur = d["x"]
    outs = []
    for _ in range(n):
        o = torch.empty_like(cur)
        tt.tt_add_bias_layernorm(o, cur, d["residual"], d["bias"], d["gamma"], d["beta"], eps)
        outs.append(o)
        cur = o
    return outs


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_dependent_chain_pdl_on_off_identical(ttlib, dtype):
    """Softmax in place 8 times, then an 8-deep LN chain: bitwise equal with PDL
    on and off, and equal to the oracle applied step by step (rounded to the
    storage dtype between steps, as the kernels do)."""
    lens = np.array([40, 23], dtype=np.int32)
    x0 = W.scores(2, 12, 40, 40, dtype, seed=W.SEED + 11)
    d0 = W.ln_inputs(40, 768, dtype, seed=W.SEED + 11)
    res = {}
    old = ttlib.get_pdl()
    try:
        for pdl in (False, True):
            ttlib.set_pdl(pdl)
            y = x0.cuda()
            L = torch.as_tensor(lens).cuda()
            for _ in range(8):
                ttlib.tt_softmax_masked(y, L, W.SCALE_BERT)
            dd = {k: v.cuda() for k, v in d0.items()}
            outs = _ln_chain(ttlib, dd, 8, W.EPS_BERT)
            torch.cuda.synchronize()
            res[pdl] = (y.cpu(), [o.cpu() for o in outs])
    finally:
        ttlib.set_pdl(old)
    assert torch.equal(res[False][0].view(torch.uint8), res[True][0].view(torch.uint8))
    for a, b in zip(res[False][1], res[True][1]):
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))
    # oracle, step by step
    ref = x0
    for _ in range(8):
        ref = oracle.softmax_masked(ref, lens, W.SCALE_BERT).to(dtype)
    assert_close("softmax", dtype, res[True][0], ref.double(), "pdl softmax chain")
    cur = d0["x"]
    for i in range(8):
        r = oracle.add_bias_layernorm(cur, d0["residual"], d0["bias"], d0["gamma"], d0["beta"],
                                      W.EPS_BERT)
        # compare step i against the oracle fed the kernel's own step i-1 output
        assert_close("layernorm", dtype, res[True][1][i], r, f"pdl ln chain step {i}")
        cur = res[True][1][i]


@pytest.mark.gpu
def test_dependent_chain_in_cuda_graph(ttlib):
    """The same dependent LN chain captured in a CUDA graph (programmatic edges)
    and replayed: identical to eager execution."""
    dtype = torch.float16
    d0 = {k: v.cuda() for k, v in W.ln_inputs(40, 768, dtype, seed=W.SEED + 12).items()}
    eager = _ln_chain(ttlib, d0, 6, W.EPS_BERT)
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    bufs = [torch.empty_like(d0["x"]) for _ in range(6)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        cur = d0["x"]
        for o in bufs:
            ttlib.tt_add_bias_layernorm(o, cur, d0["residual"], d0["bias"], d0["gamma"],
                                        d0["beta"], W.EPS_BERT)
            cur = o
    for b in bufs:
        b.zero_()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, bufs):
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))


def test_every_kernel_opens_with_pdl_scope():
    """Static check of the PDL invariant (include/tt.h Execution): every
    __global__ function in csrc/ starts with `PdlScope pdl_;` (griddepcontrol.wait
    before any global access), and every launch goes through launch_k."""
    import glob
    import os
    import re
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_2010_05680_b200", "csrc")
    n = 0
    for f in glob.glob(os.path.join(root, "*.cu")) + glob.glob(os.path.join(root, "*.cuh")):
        src = open(f).read()
        assert "<<<" not in src, f"{f}: raw <<<>>> launch bypasses launch_k (PDL attribute)"
        for m in re.finditer(r"__global__", src):
            body = src.index(") {\n", m.start()) + 4
            first = src[body:src.index("\n", body)].strip()
            assert first.startswith("PdlScope pdl_;"), (f, first)
            n += 1
    assert n >= 12


def _variants():
    try:  # the default, plus the warp-specialised / split-row schedules of the tuning build
        import paper_2010_05680_b200 as tt
        return [0] + [v for v in (5, 6) if v in tt.attention_variants()]
    except Exception:
        return [0]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", _variants())
def test_attention_block_chain_pdl_on_off_identical(ttlib, variant):
    """A whole dependent BERT attention block through the library, every kernel
    reading what the previous one wrote: QKV split + bias -> fused attention
    (tcgen05) -> head merge -> add-bias LayerNorm (residual) -> add-bias GELU.
    Bitwise identical with PDL on and off, for the default, warp-specialised
    and split-row attention schedules."""
    dtype = torch.bfloat16
    B, S, H, D = 3, 200, 4, 64
    g = torch.Generator(device="cuda").manual_seed(7)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda", dtype=dtype, generator=g)
    bqkv = torch.randn(3 * H * D, device="cuda", dtype=dtype, generator=g) * 0.1
    res = torch.randn(B * S, H * D, device="cuda", dtype=dtype, generator=g)
    bo, gam, bet = (torch.randn(H * D, device="cuda", dtype=dtype, generator=g) * 0.1
                    for _ in range(3))
    gam = gam + 1
    lens = torch.tensor([200, 77, 1], dtype=torch.int32, device="cuda")
    outs = {}
    old = ttlib.get_pdl()
    try:
        ttlib.attention_variant(variant)
        for pdl in (False, True):
            ttlib.set_pdl(pdl)
            q, k, v = (torch.empty(B, H, S, D, device="cuda", dtype=dtype) for _ in range(3))
            ttlib.tt_split_qkv_add_bias(q, k, v, qkv, bqkv, B, S, H, D)
            o = torch.empty_like(q)
            ttlib.tt_attention_fwd(o, q, k, v, lens, 0.125)
            m = torch.empty(B * S, H * D, device="cuda", dtype=dtype)
            ttlib.tt_merge_heads(m, o, B, S, H, D)
            ln = torch.empty_like(m)
            ttlib.tt_add_bias_layernorm(ln, m, res, bo, gam, bet, 1e-12)
            y = torch.empty_like(ln)
            ttlib.tt_add_bias_gelu(y, ln, bo)
            torch.cuda.synchronize()
            outs[pdl] = y.cpu()
    finally:
        ttlib.set_pdl(old)
        ttlib.attention_variant(0)
    assert torch.isfinite(outs[True].float()).all()
    assert torch.equal(outs[False].view(torch.int16), outs[True].view(torch.int16))


_FRESH_CAPTURE = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2010_05680_b200 as tt, workloads as W, oracle
# the library's first calls happen INSIDE a stream capture: the per-kernel
# occupancy query (rows per group, softmax.cu) and the dynamic-smem opt-in
# must be legal there
lens = np.array([100, 37, 64, 1], dtype=np.int32)
x = W.scores(4, 12, 100, 100, torch.float16, seed=3)
y = x.cuda()
L = torch.as_tensor(lens).cuda()
d = W.ln_inputs(4000, 768, torch.float16, seed=4)
dd = {k: v.cuda() for k, v in d.items()}
out = torch.empty_like(dd["x"])
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    tt.tt_softmax_masked(y, L, 0.125)
    tt.tt_add_bias_layernorm(out, dd["x"], dd["residual"], dd["bias"], dd["gamma"], dd["beta"], 1e-12)
y.copy_(x.cuda())
g.replay()
torch.cuda.synchronize()
ref = oracle.softmax_masked(x, lens, 0.125)
assert (y.cpu().double() - ref).abs().max().item() < 2e-3
refl = oracle.add_bias_layernorm(d["x"], d["residual"], d["bias"], d["gamma"], d["beta"], 1e-12)
assert (out.cpu().double() - refl).abs().max().item() < 2e-2
print("ok")
"""


@pytest.mark.gpu
def test_first_calls_inside_graph_capture():
    """A fresh process whose first library calls are captured into a CUDA graph."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _FRESH_CAPTURE, root], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
