#!/usr/bin/env python
"""Small invocations of every kernel family for compute-sanitizer (SURVEY §5
race / memory checking): C1, C2 S in {10, 37, 40} full and ragged, one
32 768-key row, rows of odd pitch with 16-B-but-not-32-B aligned bases, the
packed kernel, the element-wise kernels, the fused attention, LayerNorm on
every automatic band, and (with TT_LIB_PATH=libtt_tune.so) the TMA-ring
tuning candidates.

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2010_05680_b200 as tt  # noqa: E402
import workloads as W  # noqa: E402

dev = "cuda"


def sm(dtype, B, H, Sq, Sk, lens, offset_elems=0, tier=None):
    n = B * H * Sq * Sk
    buf = W.scores(1, 1, 1, n + offset_elems, dtype, device=dev, seed=Sk).reshape(-1)
    x = buf[offset_elems:].view(B, H, Sq, Sk)
    L = torch.as_tensor(np.asarray(lens, dtype=np.int32)).to(dev)
    if tier is not None:
        tt.force_tier("softmax", dtype, tier)
    tt.tt_softmax_masked(x, L, 0.125)
    tt.force_tier("softmax", dtype, -1)


def ln(dtype, rows, hidden, tier=None):
    d = W.ln_inputs(rows, hidden, dtype, device=dev, seed=hidden)
    out = torch.empty_like(d["x"])
    if tier is not None:
        tt.force_tier("layernorm", dtype, tier)
    tt.tt_add_bias_layernorm(out, d["x"], d["residual"], d["bias"], d["gamma"], d["beta"], 1e-12)
    tt.force_tier("layernorm", dtype, -1)


def main():
    DT = (torch.float32, torch.float16, torch.bfloat16)
    # C1, C2 small seqs, full and ragged
    sm(torch.float32, 1, 12, 40, 40, [40])
    ln(torch.float32, 40, 768)
    for dtype in DT:
        for S in (10, 37, 40):
            sm(dtype, 20, 12, S, S, W.lengths_full(20, S))
            sm(dtype, 20, 12, S, S, W.lengths_ragged(20, S))
            ln(dtype, 20 * S, 768)
        # a 32 768-key row (CTA tier) and odd pitches off 16-B-but-not-32-B bases
        sm(dtype, 2, 1, 1, 32768, [32768, 20000])
        sm(dtype, 3, 1, 1, 40003, [40003, 16385, 5])   # cluster tier: 3 CTAs per row
        sm(dtype, 3, 1, 1, 140003, [140003, 17505, 0])   # long tier: 8 CTAs per row, two passes
        for Sk in (37, 491, 1000):
            sm(dtype, 3, 2, 3, Sk, [Sk, Sk // 2, 0], offset_elems=16 // W.ELEM_BYTES[dtype])
        # every automatic LayerNorm band at hidden 768 / 1024 and odd hidden
        for rows in (40, 700, 1500, 5000, 20000):
            ln(dtype, rows, 768)
        ln(dtype, 3000, 1024)
        ln(dtype, 37, 1000)
        ln(dtype, 5, 4099 if dtype == torch.float32 else 4098)
        # every compiled tier (the TT_TUNING build adds the TMA rings)
        for i, name in enumerate(tt.tiers("softmax", dtype)):
            for Sk in (37, 512, 2100):
                tt.force_tier("softmax", dtype, i)
                ok = tt.softmax_plan(dtype, 1, 1, 1, Sk) == name
                tt.force_tier("softmax", dtype, -1)
                if ok:
                    sm(dtype, 3, 2, 5, Sk, [Sk, Sk // 3, 1], tier=i)
        for i, name in enumerate(tt.tiers("layernorm", dtype)):
            for h in (768, 1024, 96):
                tt.force_tier("layernorm", dtype, i)
                ok = tt.layernorm_plan(dtype, 300, h) == name
                tt.force_tier("layernorm", dtype, -1)
                if ok:
                    ln(dtype, 300, h, tier=i)
                    break
        # packed (NEXT-1)
        lens = [5, 17, 64, 1, 130]
        cu, blocks, total, nel = tt.packed_offsets(lens, 2, device=dev)
        xp = W.scores(1, 1, 1, nel, dtype, device=dev, seed=3).reshape(-1)
        tt.tt_softmax_packed(xp, cu, blocks, 2, total, max(lens), 0.125)
        # element-wise (NEXT-2)
        x = W.scores(1, 1, 37, 3 * 2 * 64, dtype, device=dev, seed=4).reshape(37, 384)
        tt.tt_add_bias_gelu(torch.empty_like(x), x, torch.zeros(384, dtype=dtype, device=dev))
        q, k, v = (torch.empty(1, 2, 37, 64, dtype=dtype, device=dev) for _ in range(3))
        tt.tt_split_qkv_add_bias(q, k, v, x, torch.zeros(384, dtype=dtype, device=dev), 1, 37, 2, 64)
        tt.tt_merge_heads(torch.empty(37, 128, dtype=dtype, device=dev), q, 1, 37, 2, 64)
    # fused attention (NEXT-3), every compiled variant
    for dtype in (torch.float16, torch.bfloat16):
        g = torch.Generator(device=dev).manual_seed(0)
        q, k, v = (torch.randn(3, 2, 200, 64, device=dev, dtype=dtype, generator=g) for _ in range(3))
        L = torch.tensor([200, 77, 0], dtype=torch.int32, device=dev)
        for var in [0] + tt.attention_variants():
            tt.attention_variant(var)
            tt.tt_attention_fwd(torch.empty_like(q), q, k, v, L, 0.125)
        tt.attention_variant(0)
    torch.cuda.synchronize()
    print("sanitize cases done (tuning build)" if tt.tuning_build() else "sanitize cases done")


if __name__ == "__main__":
    main()
