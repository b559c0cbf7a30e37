#!/usr/bin/env python
"""NEXT-3 measurement: tt_attention_fwd (tcgen05 fused masked attention) vs the
unfused path it replaces (cuBLAS QK^T -> tt_softmax_masked -> cuBLAS PV) and
torch SDPA, on BERT shapes.  Device time by CUDA events over back-to-back
calls (inputs rotated over > 4x L2).  JSON lines.

  python tools/attn_bench.py > gpurun_out/attn_bench.jsonl
"""
import json
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# the non-default variants live in the TT_TUNING build (paper_2010_05680_b200/build.py --tuning)
if "TT_LIB_PATH" not in os.environ:
    from paper_2010_05680_b200 import build as _b  # noqa: E402
    os.environ["TT_LIB_PATH"] = _b.build(tuning=True)
import paper_2010_05680_b200 as tt  # noqa: E402
import workloads as W  # noqa: E402

L2 = 126 << 20


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["bf16_tflops"]), float(d["hbm_gbs"])
    except Exception:
        return 1590.0, 6650.0


def timeit(fn, nb, reps=20):
    for i in range(3):
        fn(i % nb)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps):
        fn(i % nb)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def case(name, B, H, S, dtype, lens):
    D = 64
    tf, hbm = peaks()
    nbytes = 4 * B * H * S * D * 2
    nb = max(1, min(8, -(-4 * L2 // nbytes)))
    qkv = [[torch.randn(B, H, S, D, device="cuda", dtype=dtype) for _ in range(3)]
           for _ in range(nb)]
    outs = [torch.empty(B, H, S, D, device="cuda", dtype=dtype) for _ in range(nb)]
    L = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
    var_us = {v: float("nan") for v in range(1, 11)}
    for v in tt.attention_variants():
        tt.attention_variant(v)
        var_us[v] = timeit(lambda i: tt.tt_attention_fwd(outs[i], *qkv[i], L, 0.125), nb)
    tt.attention_variant(0)
    us = timeit(lambda i: tt.tt_attention_fwd(outs[i], *qkv[i], L, 0.125), nb)
    valid = float(np.sum(np.minimum(lens, S)))
    flops = 4.0 * H * S * valid * D            # QK^T and PV over the valid keys
    res = dict(case=name, shape=[B, H, S, D], dtype=W.DTYPE_NAMES[dtype], us=round(us, 2),
               tflops=round(flops / us / 1e6, 1), frac_bf16_peak=round(flops / us / 1e6 / tf, 3),
               hbm_GBps=round(nbytes / us / 1e3, 1), frac_hbm=round(nbytes / us / 1e3 / hbm, 3),
               bn128_us=round(var_us[1], 2), bn128x2_us=round(var_us[2], 2),
               bn64_us=round(var_us[3], 2), bn64x2_us=round(var_us[4], 2),
               ws_us=round(var_us[5], 2), split_us=round(var_us[6], 2),
               split3_us=round(var_us[7], 2), late_us=round(var_us[8], 2),
               fa_us=round(var_us[9], 2), fa64_us=round(var_us[10], 2))
    # unfused: QK^T (cuBLAS), masked softmax (ours, in place), PV (cuBLAS)
    sc = torch.empty(B, H, S, S, device="cuda", dtype=dtype)

    def unfused(i):
        q, k, v = qkv[i]
        torch.matmul(q, k.transpose(-1, -2), out=sc)
        tt.tt_softmax_masked(sc, L, 0.125)
        torch.matmul(sc, v, out=outs[i])
    res["unfused_us"] = round(timeit(unfused, nb), 2)
    mask = (torch.arange(S, device="cuda")[None, :] < L[:, None])[:, None, None, :]
    res["torch_sdpa_us"] = round(timeit(
        lambda i: F.scaled_dot_product_attention(*qkv[i], attn_mask=mask, scale=0.125), nb), 2)
    return res


def main():
    cases = [("C4 BERT-large b64 s512", 64, 16, 512, torch.bfloat16, [512] * 64),
             ("C4 ragged", 64, 16, 512, torch.bfloat16, W.lengths_ragged(64, 512, 4)),
             ("C2 BERT-base b20 s500", 20, 12, 500, torch.float16, [500] * 20),
             ("C2 BERT-base b20 s128", 20, 12, 128, torch.float16, [128] * 20),
             ("C3 64 req U{5..500}", 64, 12, int(W.c3_lengths().max()), torch.float16,
              W.c3_lengths())]
    for c in cases:
        print(json.dumps(case(*c)), flush=True)


if __name__ == "__main__":
    main()
