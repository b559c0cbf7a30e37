#!/usr/bin/env python
"""Run one op N times with an optional forced tier -- a small target for ncu.

  python tools/prof_one.py softmax bf16 64 16 512 512 [--tier NAME] [--reps 5]
  python tools/prof_one.py layernorm bf16 32768 1024 [--tier NAME]
  python tools/prof_one.py attention bf16 64 16 512 [--tier 1|2]   (B H S; tier = K/V buffering)
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2010_05680_b200 as tt  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("op")
    ap.add_argument("dtype")
    ap.add_argument("dims", nargs="+", type=int)
    ap.add_argument("--tier", default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ragged", action="store_true")
    ap.add_argument("--c3", action="store_true", help="C3 lengths (64 x U{5..500}); dims = H")
    a = ap.parse_args()
    dt = W.DTYPES[a.dtype]
    if a.tier and a.op != "attention":
        names = tt.tiers(a.op, dt)
        tt.force_tier(a.op, dt, names.index(a.tier))
    if a.op == "attention":
        B, H, S = a.dims
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v = [torch.randn(B, H, S, 64, device="cuda", dtype=dt, generator=g)
                   for _ in range(3)]
        o = torch.empty_like(q)
        lens = W.lengths_ragged(B, S) if a.ragged else W.lengths_full(B, S)
        L = torch.as_tensor(lens).cuda()
        if a.tier:
            tt.attention_variant(int(a.tier))
        for _ in range(a.reps):
            tt.tt_attention_fwd(o, q, k, v, L, 0.125)
    elif a.op == "packed":  # C3 lengths, dims = H: the padding-free layout (NEXT-1)
        lens = W.c3_lengths()
        H = a.dims[0]
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        blk = np.concatenate([[0], np.cumsum(H * lens.astype(np.int64) ** 2)]).astype(np.int64)
        x = W.scores(1, 1, 1, int(blk[-1]), dt, device="cuda").reshape(-1)
        cu_d, blk_d = torch.as_tensor(cu).cuda(), torch.as_tensor(blk[:-1]).cuda()
        print("tier:", tt.softmax_packed_plan(dt, int(lens.max())))
        for _ in range(a.reps):
            tt.tt_softmax_packed(x, cu_d, blk_d, H, int(cu[-1]), int(lens.max()), 0.125)
    elif a.op == "softmax":
        if a.c3:
            lens = W.c3_lengths()
            B, H, Sq, Sk = len(lens), a.dims[0], int(lens.max()), int(lens.max())
        else:
            B, H, Sq, Sk = a.dims
            lens = W.lengths_ragged(B, Sk) if a.ragged else W.lengths_full(B, Sk)
        x = W.scores(B, H, Sq, Sk, dt, device="cuda")
        L = torch.as_tensor(lens).cuda()
        print("tier:", tt.softmax_plan(dt, B, H, Sq, Sk))
        for _ in range(a.reps):
            tt.tt_softmax_masked(x, L, 0.125)
    else:
        rows, hidden = a.dims
        d = W.ln_inputs(rows, hidden, dt, device="cuda")
        out = torch.empty_like(d["x"])
        print("tier:", tt.layernorm_plan(dt, rows, hidden))
        for _ in range(a.reps):
            tt.tt_add_bias_layernorm(out, d["x"], d["residual"], d["bias"], d["gamma"], d["beta"],
                                     1e-12)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
