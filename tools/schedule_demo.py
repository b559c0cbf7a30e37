#!/usr/bin/env python
"""NEXT-4 end to end on a B200: build Alg. 2's cached_cost table by timing this
library's kernels (the paper's warm-up phase), then
schedule the C5 request stream with the DP (tt_dp_schedule) and compare it
with the fixed arrival-order batches of 64 -- predicted cost from the table and
measured device time of running each plan through the kernels.

  python tools/schedule_demo.py > gpurun_out/schedule_demo.json

cost[L][k] = time(softmax [k,12,L,L] + LayerNorm [k*L,768], fp16) / k, measured
on a grid (L every 16 tokens, k in {1,2,4,...,64}) and linearly interpolated
in L and k (the paper's interpolation of the warm-up table, l.873-877).
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2010_05680_b200 as tt  # noqa: E402
import workloads as W  # noqa: E402

H, HID, DT = 12, 768, torch.float16


def graph_time_us(fn, reps=20):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        g.replay()
        a.record(st)
        g.replay()
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


class Step:
    """One padded batch: softmax over [k, H, L, L] + LayerNorm over [k*L, HID]."""

    def __init__(self, maxk, maxL):
        self.sc = torch.randn(maxk * H * maxL * maxL, device="cuda").to(DT)
        d = W.ln_inputs(maxk * maxL, HID, DT, device="cuda")
        self.d = d
        self.out = torch.empty_like(d["x"])
        self.len = torch.empty(maxk, dtype=torch.int32, device="cuda")

    def run(self, lens_dev, k, L):
        s = self.sc[:k * H * L * L].view(k, H, L, L)
        tt.tt_softmax_masked(s, lens_dev[:k], W.SCALE_BERT)
        n = k * L
        tt.tt_add_bias_layernorm(self.out[:n], self.d["x"][:n], self.d["residual"][:n],
                                 self.d["bias"], self.d["gamma"], self.d["beta"], W.EPS_BERT)


def main():
    maxL, maxk = 512, 64
    step = Step(maxk, maxL)
    Ls = list(range(16, maxL + 1, 16))
    ks = [1, 2, 4, 8, 16, 32, 64]
    grid = np.zeros((len(Ls), len(ks)))
    for a, L in enumerate(Ls):
        lens = torch.full((maxk,), L, dtype=torch.int32, device="cuda")
        for b, k in enumerate(ks):
            grid[a, b] = graph_time_us(lambda: step.run(lens, k, L)) / k   # per request
    # dense table by bilinear interpolation (L linear, k linear)
    cost = np.full((maxL + 1, maxk + 1), np.nan)
    Lg, kg = np.array(Ls, float), np.array(ks, float)
    for k in range(1, maxk + 1):
        col = np.array([np.interp(k, kg, grid[a]) for a in range(len(Ls))])
        cost[1:, k] = np.interp(np.arange(1, maxL + 1), Lg, col)

    stream = np.concatenate(W.c5_stream())
    window = 64
    fixed = [list(range(i, i + window)) for i in range(0, len(stream), window)]
    dp_plans = []
    for i in range(0, len(stream), window):   # the queue content at each trigger
        plans, _ = tt.dp_schedule(stream[i:i + window], cost)
        dp_plans += [[i + j for j in b] for b in plans]

    def measure(plans):
        tot = 0.0
        for b in plans:
            L = int(stream[b].max())
            lens = torch.as_tensor(stream[b].astype(np.int32)).cuda()
            tot += graph_time_us(lambda: step.run(lens, len(b), L), reps=5)
        return tot

    res = {
        "cost_grid_us_per_request": {"L": Ls, "k": ks, "values": grid.round(3).tolist()},
        "stream": "C5: 4096 requests U{5..500}, scheduled per 64-request queue window",
        "fixed_batches": len(fixed),
        "dp_batches": len(dp_plans),
        "predicted_us": {"fixed": round(tt.schedule_cost(stream, cost, fixed), 1),
                         "dp": round(tt.schedule_cost(stream, cost, dp_plans), 1)},
        "measured_us": {"fixed": round(measure(fixed), 1), "dp": round(measure(dp_plans), 1)},
        "padded_tokens": {"fixed": int(sum(len(b) * stream[b].max() for b in fixed)),
                          "dp": int(sum(len(b) * stream[b].max() for b in dp_plans)),
                          "valid": int(stream.sum())},
    }
    print(json.dumps(res))


if __name__ == "__main__":
    main()
