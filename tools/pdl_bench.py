#!/usr/bin/env python
"""Launch-bound shapes: device time per softmax + LayerNorm step with
programmatic dependent launch on and off (include/tt_tune.h ttx_set_pdl).

SURVEY §8(d) C1/C2: "report µs/call vs an empty-kernel floor and the
CUDA-graph/PDL latency".  Each case captures REPS steps (softmax in place, then
LN reading the previous step's LN output, so the chain is dependent) into one
CUDA graph and times a replay with CUDA events on the replay stream.  The floor
is the same number of torch's smallest kernel (a 1-element add) per step pair.

  python tools/pdl_bench.py [--reps 200]      -> JSON lines
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2010_05680_b200 as tt  # noqa: E402
import workloads as W  # noqa: E402


def graph_us(fn, reps):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            fn()
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            g.replay()
            b.record(st)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / reps)
    return best


def case(name, dtype, B, H, S, rows, reps, lens=None):
    lens = W.lengths_full(B, S) if lens is None else lens
    x = W.scores(B, H, S, S, dtype, device="cuda", seed=1)
    L = torch.as_tensor(lens).cuda()
    d = W.ln_inputs(rows, 768, dtype, device="cuda", seed=1)
    o = [torch.empty_like(d["x"]) for _ in range(2)]
    state = {"i": 0}

    def step():
        tt.tt_softmax_masked(x, L, W.SCALE_BERT)
        i = state["i"]
        src = d["x"] if i == 0 else o[(i + 1) % 2]
        tt.tt_add_bias_layernorm(o[i % 2], src, d["residual"], d["bias"], d["gamma"], d["beta"],
                                 W.EPS_BERT)
        state["i"] = i + 1

    out = {"case": name, "dtype": str(dtype).split(".")[-1], "softmax": [B, H, S, S],
           "ln": [rows, 768],
           "softmax_tier": tt.softmax_plan(dtype, B, H, S, S),
           "ln_tier": tt.layernorm_plan(dtype, rows, 768)}
    for pdl in (False, True):
        tt.set_pdl(pdl)
        state["i"] = 0
        out["us_per_step_pdl" if pdl else "us_per_step"] = round(graph_us(step, reps), 3)
    tt.set_pdl(True)
    out["pdl_gain"] = round(out["us_per_step"] / out["us_per_step_pdl"], 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    z = torch.zeros(1, device="cuda")
    floor2 = graph_us(lambda: (z.add_(0), z.add_(0)), a.reps)
    print(json.dumps({"floor_us_per_2_kernels": round(floor2, 3),
                      "what": "torch 1-element add x2 per step in a CUDA graph (no PDL)"}),
          flush=True)
    print(json.dumps(case("C1 BERT-base b1 s40", torch.float32, 1, 12, 40, 40, a.reps)), flush=True)
    for S in (10, 20, 40, 64, 100, 128):
        print(json.dumps(case(f"C2 b20 s{S}", torch.float16, 20, 12, S, 20 * S, a.reps)),
              flush=True)
    lens = np.array([S for S in W.lengths_ragged(20, 64)], dtype=np.int32)
    print(json.dumps(case("C2 b20 s64 ragged", torch.float16, 20, 12, 64, 20 * 64, a.reps, lens)),
          flush=True)


if __name__ == "__main__":
    main()
