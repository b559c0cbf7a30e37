#!/usr/bin/env python
"""Quick A/B of attention variants on the BERT shapes (CUDA-graph replay,
inputs rotated over > 4x L2):  python tools/attn_quick.py [variant ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2010_05680_b200 as tt  # noqa: E402
import workloads as W  # noqa: E402

L2 = 126 << 20


def timeit(fn, nbufs, reps=20, warm=3):
    """ms per call from a CUDA-graph replay (CUDA events on the replay stream)."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(warm):
            fn(i % nbufs)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(reps):
            fn(i % nbufs)
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        g.replay()
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    variants = [int(v) for v in sys.argv[1:]] or [0, 9]
    cases = [("C4", 64, 16, 512, torch.bfloat16, W.lengths_full(64, 512)),
             ("C4 ragged", 64, 16, 512, torch.bfloat16, W.lengths_ragged(64, 512, 4)),
             ("C2 s500", 20, 12, 500, torch.float16, W.lengths_full(20, 500)),
             ("C3", 64, 12, int(W.c3_lengths().max()), torch.float16, W.c3_lengths())]
    for name, B, H, S, dt, lens in cases:
        nbytes = 4 * B * H * S * 64 * 2
        nb = max(1, min(8, -(-4 * L2 // nbytes)))
        g = torch.Generator(device="cuda").manual_seed(0)
        qkv = [[torch.randn(B, H, S, 64, device="cuda", dtype=dt, generator=g) for _ in range(3)]
               for _ in range(nb)]
        outs = [torch.empty(B, H, S, 64, device="cuda", dtype=dt) for _ in range(nb)]
        L = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        flops = 4.0 * H * S * float(np.sum(np.minimum(lens, S))) * 64
        res = {"case": name}
        for v in variants:
            tt.attention_variant(v)
            ms = timeit(lambda i: tt.tt_attention_fwd(outs[i], *qkv[i], L, 0.125), nb, reps=20)
            res[f"v{v}_us"] = round(ms * 1e3, 2)
            res[f"v{v}_tflops"] = round(flops / ms / 1e9, 1)
        tt.attention_variant(0)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
