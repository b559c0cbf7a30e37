#!/usr/bin/env python
"""Time every compiled tier (include/tt_tune.h) on one shape; prints JSON lines.

  python tools/tune.py softmax bf16 64 16 512 512      # B H Sq Sk (all keys valid)
  python tools/tune.py layernorm bf16 32768 1024       # rows hidden

Inputs are larger than L2 for the headline shapes; smaller shapes rotate over
enough buffers to exceed 4x L2.  CUDA events on the launching stream.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# every tuning candidate lives in the TT_TUNING build (paper_2010_05680_b200/build.py --tuning)
if "TT_LIB_PATH" not in os.environ:
    from paper_2010_05680_b200 import build as _b  # noqa: E402
    os.environ["TT_LIB_PATH"] = _b.build(tuning=True)
import paper_2010_05680_b200 as tt  # noqa: E402
import workloads as W  # noqa: E402

L2 = 126 * 1024 * 1024


def timeit(fn, nbufs, reps=50, warm=5):
    """ms per call: the calls are captured once into a CUDA graph and replayed,
    so host launch overhead (Python + ctypes) does not inflate small shapes;
    CUDA events on the replay stream."""
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
    op, dt = sys.argv[1], W.DTYPES[sys.argv[2]]
    dims = [int(v) for v in sys.argv[3:]]
    ragged = os.environ.get("RAGGED", "0") != "0"  # "1": U{1..Sk} draws; "c3": BASELINE C3 lengths
    e = W.ELEM_BYTES[dt]
    names = tt.tiers(op, dt)
    only = os.environ.get("ONLY")
    if op == "softmax":
        B, H, Sq, Sk = dims
        if os.environ.get("RAGGED") == "c3":
            lens = W.c3_lengths()
            B, Sk = len(lens), int(lens.max())
            dims = [B, H, Sk, Sk]
        else:
            lens = W.lengths_ragged(B, Sk) if ragged else W.lengths_full(B, Sk)
        nbytes = B * H * Sq * Sk * e
        nbufs = max(1, -(-4 * L2 // nbytes))
        bufs = [W.scores(B, H, Sq, Sk, dt, device="cuda", seed=i) for i in range(nbufs)]
        L = torch.as_tensor(lens).cuda()
        alg = W.softmax_bytes_alg(lens, H, Sq, Sk, e)
        fn = lambda i: tt.tt_softmax_masked(bufs[i], L, 0.125)  # noqa: E731
        plan = tt.softmax_plan(dt, B, H, Sq, Sk)
    else:
        rows, hidden = dims
        nbytes = 3 * rows * hidden * e
        nbufs = max(1, -(-4 * L2 // nbytes))
        ds = [W.ln_inputs(rows, hidden, dt, device="cuda", seed=i) for i in range(nbufs)]
        outs = [torch.empty_like(d["x"]) for d in ds]
        alg = W.ln_bytes_alg(rows, hidden, e)
        fn = lambda i: tt.tt_add_bias_layernorm(outs[i], ds[i]["x"], ds[i]["residual"],  # noqa
                                                ds[i]["bias"], ds[i]["gamma"], ds[i]["beta"], 1e-12)
        plan = tt.layernorm_plan(dt, rows, hidden)
    # same-traffic streaming reference (not our kernel): an SM element-wise
    # kernel -- torch.neg for softmax (1 read + 1 write; a D2D copy_ would be a
    # copy-engine memcpy inside the graph), torch add for LN (2 reads + 1 write)
    if op == "softmax":
        other = [torch.empty_like(b) for b in bufs]
        ref = lambda i: torch.neg(bufs[i], out=other[i])  # noqa: E731
        ref_bytes = 2 * bufs[0].numel() * e
    else:
        ref = lambda i: torch.add(ds[i]["x"], ds[i]["residual"], out=outs[i])  # noqa: E731
        ref_bytes = 3 * rows * hidden * e
    ms = timeit(ref, nbufs)
    print(json.dumps({"op": op, "dtype": sys.argv[2], "dims": dims, "ragged": ragged,
                      "tier": "torch-" + ("neg" if op == "softmax" else "add") + " (same traffic)",
                      "auto": False, "us": round(ms * 1e3, 2),
                      "GBps": round(ref_bytes / ms / 1e6, 1)}), flush=True)
    for i, name in enumerate([None] + names):
        if only and name and only not in name:
            continue
        tt.force_tier(op, dt, i - 1)
        chosen = tt.softmax_plan(dt, *dims) if op == "softmax" else tt.layernorm_plan(dt, *dims)
        if name is not None and chosen != name:
            continue  # tier cannot serve this shape
        ms = timeit(fn, nbufs)
        print(json.dumps({"op": op, "dtype": sys.argv[2], "dims": dims, "ragged": ragged,
                          "tier": chosen, "auto": name is None or name == plan,
                          "us": round(ms * 1e3, 2), "GBps": round(alg / ms / 1e6, 1)}), flush=True)
    tt.force_tier(op, dt, -1)


if __name__ == "__main__":
    main()
