#!/usr/bin/env python
"""Timing of the long-row softmax tier (rows beyond 131 072 keys): device time
per call (CUDA events over 10 calls on rotated buffers), algorithmic GB/s
(valid-prefix read + full-row write) and % of the measured copy peak."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2010_05680_b200 as tt  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6549.4)
cases = [(torch.bfloat16, 256, 262144, 1.0), (torch.bfloat16, 256, 262144, 0.5),
         (torch.bfloat16, 64, 1 << 20, 1.0), (torch.float32, 64, 1 << 20, 1.0),
         (torch.float16, 1024, 131073, 1.0)]
names = {}
for dt in (torch.bfloat16, torch.float16, torch.float32):
    names[dt] = [(i, n) for i, n in enumerate(tt.tiers("softmax", dt)) if n.startswith("softmax_long<")]
for (dt, rows, Sk, frac), (ti, tn) in [(c, t) for c in cases for t in names[c[0]]]:
    tt.force_tier("softmax", dt, ti)
    e = torch.tensor([], dtype=dt).element_size()
    nb = max(2, -(-4 * (126 << 20) // (rows * Sk * e)))
    xs = [torch.randn(rows, 1, 1, Sk, device="cuda", dtype=dt) for _ in range(nb)]
    L = torch.full((rows,), int(Sk * frac), dtype=torch.int32, device="cuda")
    for i in range(3):
        tt.tt_softmax_masked(xs[i % nb], L, 0.125)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a.record()
    for i in range(reps):
        tt.tt_softmax_masked(xs[i % nb], L, 0.125)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / reps * 1e3
    alg = rows * (int(Sk * frac) + Sk) * e + rows * 4
    print(json.dumps({"dtype": str(dt).split(".")[-1], "rows": rows, "Sk": Sk, "valid_frac": frac,
                      "tier": tn, "us": round(us, 2),
                      "GBps": round(alg / us / 1e3, 1), "pct_peak": round(100 * alg / us / 1e3 / PEAK, 1)}))
    tt.force_tier("softmax", dt, -1)
