#!/usr/bin/env python
"""Per-config evidence for BASELINE.md §4 (companion of tools/sweep.py).

  --ncu     run every (config, op, dtype, lengths) case of the sweep ONCE, in the
            sweep's order, so `ncu --metrics dram__bytes_read.sum,
            dram__bytes_write.sum,gpu__time_duration.sum -k regex:"softmax_|ln_"`
            gives one launch per case (DRAM bytes and duration per case);
  --oracle  time the fp64 oracle on a bounded sample of every case, on one
            host thread and on all of them (rows/s).
Prints one JSON line per case."""
import concurrent.futures as cf
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402


def cases():
    out = [("C1", "softmax", torch.float32, (1, 12, 40), [40]), ("C1", "layernorm", torch.float32, (40, 768), None)]
    for dt in (torch.float16, torch.float32):
        for S in W.C2.extra["seqs"]:
            out.append(("C2", "softmax", dt, (20, 12, S), W.lengths_full(20, S)))
            out.append(("C2", "softmax", dt, (20, 12, S), W.lengths_ragged(20, S)))
            out.append(("C2", "layernorm", dt, (20 * S, 768), None))
    for dt in (torch.float16, torch.float32):
        lens = W.c3_lengths()
        S = int(lens.max())
        out.append(("C3", "softmax", dt, (64, 12, S), lens))
        out.append(("C3", "layernorm", dt, (64 * S, 768), None))
    out.append(("C4", "softmax", torch.bfloat16, (64, 16, 512), W.lengths_full(64, 512)))
    out.append(("C4", "softmax", torch.bfloat16, (64, 16, 512), W.lengths_ragged(64, 512, 4)))
    out.append(("C4", "layernorm", torch.bfloat16, (32768, 1024), None))
    return out


def key(c):
    cfg, op, dt, shp, lens = c
    ragged = lens is not None and bool(np.any(np.asarray(lens) < shp[2]))
    shape = [shp[0], shp[1], shp[2], shp[2]] if op == "softmax" else list(shp)
    return dict(config=cfg, op=op, dtype=W.DTYPE_NAMES[dt], shape=shape, ragged=ragged)


def run_ncu():
    import paper_2010_05680_b200 as tt
    for c in cases():
        cfg, op, dt, shp, lens = c
        if op == "softmax":
            B, H, S = shp
            x = W.scores(B, H, S, S, dt, device="cuda", seed=1)
            L = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
            torch.cuda.synchronize()
            tt.tt_softmax_masked(x, L, 0.125)
        else:
            d = W.ln_inputs(*shp, dt, device="cuda", seed=1)
            o = torch.empty_like(d["x"])
            torch.cuda.synchronize()
            tt.tt_add_bias_layernorm(o, d["x"], d["residual"], d["bias"], d["gamma"], d["beta"], 1e-12)
        torch.cuda.synchronize()
        print(json.dumps(key(c)), flush=True)


def run_oracle(budget_rows=20000):
    import oracle
    cores = os.cpu_count() or 1
    for c in cases():
        cfg, op, dt, shp, lens = c
        if op == "softmax":
            B, H, S = shp
            n = min(B * H * S, budget_rows)
            rng = np.random.Generator(np.random.PCG64(1))
            rb = rng.integers(0, B, size=n)
            x = W.scores(n, 1, 1, S, dt, seed=2).reshape(n, S)
            rl = np.asarray(lens, dtype=np.int32)[rb]
            job = lambda lo, hi: oracle.softmax_rows(x[lo:hi], rl[lo:hi], 0.125)  # noqa: E731
        else:
            n = min(shp[0], budget_rows // 4)
            d = W.ln_inputs(n, shp[1], dt, seed=2)
            job = lambda lo, hi: oracle.add_bias_layernorm(d["x"][lo:hi], d["residual"][lo:hi],  # noqa
                                                           d["bias"], d["gamma"], d["beta"], 1e-12)
        t = time.perf_counter()
        job(0, n)
        t1 = time.perf_counter() - t
        step = (n + cores - 1) // cores
        t = time.perf_counter()
        with cf.ThreadPoolExecutor(cores) as ex:
            list(ex.map(lambda lo: job(lo, min(n, lo + step)), range(0, n, step)))
        tn = time.perf_counter() - t
        print(json.dumps(dict(key(c), oracle_rows=n, oracle_1t_rows_per_s=round(n / t1, 1),
                              oracle_all_rows_per_s=round(n / tn, 1), cores=cores)), flush=True)


if __name__ == "__main__":
    if "--ncu" in sys.argv:
        run_ncu()
    if "--oracle" in sys.argv:
        run_oracle()
