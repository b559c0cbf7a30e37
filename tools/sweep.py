#!/usr/bin/env python
"""Sweep BASELINE.json's configurations through both operations; one JSON line
per (config, op, dtype, lengths) with time per call, algorithmic GB/s, % of
the measured copy peak and of the nominal 8 TB/s, the same-traffic torch
reference (an SM element-wise kernel moving the same bytes: torch.neg for the
softmax, torch.add for the LayerNorm), the max abs error against the fp64
oracle on sampled rows, plus an empty-kernel launch floor for the
launch-bound small shapes.

  python tools/sweep.py > gpurun_out/sweep.jsonl
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (error column only: the timed calls never touch it)
import paper_2010_05680_b200 as tt  # noqa: E402
import workloads as W  # noqa: E402

NOMINAL_GBPS = 8000.0

L2 = 126 * 1024 * 1024


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timeit(fn, nbufs, reps):
    """Device time per call: the calls are captured once into a CUDA graph and
    the graph is replayed, so host-side launch overhead (Python + ctypes) does
    not leak into small shapes; CUDA events on the replay stream."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
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
    return a.elapsed_time(b) / reps * 1e3  # us


def nbufs_for(nbytes):
    return int(max(1, min(64, -(-4 * L2 // max(nbytes, 1)))))


def softmax_case(cfg, dtype, B, H, S, lens, pk):
    e = W.ELEM_BYTES[dtype]
    nbytes = B * H * S * S * e
    nb = nbufs_for(nbytes)
    bufs = [W.scores(B, H, S, S, dtype, device="cuda", seed=i) for i in range(nb)]
    L = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
    reps = 200 if nbytes < 64 << 20 else 50
    us = timeit(lambda i: tt.tt_softmax_masked(bufs[i], L, 0.125), nb, reps)
    # same-traffic reference: an SM element-wise kernel (torch.neg) reading and
    # writing exactly the softmax's algorithmic bytes (alg / 2 each way; for
    # ragged lengths a prefix of the buffer, timed as it is -- not a full-size
    # time scaled down, which hid the small kernels' own ramp and tail).  (A D2D
    # copy_ is a copy-engine memcpy inside a graph, ~3 TB/s: not a peer.)
    alg = W.softmax_bytes_alg(lens, H, S, S, e)
    n_ref = max(1, min(B * H * S * S, int(alg // (2 * e))))
    other = [torch.empty_like(b) for b in bufs]
    src_f = [b.view(-1)[:n_ref] for b in bufs]
    dst_f = [o.view(-1)[:n_ref] for o in other]
    us_ref = timeit(lambda i: torch.neg(src_f[i], out=dst_f[i]), nb, reps)
    # max abs error vs the oracle on 256 sampled rows of a fresh input
    x = W.scores(B, H, S, S, dtype, device="cuda", seed=12345)
    nrows = B * H * S
    idx = torch.randint(0, nrows, (min(256, nrows),), generator=torch.Generator().manual_seed(1))
    before = x.view(nrows, S)[idx.cuda()].cpu()
    tt.tt_softmax_masked(x, L, 0.125)
    got = x.view(nrows, S)[idx.cuda()].cpu().double()
    ref = oracle.softmax_rows(before, np.asarray(lens, dtype=np.int32)[(idx // (H * S)).numpy()],
                              0.125)
    err = float((got - ref).abs().max())
    return dict(config=cfg, op="softmax", dtype=W.DTYPE_NAMES[dtype], shape=[B, H, S, S],
                ragged=bool(np.any(np.asarray(lens) < S)), us=round(us, 2),
                GBps=round(alg / us / 1e3, 1), pct_peak=round(100 * alg / us / 1e3 / pk, 1),
                pct_nominal=round(100 * alg / us / 1e3 / NOMINAL_GBPS, 1),
                ref_same_traffic_us=round(us_ref, 2),
                max_abs_err=err, tier=tt.softmax_plan(dtype, B, H, S, S))


def ln_case(cfg, dtype, rows, hidden, pk):
    e = W.ELEM_BYTES[dtype]
    nbytes = 3 * rows * hidden * e
    nb = nbufs_for(nbytes)
    ds = [W.ln_inputs(rows, hidden, dtype, device="cuda", seed=i) for i in range(nb)]
    outs = [torch.empty_like(d["x"]) for d in ds]
    reps = 200 if nbytes < 64 << 20 else 50
    us = timeit(lambda i: tt.tt_add_bias_layernorm(outs[i], ds[i]["x"], ds[i]["residual"],
                                                   ds[i]["bias"], ds[i]["gamma"], ds[i]["beta"],
                                                   1e-12), nb, reps)
    us_add = timeit(lambda i: torch.add(ds[i]["x"], ds[i]["residual"], out=outs[i]), nb, reps)
    alg = W.ln_bytes_alg(rows, hidden, e)
    d = W.ln_inputs(rows, hidden, dtype, device="cuda", seed=12345)
    o = torch.empty_like(d["x"])
    tt.tt_add_bias_layernorm(o, d["x"], d["residual"], d["bias"], d["gamma"], d["beta"], 1e-12)
    idx = torch.randint(0, rows, (min(256, rows),), generator=torch.Generator().manual_seed(1)).cuda()
    ref = oracle.add_bias_layernorm(d["x"][idx].cpu(), d["residual"][idx].cpu(), d["bias"].cpu(),
                                    d["gamma"].cpu(), d["beta"].cpu(), 1e-12)
    err = float((o[idx].cpu().double() - ref).abs().max())
    return dict(config=cfg, op="layernorm", dtype=W.DTYPE_NAMES[dtype], shape=[rows, hidden],
                ragged=False, us=round(us, 2), GBps=round(alg / us / 1e3, 1),
                pct_peak=round(100 * alg / us / 1e3 / pk, 1),
                pct_nominal=round(100 * alg / us / 1e3 / NOMINAL_GBPS, 1),
                ref_same_traffic_us=round(us_add, 2), max_abs_err=err,
                tier=tt.layernorm_plan(dtype, rows, hidden))


def next2_cases(pk):
    """NEXT-2 element-wise kernels on BERT shapes (read + write every byte once)."""
    out = []
    for dtype, B, S, H, D in ((torch.float16, 20, 128, 12, 64), (torch.bfloat16, 64, 512, 16, 64)):
        e = W.ELEM_BYTES[dtype]
        rows, hid = B * S, H * D
        # GELU on the FFN-up output [rows, 4*hidden]
        n = 4 * hid
        nb = nbufs_for(2 * rows * n * e)
        xs = [W.scores(1, 1, rows, n, dtype, device="cuda", seed=i, std=2.0).reshape(rows, n)
              for i in range(nb)]
        b = torch.zeros(n, dtype=dtype, device="cuda")
        ys = [torch.empty_like(x) for x in xs]
        us = timeit(lambda i: tt.tt_add_bias_gelu(ys[i], xs[i], b), nb, 50)
        us_c = timeit(lambda i: torch.neg(xs[i], out=ys[i]), nb, 50)
        alg = 2 * rows * n * e + n * e
        out.append(dict(config=f"BERT b{B} s{S}", op="add_bias_gelu", dtype=W.DTYPE_NAMES[dtype],
                        shape=[rows, n], ragged=False, us=round(us, 2),
                        GBps=round(alg / us / 1e3, 1), pct_peak=round(100 * alg / us / 1e3 / pk, 1),
                        ref_same_traffic_us=round(us_c, 2), tier="add_bias_gelu<V16>"))
        # QKV split [rows, 3*hid] -> 3 x [B, H, S, D]; head merge [B, H, S, D] -> [rows, hid]
        nb = nbufs_for(2 * rows * 3 * hid * e)
        qkv = [W.scores(1, 1, rows, 3 * hid, dtype, device="cuda", seed=i).reshape(rows, 3 * hid)
               for i in range(nb)]
        bias = torch.zeros(3 * hid, dtype=dtype, device="cuda")
        outs = [[torch.empty(B, H, S, D, dtype=dtype, device="cuda") for _ in range(3)]
                for _ in range(nb)]
        us = timeit(lambda i: tt.tt_split_qkv_add_bias(*outs[i], qkv[i], bias, B, S, H, D), nb, 50)
        us_c = timeit(lambda i: torch.neg(qkv[i].view(-1)[:rows * hid], out=outs[i][0].view(-1)), nb, 50)
        alg = 2 * rows * 3 * hid * e + 3 * hid * e
        out.append(dict(config=f"BERT b{B} s{S}", op="split_qkv_add_bias", dtype=W.DTYPE_NAMES[dtype],
                        shape=[rows, 3 * hid], ragged=False, us=round(us, 2),
                        GBps=round(alg / us / 1e3, 1), pct_peak=round(100 * alg / us / 1e3 / pk, 1),
                        ref_same_traffic_us=round(3 * us_c, 2), tier="split_qkv<V16>"))
        ms = [torch.empty(rows, hid, dtype=dtype, device="cuda") for _ in range(nb)]
        us = timeit(lambda i: tt.tt_merge_heads(ms[i], outs[i][0], B, S, H, D), nb, 50)
        us_c = timeit(lambda i: torch.neg(outs[i][0].view(-1), out=ms[i].view(-1)), nb, 50)
        alg = 2 * rows * hid * e
        out.append(dict(config=f"BERT b{B} s{S}", op="merge_heads", dtype=W.DTYPE_NAMES[dtype],
                        shape=[B, H, S, D], ragged=False, us=round(us, 2),
                        GBps=round(alg / us / 1e3, 1), pct_peak=round(100 * alg / us / 1e3 / pk, 1),
                        ref_same_traffic_us=round(us_c, 2), tier="merge_heads<V16>"))
    return out


def main():
    pk = peak()
    if "--next2" in sys.argv:
        for r in next2_cases(pk):
            print(json.dumps(r), flush=True)
        return
    # per-kernel floor inside a graph: torch's smallest kernel (1-element add)
    z = torch.zeros(1, device="cuda")
    floor = timeit(lambda i: z.add_(0), 1, 500)
    print(json.dumps({"launch_floor_us": round(floor, 2), "peak_GBps": pk}), flush=True)
    out = []
    out.append(softmax_case("C1", torch.float32, 1, 12, 40, [40], pk))
    out.append(ln_case("C1", torch.float32, 40, 768, pk))
    for dtype in (torch.float16, torch.float32):
        for S in W.C2.extra["seqs"]:
            out.append(softmax_case("C2", dtype, 20, 12, S, W.lengths_full(20, S), pk))
            out.append(softmax_case("C2", dtype, 20, 12, S, W.lengths_ragged(20, S), pk))
            out.append(ln_case("C2", dtype, 20 * S, 768, pk))
    for dtype in (torch.float16, torch.float32):
        lens = W.c3_lengths()
        S = int(lens.max())
        out.append(softmax_case("C3", dtype, 64, 12, S, lens, pk))
        out.append(ln_case("C3", dtype, 64 * S, 768, pk))
    out.append(softmax_case("C4", torch.bfloat16, 64, 16, 512, W.lengths_full(64, 512), pk))
    out.append(softmax_case("C4", torch.bfloat16, 64, 16, 512, W.lengths_ragged(64, 512, 4), pk))
    out.append(ln_case("C4", torch.bfloat16, 32768, 1024, pk))
    for r in out:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
