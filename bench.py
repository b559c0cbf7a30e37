#!/usr/bin/env python
"""bench.py -- throughput of the batch-reduction hot path on B200.

One "step" = one pass of the whole hot path over one batch: the in-place
masked softmax over the attention scores followed by
the fused add-bias + residual + LayerNorm (LN-1..LN-3), both through the C ABI
of libtt.so.

Default workload (N=1): C4 = BERT-large, 16 heads, hidden 1024, batch 64,
seq 512, bf16 -- the largest single-GPU configuration in BASELINE.json and the
headline bandwidth-bound case (scores 512 MiB + LN 192 MiB, larger than the
126 MB L2, so no flush is needed between steps).  At N GPUs every rank runs its
own C4 batch (weak scaling; no data-path collective).
`--workload c5` runs the 4096-request stream sharded by LPT (strong scaling).

Metric (BASELINE.json): achieved HBM GB/s (algorithmic bytes)
and rows/s for softmax & LayerNorm.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c4|c3|c5] [--e2e-steps E] [--no-cpu-baseline]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "achieved HBM GB/s (% of B200 peak) and rows/s for softmax & LayerNorm"
UNIT = "GB/s"


# ------------------------------------------------------------------ workloads
class Workload:
    """A list of (softmax batch, LN batch) units resident on one device."""

    def __init__(self, name, dtype, heads, hidden, batches, scale=W.SCALE_BERT, eps=W.EPS_BERT,
                 packed=False):
        self.name, self.dtype, self.heads, self.hidden = name, dtype, heads, hidden
        self.batches = batches          # list of np.int32 length arrays (one per batch)
        self.scale, self.eps = scale, eps
        self.e = W.ELEM_BYTES[dtype]
        # packed: padding-free layout: request r is a dense
        # [H, L_r, L_r] block; LayerNorm runs on sum(L_r) tokens
        self.packed = packed

    def shapes(self, lens):
        S = int(lens.max())
        if self.packed:
            return (int(self.heads * (lens.astype(np.int64) ** 2).sum()),), (int(lens.sum()),
                                                                              self.hidden)
        return (len(lens), self.heads, S, S), (len(lens) * S, self.hidden)

    def bytes_softmax(self, lens):
        if self.packed:   # every key read once and written once, + cu_seqlens / cu_blocks
            return int(2 * self.heads * (lens.astype(np.int64) ** 2).sum() * self.e
                       + 12 * len(lens) + 4)
        S = int(lens.max())
        return W.softmax_bytes_alg(lens, self.heads, S, S, self.e)

    def bytes_ln(self, lens):
        if self.packed:
            return W.ln_bytes_alg(int(lens.sum()), self.hidden, self.e)
        return W.ln_bytes_alg(len(lens) * int(lens.max()), self.hidden, self.e)

    def rows(self, lens):
        if self.packed:
            return self.heads * int(lens.sum()), int(lens.sum())
        S = int(lens.max())
        return len(lens) * self.heads * S, len(lens) * S


def make_workload(name: str, rank: int, world: int):
    """Returns (Workload with this rank's batches, description dict, scaling)."""
    if name == "c4":
        c = W.C4
        lens = W.lengths_full(c.extra["batch"], c.extra["seq"])
        wl = Workload("C4", torch.bfloat16, c.heads, c.hidden, [lens])
        desc = {"workload": "C4: BERT-large heads=16 hidden=1024 batch=64 seq=512 bf16, per rank",
                "softmax_shape": [64, 16, 512, 512], "ln_shape": [32768, 1024],
                "global_batch": 64 * world, "seq_len": 512, "heads": 16, "hidden": 1024,
                "scale": W.SCALE_BERT, "eps": W.EPS_BERT,
                "l2": "inputs larger than L2 (softmax 512 MiB, LN 192 MiB per step vs 126 MB)",
                "parallelism": f"dp{world} (independent request batches, no data-path collective)"}
        return wl, desc, "weak"
    if name == "c3":
        c = W.C3
        lens = W.c3_lengths(salt=rank)
        wl = Workload("C3", torch.float16, c.heads, c.hidden, [lens])
        desc = {"workload": "C3: 64 requests U{5..500} padded to Smax, BERT-base fp16, per rank",
                "smax": int(lens.max()), "global_batch": 64 * world, "heads": 12, "hidden": 768,
                "l2": "inputs larger than L2", "parallelism": f"dp{world}"}
        return wl, desc, "weak"
    if name == "c5":
        from paper_2010_05680_b200.sharding import lpt_partition
        c = W.C5
        allb = W.c5_stream()
        tmp = Workload("C5", torch.float16, c.heads, c.hidden, allb)
        costs = [tmp.bytes_softmax(l) + tmp.bytes_ln(l) for l in allb]
        mine = lpt_partition(costs, world)[rank]
        wl = Workload("C5", torch.float16, c.heads, c.hidden, [allb[i] for i in mine])
        wl.batch_ids = mine
        desc = {"workload": "C5: 4096 requests U{5..500}, 64 batches of 64, fp16, LPT-sharded",
                "global_batch": 4096, "heads": 12, "hidden": 768,
                "l2": "inputs larger than L2", "parallelism": f"dp{world} (LPT batch shards)"}
        return wl, desc, "strong"
    if name in ("c3p", "c5p"):
        wl, desc, scaling = make_workload(name[:2], rank, world)
        wl.packed = True
        wl.name += "p"
        desc["workload"] = desc["workload"].replace("padded to Smax", "packed") + \
            " -- packed, padding-free layout (NEXT-1: tt_softmax_packed + LN on sum(L) tokens)"
        return wl, desc, scaling
    raise SystemExit(f"unknown workload {name}")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, dev: torch.device, period_s: float = 0.00025):
        self.samples, self.reasons, self.ok = [], 0, False
        self.period, self.stop_ev = period_s, threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            pr = torch.cuda.get_device_properties(dev)
            try:  # NVML indices ignore CUDA_VISIBLE_DEVICES: match by PCI address
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(dev.index or 0)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = repr(e)

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r) & ~0x1
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b]}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel_key: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed
    ncu --set full capture (profiles/traffic.json), if one matches this kernel."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        v = d.get(kernel_key)
        return None if v is None else float(v["dram_bytes_per_launch"])
    except Exception:
        return None


# ------------------------------------------------------------------ our arm
def _units(tt, wl, rank, scaling, dev, stream):
    """This rank's batches, generated on the device (resident in HBM before
    any timed region)."""
    units = []
    with torch.cuda.stream(stream):
        for bi, lens in enumerate(wl.batches):
            sshape, lshape = wl.shapes(lens)
            bid = wl.batch_ids[bi] if hasattr(wl, "batch_ids") else bi
            seed = W.SEED + 10007 * bid + (7919 * rank if scaling == "weak" else 0)
            x = (W.scores(1, 1, 1, sshape[0], wl.dtype, device=dev, seed=seed) if wl.packed
                 else W.scores(*sshape, wl.dtype, device=dev, seed=seed))
            d = W.ln_inputs(lshape[0], lshape[1], wl.dtype, device=dev, seed=seed + 1)
            if wl.packed:
                cu, blocks, total, _ = tt.packed_offsets(lens, wl.heads, device=dev)
                x = x.reshape(-1)
            else:
                cu = blocks = total = None
            units.append(dict(lens=lens, bid=bid, scores=x, L=torch.as_tensor(lens).to(dev),
                              cu=cu, blocks=blocks, total=total, maxlen=int(lens.max()),
                              out=torch.empty_like(d["x"]), **d))
    stream.synchronize()
    return units


def _step_fn(tt, wl, units, stream, nstreams=1):
    """One step over this rank's batches.  With several batches and nstreams > 1
    the batches are dealt round-robin over that many CUDA streams forked from
    and joined back into `stream` every step (a batch's softmax and LayerNorm
    stay in order on one stream), so one kernel's tail overlaps the next
    batch's kernels -- how a server would issue independent requests."""
    streams = [stream] + [torch.cuda.Stream(device=stream.device)
                          for _ in range(max(1, nstreams) - 1)] if len(units) > 1 else [stream]
    fork = torch.cuda.Event()
    joins = [torch.cuda.Event() for _ in streams]

    def step(ev=None):
        if len(streams) > 1:
            fork.record(stream)
            for st in streams[1:]:
                st.wait_event(fork)
        for i, u in enumerate(units):
            st = streams[i % len(streams)]
            if ev is not None:
                ev[0].record(st)
            if wl.packed:
                tt.tt_softmax_packed(u["scores"], u["cu"], u["blocks"], wl.heads, u["total"],
                                     u["maxlen"], wl.scale, stream=st)
            else:
                tt.tt_softmax_masked(u["scores"], u["L"], wl.scale, stream=st)
            if ev is not None:
                ev[1].record(st)
            tt.tt_add_bias_layernorm(u["out"], u["x"], u["residual"], u["bias"], u["gamma"],
                                     u["beta"], wl.eps, stream=st)
            if ev is not None:
                ev[2].record(st)
        if len(streams) > 1:
            for st, j in zip(streams[1:], joins[1:]):
                j.record(st)
                stream.wait_event(j)
    return step


def _timed(step, K, n_events, dist, dev, stream, coll_dev):
    """K steps bracketed by barrier + synchronize on both sides, CUDA events on
    the launching stream, NVML clocks sampled during the region; returns
    (max-over-ranks ms, local ms, per-kernel event triples, clock summary)."""
    from paper_2010_05680_b200 import sharding
    per_kernel = [[torch.cuda.Event(enable_timing=True) for _ in range(3)]
                  for _ in range(min(K, n_events))]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        t0.record(stream)
        for k in range(K):
            step(per_kernel[k] if k < len(per_kernel) else None)
        t1.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_local = t0.elapsed_time(t1)
    ms = sharding.max_over_ranks(ms_local, coll_dev) if dist else ms_local
    return ms, ms_local, per_kernel, clk.summary()


def _digests(units):
    """Per-batch digests of the FULL softmax output (in place) and LN output."""
    from paper_2010_05680_b200 import sharding
    return {int(u["bid"]): (sharding.device_digest(u["scores"]), sharding.device_digest(u["out"]))
            for u in units}


def _stream_record(dist, units, digests, ms, ms_local, rank, world, wl, K, scaling):
    """Gather (rank, ms, batches, per-batch digests) to every rank; returns the
    whole-stream aggregate seen by rank 0."""
    from paper_2010_05680_b200 import sharding
    mine = {"rank": rank, "ms": ms_local, "batches": sorted(digests),
            "digests": digests,
            "bytes": sum(wl.bytes_softmax(u["lens"]) + wl.bytes_ln(u["lens"]) for u in units),
            "rows": [sum(wl.rows(u["lens"])[0] for u in units),
                     sum(wl.rows(u["lens"])[1] for u in units)]}
    allr = sharding.gather_objects(mine) if dist else [mine]
    bd = {}
    for r in allr:
        for k, v in r["digests"].items():
            bd[int(k)] = sharding.combine_digests(v)
    tot_bytes = sum(r["bytes"] for r in allr)
    return {
        "value": round(tot_bytes * K / (ms / 1e3) / 1e9, 2), "ms_per_step": round(ms / K, 6),
        "bytes_per_step": int(tot_bytes),
        "rows_per_s": {"softmax": round(sum(r["rows"][0] for r in allr) * K / (ms / 1e3), 1),
                       "layernorm": round(sum(r["rows"][1] for r in allr) * K / (ms / 1e3), 1)},
        "stream_digest": f"{sharding.stream_digest(bd):016x}",
        "batches": len(bd),
        "ranks": [{"rank": r["rank"], "ms": round(r["ms"], 3), "batches": len(r["batches"]),
                   "digest": f"{sharding.stream_digest({int(k): sharding.combine_digests(v) for k, v in r['digests'].items()}):016x}"}
                  for r in sorted(allr, key=lambda r: r["rank"])],
    }


def run_ours(args, rank, world, local_rank):
    import datetime
    import paper_2010_05680_b200 as tt

    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local_rank % max(ndev, 1))
    torch.cuda.set_device(dev)
    dist = None
    coll_dev = dev
    if world > 1:
        import torch.distributed as dist
        timeout = datetime.timedelta(seconds=args.dist_timeout)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev, timeout=timeout)
        else:   # gloo: several ranks may share one GPU (tests); collectives on host tensors
            dist.init_process_group("gloo", timeout=timeout)
            coll_dev = torch.device("cpu")
    tt.lib()
    wl, desc, scaling = make_workload(args.workload, rank, world)
    stream = torch.cuda.Stream(device=dev)
    units = _units(tt, wl, rank, scaling, dev, stream)

    if len(units) > 1:
        desc["streams"] = args.streams
    plan_sm = (tt.softmax_packed_plan(wl.dtype, max(u["maxlen"] for u in units)) if wl.packed
               else tt.softmax_plan(wl.dtype, *units[0]["scores"].shape))
    plan_ln = tt.layernorm_plan(wl.dtype, *units[0]["x"].shape)
    b_sm = sum(wl.bytes_softmax(u["lens"]) for u in units)
    b_ln = sum(wl.bytes_ln(u["lens"]) for u in units)

    step = _step_fn(tt, wl, units, stream, args.streams)
    for _ in range(args.warmup):
        step()
    stream.synchronize()

    # ---- timed region: K steps
    K = args.steps
    n_ev = args.kernel_events if len(units) == 1 else 0
    ms, ms_local, per_kernel, clocks = _timed(step, K, n_ev, dist, dev, stream, coll_dev)
    sm_ms = [e[0].elapsed_time(e[1]) for e in per_kernel]
    ln_ms = [e[1].elapsed_time(e[2]) for e in per_kernel]

    # ---- per-batch digests of every output, gathered over the process group
    rec = _stream_record(dist, units, _digests(units), ms, ms_local, rank, world, wl, K, scaling)

    # ---- end to end through the staged C-ABI call with pinned host buffers
    e2e = (run_e2e(args, tt, wl, units, stream, dist, dev, world, coll_dev)
           if args.e2e_steps > 0 and not wl.packed else None)

    # ---- C5 strong-scaling sub-record (the BASELINE config-5 stream, LPT-sharded)
    c5 = None
    if args.workload == "c4" and args.c5_steps > 0:
        del units, step
        torch.cuda.empty_cache()
        wl5, desc5, sc5 = make_workload("c5", rank, world)
        u5 = _units(tt, wl5, rank, sc5, dev, stream)
        st5 = _step_fn(tt, wl5, u5, stream, args.streams)
        for _ in range(3):
            st5()
        stream.synchronize()
        ms5, ms5_local, _, clk5 = _timed(st5, args.c5_steps, 0, dist, dev, stream, coll_dev)
        c5 = _stream_record(dist, u5, _digests(u5), ms5, ms5_local, rank, world, wl5,
                            args.c5_steps, sc5)
        c5.update({"workload": desc5["workload"], "scaling": sc5, "steps": args.c5_steps,
                   "streams": args.streams,
                   "warmup": 3, "clocks": clk5,
                   "kernels": {"softmax": tt.softmax_plan(wl5.dtype, *u5[0]["scores"].shape),
                               "layernorm": tt.layernorm_plan(wl5.dtype, *u5[0]["x"].shape)}})
        del u5, st5

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return None

    value = rec["value"]
    peak, peak_src = measured_peak()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(ms / K, 6), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32",
        "arith": "fp32", "storage": W.DTYPE_NAMES[wl.dtype],
        "data": "synthetic (seeded; logits N(0,8^2), LN inputs N(0,1); SURVEY §8(d) recipe)",
        "config": desc,
        "rows_per_s": rec["rows_per_s"],
        "pct_of_peak": round(100.0 * value / (peak * world), 2),
        "pct_of_nominal_8TBps": round(100.0 * value / (8000.0 * world), 2),
        "gpu_launches": 2 * len(wl.batches) * K,
        "kernels": {"softmax": plan_sm, "layernorm": plan_ln},
    }
    if sm_ms:
        sm_avg, ln_avg = float(np.mean(sm_ms)), float(np.mean(ln_ms))
        ach_sm = b_sm / (sm_avg / 1e3) / 1e9
        ach_ln = b_ln / (ln_avg / 1e3) / 1e9
        out["roofline"] = {
            "bound": "hbm", "kernel": plan_sm, "achieved": round(ach_sm, 1), "peak": peak,
            "unit": "GB/s", "frac": round(ach_sm / peak, 4),
            "traffic": ncu_traffic(f"{wl.name}:{plan_sm}"),
            "bytes_alg_per_launch": b_sm, "avg_launch_us": round(sm_avg * 1e3, 2),
            "share_of_step": round(sm_avg / (ms_local / K), 4), "peak_source": peak_src,
        }
        out["roofline_layernorm"] = {
            "bound": "hbm", "kernel": plan_ln, "achieved": round(ach_ln, 1), "peak": peak,
            "unit": "GB/s", "frac": round(ach_ln / peak, 4),
            "traffic": ncu_traffic(f"{wl.name}:{plan_ln}"),
            "bytes_alg_per_launch": b_ln, "avg_launch_us": round(ln_avg * 1e3, 2),
            "share_of_step": round(ln_avg / (ms_local / K), 4),
        }
    out["clocks"] = clocks
    out["e2e"] = e2e
    out["stream_digest"] = rec["stream_digest"]
    out["ranks"] = rec["ranks"] if world > 1 else None
    if c5 is not None:
        out["c5_stream"] = c5
    if world > 1:
        out["backend"] = args.backend
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl, budget_s=args.cpu_budget)
    if dist:
        dist.destroy_process_group()
    return out


def run_e2e(args, tt, wl, units, stream, dist, dev, world, coll_dev):
    """Same metric end to end: per step, H2D of the step's inputs from pinned
    host memory, both kernels, D2H of both results, through the staged C ABI."""
    hosts = []
    for u in units:
        hosts.append(dict(scores=u["scores"].cpu().pin_memory(),
                          L=torch.as_tensor(u["lens"]).pin_memory(),
                          x=u["x"].cpu().pin_memory(), residual=u["residual"].cpu().pin_memory(),
                          out=torch.empty_like(u["x"], device="cpu").pin_memory()))
    h2d = sum(h["scores"].numel() * h["scores"].element_size() + h["L"].numel() * 4
              + 2 * h["x"].numel() * h["x"].element_size() for h in hosts)
    d2h = sum(h["scores"].numel() * h["scores"].element_size()
              + h["out"].numel() * h["out"].element_size() for h in hosts)

    # D2H of chunk i on a second stream under the H2D of chunk i+1 (PCIe is
    # full duplex); `stream` waits for the last D2H inside each call
    copy_stream = torch.cuda.Stream(device=dev)
    chunks = args.e2e_chunks

    def step():
        for u, h in zip(units, hosts):
            tt.tt_softmax_masked_staged_overlap(h["scores"], h["L"], u["scores"], u["L"],
                                                wl.scale, chunks, stream=stream,
                                                copy_stream=copy_stream)
            tt.tt_add_bias_layernorm_staged_overlap(h["out"], h["x"], h["residual"], u["out"],
                                                    u["x"], u["residual"], u["bias"], u["gamma"],
                                                    u["beta"], wl.eps, chunks, stream=stream,
                                                    copy_stream=copy_stream)

    for _ in range(2):
        step()
    stream.synchronize()
    E = args.e2e_steps
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(E):
        step()
    b.record(stream)
    stream.synchronize()
    ms = a.elapsed_time(b)
    if dist:
        from paper_2010_05680_b200 import sharding
        ms = sharding.max_over_ranks(ms, coll_dev)
    per_step_bytes = sum(wl.bytes_softmax(u["lens"]) + wl.bytes_ln(u["lens"]) for u in units)
    mult = world
    value = per_step_bytes * mult * E / (ms / 1e3) / 1e9
    return {"value": round(value, 2), "unit": UNIT, "steps": E, "ms_per_step": round(ms / E, 3),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "chunks": chunks,
            "api": "tt_softmax_masked_staged_overlap + tt_add_bias_layernorm_staged_overlap "
                   "(pinned host; D2H on a second stream under the next chunk's H2D)"}


# ------------------------------------------------------------------ oracle timing
def _oracle_sample(wl, frac, seed=0):
    """A bounded sample of the workload for the CPU oracle: `frac` of the
    softmax rows and of the LN rows of each batch (same shapes/distributions)."""
    samples = []
    for bi, lens in enumerate(wl.batches):
        B, H, S = len(lens), wl.heads, int(lens.max())
        R, hid = wl.shapes(lens)[1]
        rng = np.random.Generator(np.random.PCG64(seed + bi))
        if wl.packed:
            # rows of the packed layout: request r contributes H*L_r rows of L_r keys
            nrows_sm = max(1, int(round(H * int(lens.sum()) * frac)))
            w = lens.astype(np.float64) / lens.sum()
            rb = rng.choice(B, size=nrows_sm, p=w)
        else:
            nrows_sm = max(1, int(round(B * H * S * frac)))
            # rows keep their request's length: pick the batch index of each sampled row
            rb = rng.integers(0, B, size=nrows_sm)
        nrows_ln = max(1, int(round(R * frac)))
        x = W.scores(nrows_sm, 1, 1, S, wl.dtype, seed=W.SEED + bi)
        d = W.ln_inputs(nrows_ln, hid, wl.dtype, seed=W.SEED + bi + 1)
        samples.append(dict(x=x.reshape(nrows_sm, S), lens=lens[rb], d=d, S=S, hid=hid,
                            nrows_sm=nrows_sm, nrows_ln=nrows_ln))
    return samples


def _oracle_run(samples, wl, cores):
    """Run the oracle (as it stands) over the sample, row-partitioned across
    `cores` host threads (ctypes releases the GIL).  Returns (seconds, bytes, rows)."""
    import concurrent.futures as cf
    import oracle
    jobs = []
    for s in samples:
        for lo, hi in _chunks(s["nrows_sm"], cores):
            jobs.append(("sm", s, lo, hi))
        for lo, hi in _chunks(s["nrows_ln"], cores):
            jobs.append(("ln", s, lo, hi))

    def work(j):
        kind, s, lo, hi = j
        if kind == "sm":
            oracle.softmax_rows(s["x"][lo:hi], s["lens"][lo:hi], wl.scale)
        else:
            d = s["d"]
            oracle.add_bias_layernorm(d["x"][lo:hi], d["residual"][lo:hi], d["bias"], d["gamma"],
                                      d["beta"], wl.eps)

    t = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(work, jobs))
    dt = time.perf_counter() - t
    nbytes = 0
    rows = 0
    for s in samples:
        L = np.clip(s["lens"].astype(np.int64), 0, s["S"])
        if wl.packed:
            nbytes += 2 * int(L.sum()) * wl.e
        else:
            nbytes += int(L.sum()) * wl.e + s["nrows_sm"] * s["S"] * wl.e
        nbytes += W.ln_bytes_alg(s["nrows_ln"], s["hid"], wl.e)
        rows += s["nrows_sm"] + s["nrows_ln"]
    return dt, nbytes, rows


def _chunks(n, k):
    k = max(1, min(k, n))
    step = (n + k - 1) // k
    return [(i, min(n, i + step)) for i in range(0, n, step)]


def _calibrate(wl, cores, target_s):
    frac = 1.0 / 4096
    while True:
        dt, _, _ = _oracle_run(_oracle_sample(wl, frac), wl, cores)
        if dt > 0.25 or frac >= 1.0:
            break
        frac = min(1.0, frac * 4)
    return min(1.0, frac * max(target_s, 0.01) / max(dt, 1e-6))


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(wl, budget_s=10.0):
    """The oracle as it stands on this box's host cores: all threads (the
    reported value) and one thread (same sample, for the per-core figure)."""
    cores = os.cpu_count() or 1
    frac = _calibrate(wl, cores, budget_s)
    sample = _oracle_sample(wl, frac, seed=1)
    dt, nbytes, rows = _oracle_run(sample, wl, cores)
    frac1 = frac / max(1, cores)
    s1 = _oracle_sample(wl, frac1, seed=1)
    dt1, nb1, rows1 = _oracle_run(s1, wl, 1)
    return {"value": round(nbytes / dt / 1e9, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
            "rows_per_s": round(rows / dt, 1), "seconds": round(dt, 2),
            "one_thread": {"value": round(nb1 / dt1 / 1e9, 4), "unit": UNIT,
                           "rows_per_s": round(rows1 / dt1, 1), "seconds": round(dt1, 2),
                           "sample": f"{frac1:.4%} of the rows"},
            "cpu_model": _cpu_model(),
            "sample": f"{frac:.4%} of the {wl.name} softmax rows and LN rows "
                      f"(same shapes and value distributions), fp64 C oracle, "
                      f"row-partitioned over {cores} host threads"}


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The oracle as it stands, timed on the host cores, same metric/config."""
    if rank != 0:
        return None
    wl, desc, scaling = make_workload(args.workload, 0, 1)
    cores = os.cpu_count() or 1
    K, Wm = args.steps, args.warmup
    per_step_target = max(0.02, min(1.0, args.ref_budget / max(1, K + Wm)))
    frac = _calibrate(wl, cores, per_step_target)
    sample = _oracle_sample(wl, frac, seed=2)
    for _ in range(Wm):
        _oracle_run(sample, wl, cores)
    tot_t, tot_b, tot_r = 0.0, 0, 0
    for _ in range(K):
        dt, nb, nr = _oracle_run(sample, wl, cores)
        tot_t += dt
        tot_b += nb
        tot_r += nr
    value = tot_b / tot_t / 1e9
    samp = (f"{frac:.4%} of the {wl.name} softmax and LN rows per step, fp64 C oracle, "
            f"{cores} host threads")
    return {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": Wm, "ms_per_step": round(1e3 * tot_t / K, 3),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded; same recipe as ours)", "config": desc,
            "impl": "reference", "gpu_launches": 0,
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores,
                             "kind": "oracle", "sample": samp},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "rows_per_s": round(tot_r / tot_t, 1)}


def _spawn(n: int) -> int:
    """`--gpus N` without torchrun: start N copies of this script with the
    torch.distributed environment (one process per GPU, rendezvous on
    127.0.0.1); rank 0's stdout is this process's stdout.  Returns the worst
    exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    return max(p.wait() for p in procs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c4", "c3", "c5", "c3p", "c5p"], default="c4")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-chunks", type=int, default=8,
                    help="pieces per staged call (D2H of one under the H2D of the next)")
    ap.add_argument("--kernel-events", type=int, default=1000000,
                    help="per-kernel CUDA events for the first N timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ref-budget", type=float, default=90.0)
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="process-group backend for N > 1 (gloo: ranks may share a GPU; tests)")
    ap.add_argument("--dist-timeout", type=float, default=600.0,
                    help="process-group timeout, seconds")
    ap.add_argument("--streams", type=int, default=2,
                    help="CUDA streams the batches of a multi-batch step are dealt over")
    ap.add_argument("--c5-steps", type=int, default=10,
                    help="timed steps of the C5 strong-scaling sub-record (c4 workload; 0: off)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if "RANK" not in os.environ and args.gpus > 1:
        raise SystemExit(_spawn(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local_rank)
    if out is not None and rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
