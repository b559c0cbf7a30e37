"""Multi-process path of bench.py through the CUDA kernels.

`bench.py --gpus 2 --backend gloo` spawns two ranks by itself (no torchrun);
with gloo both ranks may share the single GPU a test box has.  The C5 request
stream is LPT-sharded over the ranks with no data-path collective; the
per-batch digests of the FULL softmax and LayerNorm outputs, gathered over the
process group, must give the same whole-stream digest as one rank (sharding
invariance, bit for bit)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _bench(n, *extra):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--backend", "gloo",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "0", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_c5_stream_two_ranks_match_one_rank_bit_for_bit():
    one = _bench(1, "--workload", "c5")
    two = _bench(2, "--workload", "c5")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert one["config"]["workload"] == two["config"]["workload"]
    assert two["scaling"] == "strong"
    assert [r["rank"] for r in two["ranks"]] == [0, 1]
    assert sum(r["batches"] for r in two["ranks"]) == 64
    assert one["stream_digest"] == two["stream_digest"]


def test_c4_line_carries_c5_strong_scaling_sub_record():
    two = _bench(2, "--workload", "c4", "--c5-steps", "2")
    assert two["scaling"] == "weak" and two["backend"] == "gloo"
    assert len({r["digest"] for r in two["ranks"]}) == 2       # each rank: its own C4 batch
    c5 = two["c5_stream"]
    assert c5["scaling"] == "strong" and c5["batches"] == 64 and c5["value"] > 0
    one = _bench(1, "--workload", "c4", "--c5-steps", "2")
    assert one["c5_stream"]["stream_digest"] == c5["stream_digest"]
