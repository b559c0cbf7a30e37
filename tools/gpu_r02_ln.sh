# Round 2: GPU tests on the product library, then LayerNorm tier timings from
# the tuning build (libtt_tune.so) on the BERT LayerNorm shapes.
set -x
mkdir -p gpurun_out/ln
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
tail -5 gpurun_out/pytest_gpu.txt
for spec in "bf16 32768 1024" "f16 31808 768" "f16 10000 768" "f16 5120 768" "f32 31808 768" "f32 10000 768" "f32 6000 768" "bf16 31808 768"; do
  set -- $spec
  TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 300 python tools/tune.py layernorm $spec > gpurun_out/ln/tune_$1_$2_$3.jsonl 2>&1
done
python - <<'PY' > gpurun_out/ln/refs.jsonl
import sys, json, torch
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import sweep, workloads as W
pk = sweep.peak()
for dt, rows, hid in (("bf16", 32768, 1024), ("f16", 31808, 768), ("f16", 10000, 768), ("f16", 5120, 768), ("f32", 31808, 768), ("f32", 10000, 768), ("f32", 6000, 768)):
    print(json.dumps(sweep.ln_case("ref", W.DTYPES[dt], rows, hid, pk)))
PY
ls -la gpurun_out/ln
