# Segmented (one-request CTAs) softmax warp tiers: GPU parity + sweep + tuning of the 16-bit 256-320 band.
set -x
mkdir -p gpurun_out/seg
timeout 1200 python -m pytest tests/test_parity_softmax.py tests/test_parity_packed.py tests/test_pdl.py -q -p no:cacheprovider -x 2>&1 | tail -5 > gpurun_out/seg/pytest.txt
timeout 1200 python tools/sweep.py > gpurun_out/seg/sweep.jsonl 2> gpurun_out/seg/sweep.err
for spec in "f16 20 12 300 300" "f16 20 12 256 256"; do
  for rg in 0 1; do
    RAGGED=$rg ONLY=G8 TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 300 python tools/tune.py softmax $spec > gpurun_out/seg/tune_${spec// /_}_r$rg.jsonl 2>&1
  done
done
RAGGED=c3 TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 300 python tools/tune.py softmax f16 64 12 497 497 > gpurun_out/seg/tune_c3.jsonl 2>&1
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/seg/bench.json 2> gpurun_out/seg/bench.err
