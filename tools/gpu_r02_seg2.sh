set -x
mkdir -p gpurun_out/seg2
timeout 1200 python -m pytest tests/test_parity_softmax.py -q -p no:cacheprovider -x 2>&1 | tail -3 > gpurun_out/seg2/pytest.txt
for spec in "f16 20 12 300 300" "bf16 20 12 300 300" "f16 20 12 256 256"; do
  for rg in 0 1; do
    RAGGED=$rg ONLY=G8 TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 300 python tools/tune.py softmax $spec > gpurun_out/seg2/tune_${spec// /_}_r$rg.jsonl 2>&1
  done
done
timeout 1200 python tools/sweep.py > gpurun_out/seg2/sweep.jsonl 2> gpurun_out/seg2/sweep.err
