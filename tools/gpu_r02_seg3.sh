set -x
mkdir -p gpurun_out/seg3
timeout 1200 python -m pytest tests/test_parity_softmax.py -q -p no:cacheprovider -x 2>&1 | tail -3 > gpurun_out/seg3/pytest.txt
RAGGED=c3 ONLY=G32,NV1 TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 300 python tools/tune.py softmax f16 64 12 497 497 > gpurun_out/seg3/tune_c3.jsonl 2>&1
for spec in "f16 20 12 400 400" "f16 20 12 500 500"; do
  RAGGED=1 ONLY=V32,G32,NV1 TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 300 python tools/tune.py softmax $spec > gpurun_out/seg3/tune_${spec// /_}_r1.jsonl 2>&1
done
timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/seg3/bench_c5.json 2> gpurun_out/seg3/bench.err
