# A/B of libtt.so against paper_2010_05680_b200/libtt_old.so on the tuned shapes (SPECS) and the bench
mkdir -p gpurun_out/ab
SPECS=${SPECS:-"layernorm bf16 32768 1024;layernorm f16 31808 768;layernorm f16 10000 768;layernorm f32 31808 768"}
IFS=';' read -ra LIST <<< "$SPECS"
for rep in 1 2; do
for spec in "${LIST[@]}"; do
  name=$(echo $spec | tr ' ' '_')
  ONLY=xx timeout 300 python tools/tune.py $spec > gpurun_out/ab/new_${name}_$rep.jsonl 2>&1
  ONLY=xx TT_LIB_PATH=paper_2010_05680_b200/libtt_old.so timeout 300 python tools/tune.py $spec > gpurun_out/ab/old_${name}_$rep.jsonl 2>&1
done
done
timeout 300 python bench.py --steps 500 --warmup 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab/bench_new.json 2>/dev/null
TT_LIB_PATH=paper_2010_05680_b200/libtt_old.so timeout 300 python bench.py --steps 500 --warmup 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab/bench_old.json 2>/dev/null
timeout 600 python -m pytest tests/test_parity_layernorm.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/ab/pytest.txt
