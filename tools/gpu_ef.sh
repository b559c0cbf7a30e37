mkdir -p gpurun_out/ef
for i in 1 2; do
timeout 300 python bench.py --steps 500 --warmup 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ef/base_$i.json 2>/dev/null
TT_LIB_PATH=paper_2010_05680_b200/libtt_ef.so timeout 300 python bench.py --steps 500 --warmup 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ef/ef_$i.json 2>/dev/null
done
ONLY=xx timeout 300 python tools/tune.py layernorm bf16 32768 1024 > gpurun_out/ef/ln_base.jsonl 2>&1
ONLY=xx TT_LIB_PATH=paper_2010_05680_b200/libtt_ef.so timeout 300 python tools/tune.py layernorm bf16 32768 1024 > gpurun_out/ef/ln_ef.jsonl 2>&1
ONLY=xx timeout 300 python tools/tune.py softmax bf16 64 16 512 512 > gpurun_out/ef/sm_base.jsonl 2>&1
ONLY=xx TT_LIB_PATH=paper_2010_05680_b200/libtt_ef.so timeout 300 python tools/tune.py softmax bf16 64 16 512 512 > gpurun_out/ef/sm_ef.jsonl 2>&1
