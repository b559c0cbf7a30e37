set -x
mkdir -p gpurun_out/lntune
export TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so
for dt in f16 f32; do for rows in 5120 6000 8000 10000; do
timeout 600 python tools/tune.py layernorm $dt $rows 768 > gpurun_out/lntune/tune_${dt}_${rows}.jsonl 2>/dev/null
done; done
