# LayerNorm mid-size band (C2 S = 128 .. 500: 2560 .. 10000 rows of 768)
mkdir -p gpurun_out/lnmid
for rows in 2560 4000 5120 6000 8000 10000; do for dt in f16 f32; do
ONLY=ln_rows timeout 300 python tools/tune.py layernorm $dt $rows 768 > gpurun_out/lnmid/${dt}_${rows}.jsonl 2>&1
done; done
