# LayerNorm tiny band (C1 / C2 S = 10 .. 100: 40 .. 2000 rows of 768)
mkdir -p gpurun_out/lntiny
for rows in 40 200 400 800 1280 2000; do for dt in f16 f32; do
ONLY=ln_rows timeout 300 python tools/tune.py layernorm $dt $rows 768 > gpurun_out/lntiny/${dt}_${rows}.jsonl 2>&1
done; done
