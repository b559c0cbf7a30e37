# Softmax tiny shapes (C1, C2 S = 10 .. 100)
mkdir -p gpurun_out/smtiny
timeout 300 python tools/tune.py softmax f32 1 12 40 40 > gpurun_out/smtiny/f32_c1.jsonl 2>&1
for S in 10 20 40 64 100; do
timeout 300 python tools/tune.py softmax f16 20 12 $S $S > gpurun_out/smtiny/f16_$S.jsonl 2>&1
timeout 300 python tools/tune.py softmax f32 20 12 $S $S > gpurun_out/smtiny/f32_$S.jsonl 2>&1
done
