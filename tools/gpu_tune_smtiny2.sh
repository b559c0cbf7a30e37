mkdir -p gpurun_out/smtiny2
for S in 100 128; do
ONLY=f32,V16,G8 timeout 300 python tools/tune.py softmax f32 20 12 $S $S > gpurun_out/smtiny2/f32_$S.jsonl 2>&1
ONLY=f32,V16,G8 RAGGED=1 timeout 300 python tools/tune.py softmax f32 20 12 $S $S > gpurun_out/smtiny2/f32_${S}r.jsonl 2>&1
done
for S in 20 40 64; do
ONLY=f32,V16,G8 RAGGED=1 timeout 300 python tools/tune.py softmax f32 20 12 $S $S > gpurun_out/smtiny2/f32_${S}r.jsonl 2>&1
done
ONLY=f32,V16,G8 timeout 300 python tools/tune.py softmax f32 1 12 40 40 > gpurun_out/smtiny2/f32_c1.jsonl 2>&1
