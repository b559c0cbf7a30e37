# Re-tune the 16-bit (384, 512] softmax band with the current build (narrow-NV paths)
mkdir -p gpurun_out/t512
RAGGED=c3 timeout 300 python tools/tune.py softmax f16 64 12 491 491 > gpurun_out/t512/c3_f16.jsonl 2>&1
timeout 300 python tools/tune.py softmax f16 20 12 500 500 > gpurun_out/t512/f16_500.jsonl 2>&1
RAGGED=1 timeout 300 python tools/tune.py softmax f16 20 12 500 500 > gpurun_out/t512/f16_500r.jsonl 2>&1
timeout 300 python tools/tune.py softmax f16 20 12 400 400 > gpurun_out/t512/f16_400.jsonl 2>&1
RAGGED=1 timeout 300 python tools/tune.py softmax f16 20 12 400 400 > gpurun_out/t512/f16_400r.jsonl 2>&1
timeout 300 python tools/tune.py softmax bf16 64 16 512 512 > gpurun_out/t512/c4.jsonl 2>&1
RAGGED=1 timeout 300 python tools/tune.py softmax bf16 64 16 512 512 > gpurun_out/t512/c4r.jsonl 2>&1
