set -x
timeout 900 python -m pytest tests/test_parity_softmax.py tests/test_parity_packed.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/pf_pytest.txt
mkdir -p gpurun_out/pf
RAGGED=c3 timeout 600 python tools/tune.py softmax f16 64 12 491 491 > gpurun_out/pf/c3_f16.jsonl 2>&1
RAGGED=c3 timeout 600 python tools/tune.py softmax f32 64 12 491 491 > gpurun_out/pf/c3_f32.jsonl 2>&1
timeout 600 python tools/tune.py softmax f16 20 12 500 500 > gpurun_out/pf/c2_f16_500.jsonl 2>&1
RAGGED=1 timeout 600 python tools/tune.py softmax f16 20 12 500 500 > gpurun_out/pf/c2r_f16_500.jsonl 2>&1
timeout 600 python tools/tune.py softmax f16 20 12 400 400 > gpurun_out/pf/c2_f16_400.jsonl 2>&1
RAGGED=1 timeout 600 python tools/tune.py softmax f16 20 12 400 400 > gpurun_out/pf/c2r_f16_400.jsonl 2>&1
timeout 600 python tools/tune.py softmax f16 20 12 300 300 > gpurun_out/pf/c2_f16_300.jsonl 2>&1
RAGGED=1 timeout 600 python tools/tune.py softmax f32 20 12 300 300 > gpurun_out/pf/c2r_f32_300.jsonl 2>&1
timeout 600 python tools/tune.py softmax bf16 64 16 512 512 > gpurun_out/pf/c4.jsonl 2>&1
timeout 600 python tools/tune.py softmax f16 20 12 256 256 > gpurun_out/pf/c2_f16_256.jsonl 2>&1
timeout 600 python tools/tune.py softmax f16 20 12 200 200 > gpurun_out/pf/c2_f16_200.jsonl 2>&1
