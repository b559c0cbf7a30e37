# quick: reference streaming kernels vs current auto tiers on the headline shapes
set -x
for spec in "softmax bf16 64 16 512 512" "softmax f16 64 12 491 491" "layernorm bf16 32768 1024" "layernorm f16 31424 768" "layernorm f32 10000 768"; do
  name=$(echo $spec | tr ' ' '_')
  ONLY=${ONLY:-_} timeout 900 python tools/tune.py $spec > gpurun_out/tune_$name.jsonl 2>&1
done
