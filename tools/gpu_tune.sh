# Tier sweep only (tools/tune.py) on the headline shapes.  ONLY=<substring> filters tiers.
set -x
for spec in "softmax bf16 64 16 512 512" "softmax f16 64 12 491 491" "softmax f32 20 12 500 500" "layernorm bf16 32768 1024" "layernorm f16 31424 768" "layernorm f32 10000 768"; do
  name=$(echo $spec | tr ' ' '_')
  timeout 900 python tools/tune.py $spec > gpurun_out/tune_$name.jsonl 2>&1
done
RAGGED=1 timeout 900 python tools/tune.py softmax f16 64 12 491 491 > gpurun_out/tune_softmax_ragged_f16_491.jsonl 2>&1
