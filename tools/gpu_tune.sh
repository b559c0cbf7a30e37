# Tier sweep (tools/tune.py).  SPECS overrides the shape list; ONLY filters tiers.
set -x
SPECS=${SPECS:-"softmax bf16 64 16 512 512;softmax f16 64 12 491 491;softmax f32 20 12 500 500;layernorm bf16 32768 1024;layernorm f16 31424 768;layernorm f32 10000 768"}
IFS=';' read -ra LIST <<< "$SPECS"
for spec in "${LIST[@]}"; do
  name=$(echo $spec | tr ' ' '_')
  timeout 900 python tools/tune.py $spec > gpurun_out/tune_$name.jsonl 2>&1
done
if [ "${RAGGED_C3:-1}" = 1 ]; then
RAGGED=1 timeout 900 python tools/tune.py softmax f16 64 12 491 491 > gpurun_out/tune_softmax_ragged_f16_491.jsonl 2>&1
fi
