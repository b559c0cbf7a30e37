set -x
mkdir -p gpurun_out/ln2
for spec in "bf16 32768 1024" "f16 31808 768" "f32 10000 768" "f16 10000 768"; do
  set -- $spec
  ONLY=ln_rows TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 300 python tools/tune.py layernorm $spec > gpurun_out/ln2/tune_$1_$2_$3.jsonl 2>&1
done
