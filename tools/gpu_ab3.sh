# A/B/C of library builds (TT_LIB_PATH) on tuned shapes: LIBS="name=path ...";
# SPECS entries prefixed R: run with ragged lengths, C3: with the C3 lengths
mkdir -p gpurun_out/ab3
SPECS=${SPECS:-"layernorm f16 31808 768;layernorm bf16 32768 1024;layernorm f16 10000 768;softmax f16 20 12 128 128;softmax bf16 64 16 512 512"}
IFS=';' read -ra LIST <<< "$SPECS"
for rep in 1 2; do
for spec in "${LIST[@]}"; do
  rg=0; case "$spec" in R:*) rg=1; spec=${spec#R:};; C3:*) rg=c3; spec=${spec#C3:};; esac
  name=$(echo $spec | tr ' ' '_')_r$rg
  for lib in $LIBS; do
    n=${lib%%=*}; p=${lib#*=}
    RAGGED=$rg ONLY=xx TT_LIB_PATH=$p timeout 300 python tools/tune.py $spec > gpurun_out/ab3/${n}_${name}_$rep.jsonl 2>&1
  done
done
done
if [ "${BENCH:-0}" = 1 ]; then
for rep in 1 2; do for lib in $LIBS; do
  n=${lib%%=*}; p=${lib#*=}
  TT_LIB_PATH=$p timeout 300 python bench.py --steps 500 --warmup 10 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab3/bench_${n}_$rep.json 2>/dev/null
done; done
fi
