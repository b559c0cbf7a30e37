# Round-2 counter evidence for the shapes under 80 % (VERDICT r01 "what's missing" 3):
# one ncu --set full capture per shape, summarised on the box (the .ncu-rep embeds
# the whole fatbin), plus the sweep of every BASELINE shape.
set -x
mkdir -p gpurun_out
RND=${RND:-r02}
P="ncu --set full --import-source on --clock-control none -s 2 -c 1"
run() {  # name kregex args...
  name=$1; kre=$2; shift 2
  timeout 300 $P -k regex:$kre -o gpurun_out/prof_$name python tools/prof_one.py "$@" > gpurun_out/prof_$name.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_$name.ncu-rep > gpurun_out/${RND}_ncu_$name.txt 2>&1
  python tools/ncu_sass.py gpurun_out/prof_$name.ncu-rep 25 > gpurun_out/${RND}_sass_$name.txt 2>&1
  rm -f gpurun_out/prof_$name.ncu-rep
}
if [ "${PROF:-1}" = 1 ]; then
run c3_f16_sm softmax_ softmax f16 12 --c3
run c2_f16_s300_ragged_sm softmax_ softmax f16 20 12 300 300 --ragged
run c2_f16_s256_full_sm softmax_ softmax f16 20 12 256 256
run c2_f32_s300_ln ln_ layernorm f32 6000 768
run c4_bf16_ln ln_ layernorm bf16 32768 1024
run c3_f16_ln ln_ layernorm f16 31488 768
fi
if [ "${SWEEP:-1}" = 1 ]; then
timeout 1200 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
fi
if [ "${BENCH:-1}" = 1 ]; then
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c5.json 2>> gpurun_out/bench.err
fi
ls -la gpurun_out
