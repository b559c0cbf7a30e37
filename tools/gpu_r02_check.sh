# Round 2: GPU tests + sweep + bench on the current product build.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
tail -5 gpurun_out/pytest_gpu.txt
if [ "${SWEEP:-1}" = 1 ]; then timeout 1200 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; fi
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
