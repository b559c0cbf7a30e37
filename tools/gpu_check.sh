# One gpurun pass: smoke, GPU tests, bench, optional tier sweep and ncu.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
tail -4 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "${TUNE:-1}" = 1 ]; then bash tools/gpu_tune.sh; fi
if [ "${NCU:-0}" = 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"softmax_|ln_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 10 --e2e-steps 0 --no-cpu-baseline --kernel-events 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"softmax_|ln_" -s 20 -c 2 -o gpurun_out/prof_c4 python bench.py --steps 5 --warmup 10 --e2e-steps 0 --no-cpu-baseline --kernel-events 0 > gpurun_out/ncu_full.log 2>&1
fi
