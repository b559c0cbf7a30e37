set -x
mkdir -p gpurun_out/mask
timeout 1200 python -m pytest tests/test_parity_softmax.py tests/test_parity_packed.py tests/test_pdl.py -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/mask/pytest.txt
timeout 900 python tools/sweep.py > gpurun_out/mask/sweep.jsonl 2> gpurun_out/mask/sweep.err
python tools/sweep_table.py gpurun_out/mask/sweep.jsonl > gpurun_out/mask/sweep.txt
timeout 600 python bench.py --workload c5p --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/mask/bench_c5p.json 2> gpurun_out/mask/bench.err
timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/mask/bench_c5.json 2>> gpurun_out/mask/bench.err
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/mask/bench.json 2>> gpurun_out/mask/bench.err
cat gpurun_out/mask/pytest.txt
