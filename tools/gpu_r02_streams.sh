set -x
mkdir -p gpurun_out/streams
timeout 900 python -m pytest tests/test_parity_layernorm.py tests/test_parity_layernorm_robust.py tests/test_multigpu_bench.py -q -p no:cacheprovider -x 2>&1 | tail -3 > gpurun_out/streams/pytest.txt
for ns in 1 2 3 4; do
  timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --streams $ns > gpurun_out/streams/c5_s$ns.json 2>> gpurun_out/streams/err.txt
  timeout 600 python bench.py --workload c5p --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --streams $ns > gpurun_out/streams/c5p_s$ns.json 2>> gpurun_out/streams/err.txt
done
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/streams/c4.json 2>> gpurun_out/streams/err.txt
