# Round 2 full validation: smoke, every GPU test (product build), the tuning
# build's attention variants, compute-sanitizer on both builds, bench lines.
set -x
mkdir -p gpurun_out/full gpurun_out/sanitize
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/full/pytest_gpu.txt
TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 900 python -m pytest tests/test_parity_attention.py tests/test_pdl.py -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/full/pytest_tune_attn.txt
if [ "${SAN:-1}" = 1 ]; then bash tools/gpu_r02_sanitize.sh > gpurun_out/full/sanitize.log 2>&1; fi
timeout 900 python bench.py --steps 500 --warmup 10 > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err
timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/full/bench_c5.json 2>> gpurun_out/full/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/full/bench_ref.json 2>> gpurun_out/full/bench.err
tail -3 gpurun_out/full/pytest_gpu.txt
