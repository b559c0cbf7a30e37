# End-of-round pass: GPU tests, smoke, reference arm, C5 stream, then the profile refresh.
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python tools/pdl_bench.py > gpurun_out/pdl_bench.jsonl 2>/dev/null
timeout 300 python tools/attn_bench.py > gpurun_out/attn_bench.jsonl 2>/dev/null
bash tools/gpu_prof_c4.sh
