# PDL pass: full GPU tests, launch-bound step timing with PDL on/off, bench line
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python tools/pdl_bench.py > gpurun_out/pdl_bench.jsonl 2> gpurun_out/pdl_bench.err
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
