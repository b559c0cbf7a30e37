set -x
mkdir -p gpurun_out/e2e
timeout 120 python tools/pcie_bw.py 512 > gpurun_out/e2e/pcie.json 2>&1
for c in 8 16 32 64; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-chunks $c > gpurun_out/e2e/bench_c$c.json 2> gpurun_out/e2e/bench_c$c.err
done
cat gpurun_out/e2e/pcie.json
for c in 8 16 32 64; do python -c "import json,sys; d=json.load(open('gpurun_out/e2e/bench_c$c.json')); print($c, d['e2e'])"; done
