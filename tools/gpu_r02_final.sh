# Round-2 final evidence: GPU tests on both builds, sanitizer, bench lines
# (C4 + C5 sub-record, C5 stream, oracle arm), ncu launch list + full capture of
# the bench kernels (profiles/traffic.json), sweeps, BASELINE table inputs.
set -x
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/final/pytest_gpu.txt
TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 1500 python -m pytest tests/test_parity_attention.py tests/test_parity_softmax.py::test_every_compiled_tier tests/test_parity_layernorm_robust.py::test_robust_cases_on_every_compiled_tier tests/test_pdl.py -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/final/pytest_tune.txt
if [ "${SAN:-1}" = 1 ]; then bash tools/gpu_r02_sanitize.sh > gpurun_out/final/sanitize.log 2>&1; fi
timeout 900 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/final/bench.err
cp gpurun_out/bench.json gpurun_out/final/bench.json
timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/final/bench_c5.json 2>> gpurun_out/final/bench.err
timeout 600 python bench.py --workload c5p --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/final/bench_c5p.json 2>> gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.json 2>> gpurun_out/final/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"softmax_|ln_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 10 --e2e-steps 0 --no-cpu-baseline --kernel-events 0 --c5-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"softmax_|ln_" -s 20 -c 2 -o gpurun_out/prof_c4 python bench.py --steps 5 --warmup 10 --e2e-steps 0 --no-cpu-baseline --kernel-events 0 --c5-steps 0 > gpurun_out/ncu_full.log 2>&1
timeout 1200 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python tools/sweep.py --next2 > gpurun_out/sweep_next2.jsonl 2>> gpurun_out/sweep.err
python tools/make_profiles.py r02 > gpurun_out/make_profiles.log 2>&1
python tools/sweep_table.py gpurun_out/sweep.jsonl > profiles/r02_sweep.txt
python tools/sweep_table.py gpurun_out/sweep_next2.jsonl > profiles/r02_sweep_next2.txt
mkdir -p gpurun_out/profiles_box && cp profiles/r02_launches.csv profiles/r02_ncu_full.txt profiles/r02_sass_*.txt profiles/r02_bench.json profiles/traffic.json profiles/r02_sweep.txt profiles/r02_sweep_next2.txt gpurun_out/profiles_box/ 2>/dev/null
rm -f gpurun_out/prof_c4.ncu-rep
tail -n 3 gpurun_out/final/pytest_gpu.txt gpurun_out/final/pytest_tune.txt
