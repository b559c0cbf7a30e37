# Round profile of the bench step: bench line, ncu launch list (cold-cache,
# serialised) and one ncu --set full capture of each bench kernel.
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"softmax_|ln_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 10 --e2e-steps 0 --no-cpu-baseline --kernel-events 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"softmax_|ln_" -s 20 -c 2 -o gpurun_out/prof_c4 python bench.py --steps 5 --warmup 10 --e2e-steps 0 --no-cpu-baseline --kernel-events 0 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
if [ "${SWEEP:-1}" = 1 ]; then
timeout 1200 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python tools/sweep.py --next2 > gpurun_out/sweep_next2.jsonl 2>> gpurun_out/sweep.err
fi
# summarise on the box (the .ncu-rep embeds the whole fatbin and exceeds gpurun's copy-back cap)
python tools/make_profiles.py r01 > gpurun_out/make_profiles.log 2>&1
mkdir -p gpurun_out/profiles_box && cp profiles/r01_launches.csv profiles/r01_ncu_full.txt profiles/r01_sass_c4.txt profiles/r01_bench.json profiles/traffic.json gpurun_out/profiles_box/ 2>/dev/null
cp profiles/r01_sweep.txt profiles/r01_sweep_next2.txt gpurun_out/profiles_box/ 2>/dev/null
rm -f gpurun_out/prof_c4.ncu-rep
