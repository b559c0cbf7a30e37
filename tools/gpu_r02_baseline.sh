# BASELINE.md §4 evidence: sweep (time, GB/s, % peak, % nominal, max err), one ncu
# launch per case (DRAM bytes), oracle rows/s on 1 and all host threads.
set -x
mkdir -p gpurun_out/bl
timeout 1200 python tools/sweep.py > gpurun_out/bl/sweep.jsonl 2> gpurun_out/bl/sweep.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"softmax_|ln_" --csv --log-file gpurun_out/bl/ncu.csv python tools/baseline_cases.py --ncu > gpurun_out/bl/ncu_cases.jsonl 2> gpurun_out/bl/ncu.err
timeout 900 python tools/baseline_cases.py --oracle > gpurun_out/bl/oracle.jsonl 2> gpurun_out/bl/oracle.err
lscpu > gpurun_out/bl/lscpu.txt 2>&1
ls -la gpurun_out/bl
