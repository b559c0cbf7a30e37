mkdir -p gpurun_out/pk
for rep in 1 2; do for r in 4 8 16; do for w in c3p c5p; do
TT_LIB_PATH=paper_2010_05680_b200/libtt_pk$r.so timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/pk/${w}_rpg${r}_$rep.json 2>/dev/null
done; done; done
