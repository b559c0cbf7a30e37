mkdir -p gpurun_out/attn
for v in 9 0; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention -s 2 -c 1 -o gpurun_out/attn/prof_v$v python tools/prof_one.py attention bf16 64 16 512 --tier $v > gpurun_out/attn/prof_v$v.log 2>&1
python tools/ncu_summary.py gpurun_out/attn/prof_v$v.ncu-rep > gpurun_out/attn/ncu_v$v.txt 2>&1
python tools/ncu_sass.py gpurun_out/attn/prof_v$v.ncu-rep 30 > gpurun_out/attn/sass_v$v.txt 2>&1
rm -f gpurun_out/attn/prof_v$v.ncu-rep
done
