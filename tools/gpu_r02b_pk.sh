set -x
mkdir -p gpurun_out/pk2
P="ncu --set full --import-source on --clock-control none -s 2 -c 1"
timeout 300 $P -k regex:softmax_packed -o gpurun_out/pk2/prof_pk python tools/prof_one.py packed f16 12 > gpurun_out/pk2/prof_pk.log 2>&1
python tools/ncu_summary.py gpurun_out/pk2/prof_pk.ncu-rep > gpurun_out/pk2/ncu_pk.txt 2>&1
python tools/ncu_sass.py gpurun_out/pk2/prof_pk.ncu-rep 30 > gpurun_out/pk2/sass_pk.txt 2>&1
ncu -i gpurun_out/pk2/prof_pk.ncu-rep --page source --csv --print-source sass > gpurun_out/pk2/src_pk.csv 2>/dev/null
rm -f gpurun_out/pk2/prof_pk.ncu-rep
