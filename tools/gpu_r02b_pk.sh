set -x
mkdir -p gpurun_out/pk
P="ncu --set full --import-source on --clock-control none -s 2 -c 1"
timeout 300 $P -k regex:softmax_packed -o gpurun_out/pk/prof_pk python tools/prof_one.py packed f16 12 > gpurun_out/pk/prof_pk.log 2>&1
python tools/ncu_summary.py gpurun_out/pk/prof_pk.ncu-rep > gpurun_out/pk/ncu_pk.txt 2>&1
python tools/ncu_sass.py gpurun_out/pk/prof_pk.ncu-rep 40 > gpurun_out/pk/sass_pk.txt 2>&1
rm -f gpurun_out/pk/prof_pk.ncu-rep
