# ncu --set full of selected tiers (one launch each after 2 warm-up launches).
set -x
P="ncu --set full --import-source on --clock-control none -k regex:softmax_|ln_ -s 2 -c 1"
$P -o gpurun_out/prof_sm_m6 python tools/prof_one.py softmax bf16 64 16 512 512 --tier "softmax_rows<bf16,V32,G32,NV1,R1,T256,M6>" > /dev/null 2>&1
$P -o gpurun_out/prof_sm_tma python tools/prof_one.py softmax bf16 64 16 512 512 --tier "softmax_tma<bf16,V16,G32,NV2,W4>" > /dev/null 2>&1
$P -o gpurun_out/prof_ln_m6 python tools/prof_one.py layernorm bf16 32768 1024 --tier "ln_rows<bf16,V32,G32,NV2,R1,T128,M6>" > /dev/null 2>&1
$P -o gpurun_out/prof_ln_tma python tools/prof_one.py layernorm bf16 32768 1024 --tier "ln_tma<bf16,V16,G32,NV4,W4>" > /dev/null 2>&1
ls -la gpurun_out/
