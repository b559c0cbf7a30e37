set -x
mkdir -p gpurun_out/lnwave
timeout 1200 python -m pytest tests/test_parity_layernorm.py tests/test_parity_layernorm_robust.py tests/test_abi.py -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/lnwave/pytest.txt
export TT_LIB_PATH=paper_2010_05680_b200/libtt.so
for rows in 5600 6000 6500 7000 7500; do
timeout 600 python tools/tune.py layernorm f16 $rows 768 > gpurun_out/lnwave/tune_f16_$rows.jsonl 2>/dev/null
done
cat gpurun_out/lnwave/pytest.txt
