set -x
mkdir -p gpurun_out/next2
timeout 900 python -m pytest tests/test_parity_next2.py -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/next2/pytest.txt
timeout 600 python tools/sweep.py --next2 > gpurun_out/next2/sweep.jsonl 2> gpurun_out/next2/sweep.err
python tools/sweep_table.py gpurun_out/next2/sweep.jsonl > gpurun_out/next2/sweep.txt
cat gpurun_out/next2/pytest.txt gpurun_out/next2/sweep.txt
