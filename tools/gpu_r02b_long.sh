set -x
mkdir -p gpurun_out/long
timeout 1200 python -m pytest tests/test_parity_softmax.py tests/test_abi.py -q -x -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/long/pytest3.txt
timeout 300 python tools/long_rows.py > gpurun_out/long/timing3.jsonl 2>&1
cat gpurun_out/long/pytest3.txt gpurun_out/long/timing3.jsonl
