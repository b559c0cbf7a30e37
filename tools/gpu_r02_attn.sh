# Round 2: parity of every attention variant (tuning build: 1..9) and timings.
set -x
mkdir -p gpurun_out/attn
TT_LIB_PATH=paper_2010_05680_b200/libtt_tune.so timeout 900 python -m pytest tests/test_parity_attention.py tests/test_pdl.py -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/attn/pytest_tune.txt
timeout 600 python -m pytest tests/test_parity_attention.py -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/attn/pytest_prod.txt
timeout 600 python tools/attn_bench.py > gpurun_out/attn/bench.jsonl 2> gpurun_out/attn/bench.err
tail -3 gpurun_out/attn/*.txt; cat gpurun_out/attn/bench.jsonl
