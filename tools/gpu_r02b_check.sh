# Round 2 (re-entry): HEAD verification on a fresh box -- smoke, GPU tests,
# bench line, attention baseline timings and a source-level ncu capture of the
# default attention kernel.
set -x
mkdir -p gpurun_out/chk
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/chk/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/chk/bench.json 2> gpurun_out/chk/bench.err
timeout 300 python tools/attn_quick.py 0 12 13 14 > gpurun_out/chk/attn.jsonl 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:attention -s 2 -c 1 -o gpurun_out/chk/prof_attn python tools/prof_one.py attention bf16 64 16 512 > gpurun_out/chk/prof_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/chk/prof_attn.ncu-rep > gpurun_out/chk/ncu_attn.txt 2>&1
python tools/ncu_sass.py gpurun_out/chk/prof_attn.ncu-rep 60 > gpurun_out/chk/sass_attn.txt 2>&1
ncu -i gpurun_out/chk/prof_attn.ncu-rep --page source --csv --print-source sass > gpurun_out/chk/attn_source.csv 2>/dev/null
rm -f gpurun_out/chk/prof_attn.ncu-rep
tail -3 gpurun_out/chk/pytest_gpu.txt; cat gpurun_out/chk/bench.json gpurun_out/chk/attn.jsonl
