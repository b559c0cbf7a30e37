# Round-2 first GPU pass: smoke, GPU tests, then counter evidence for the
# sub-80 % shapes, the sweep and the bench lines (tools/gpu_r02_prof.sh).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
tail -4 gpurun_out/pytest_gpu.txt
bash tools/gpu_r02_prof.sh
