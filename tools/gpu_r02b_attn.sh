set -x
mkdir -p gpurun_out/attn3
timeout 300 python tools/attn_trace_p.py > gpurun_out/attn3/trace_p.json 2>&1
cat gpurun_out/attn3/trace_p.json
