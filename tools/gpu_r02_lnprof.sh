set -x
mkdir -p gpurun_out/lnprof
P="ncu --set full --import-source on --clock-control none -s 2 -c 1"
for spec in "c4 bf16 32768 1024" "c3 f16 31808 768" "c2 f32 10000 768"; do
  set -- $spec; name=$1; shift
  timeout 300 $P -k regex:ln_ -o gpurun_out/lnprof/$name python tools/prof_one.py layernorm "$@" > gpurun_out/lnprof/$name.log 2>&1
  python tools/ncu_summary.py gpurun_out/lnprof/$name.ncu-rep > gpurun_out/lnprof/ncu_$name.txt 2>&1
  python tools/ncu_sass.py gpurun_out/lnprof/$name.ncu-rep 25 > gpurun_out/lnprof/sass_$name.txt 2>&1
  rm -f gpurun_out/lnprof/$name.ncu-rep
done
# torch.add reference under the same capture
cat > /tmp/addref.py <<'PY'
import torch
x = torch.randn(32768, 1024, device="cuda", dtype=torch.bfloat16); r = torch.randn_like(x); o = torch.empty_like(x)
for _ in range(5): torch.add(x, r, out=o)
torch.cuda.synchronize()
PY
timeout 300 $P -k regex:elementwise -o gpurun_out/lnprof/addref python /tmp/addref.py > gpurun_out/lnprof/addref.log 2>&1
python tools/ncu_summary.py gpurun_out/lnprof/addref.ncu-rep > gpurun_out/lnprof/ncu_addref.txt 2>&1
rm -f gpurun_out/lnprof/addref.ncu-rep
