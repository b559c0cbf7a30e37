# compute-sanitizer over tools/sanitize_cases.py: product and tuning builds,
# memcheck / racecheck / synccheck / initcheck.
set -x
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for lib in libtt.so libtt_tune.so; do
  for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    TT_LIB_PATH=paper_2010_05680_b200/$lib timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py > gpurun_out/sanitize/${lib%.so}_$tool.log 2>&1
    echo "$lib $tool rc=$?" >> gpurun_out/sanitize/summary.txt
  done
done
cat gpurun_out/sanitize/summary.txt
