# ncu --set full of selected tiers: PROF="name|op dtype dims|tier;..." (one launch after 2 warm-ups)
set -x
P="ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-softmax_|ln_} -s 2 -c 1"
IFS=';' read -ra JOBS <<< "$PROF"
for j in "${JOBS[@]}"; do
  IFS='|' read -r name spec tier extra <<< "$j"
  if [ -n "$tier" ]; then
    $P -o gpurun_out/prof_$name python tools/prof_one.py $spec --tier "$tier" $extra > gpurun_out/prof_$name.log 2>&1
  else
    $P -o gpurun_out/prof_$name python tools/prof_one.py $spec $extra > gpurun_out/prof_$name.log 2>&1
  fi
done
ls -la gpurun_out/
