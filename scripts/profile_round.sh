#!/bin/bash
# Round profiling pass on the GPU box (run under gpurun from the repo root):
#   1. the default bench line (headline), 2. the ncu launch list of that same
#   command, 3. one ncu --set full capture per construction kernel variant
#   (k_tour_lean: atomic/relaxed, k_spm_lean: spm, k_deferred: deferred).
set -u
mkdir -p gpurun_out
R=${ROUND:-r02}
timeout 600 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
tail -c 3000 gpurun_out/bench_$R.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$R.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-variants \
  > /dev/null 2>&1
for spec in "atomic:k_tour_lean" "relaxed:k_tour_lean" "spm:k_spm_lean" "deferred:k_deferred"; do
  v=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 \
    -o gpurun_out/prof_${R}_$v python scripts/colony_run.py --variant $v --iters 3 \
    > gpurun_out/ncu_${R}_$v.log 2>&1
  tail -1 gpurun_out/ncu_${R}_$v.log
done
