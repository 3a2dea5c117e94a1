#!/bin/bash
# Round profiling pass on the GPU box (run under gpurun from the repo root):
#   1. the default bench line (headline), 2. the ncu launch list of that same
#   command, 3. one ncu --set full capture per construction kernel variant.
set -u
mkdir -p gpurun_out
R=${ROUND:-r01}
timeout 600 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
tail -c 3000 gpurun_out/bench_$R.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$R.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
  > /dev/null 2>&1
for spec in "atomic:k_construct_dense" "relaxed:k_construct_dense" "spm:k_construct_spm" "deferred:k_deferred"; do
  v=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 \
    -o gpurun_out/prof_${R}_$v python bench.py --variant $v --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_${R}_$v.log 2>&1
  tail -1 gpurun_out/ncu_${R}_$v.log
done
