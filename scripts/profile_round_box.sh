#!/bin/bash
# profile_round.sh, then the ncu reports reduced on the box (summary JSON + top
# SASS lines) so gpurun_out stays under the copy-back limit.
set -u
R=${ROUND:-r02g}
ROUND=$R bash scripts/profile_round.sh
mkdir -p gpurun_out/sum_$R
for v in atomic relaxed spm deferred; do
  b=$(python -c "
import sys; sys.path.insert(0,'.'); import bench
print(bench.algorithmic_bytes_per_tour(2392,32,1,'$v')*2392)")
  python scripts/ncu_summary.py gpurun_out/prof_${R}_$v.ncu-rep --label $v --bytes-per-launch $b \
    --json gpurun_out/sum_$R/ncu_construct_summary.json > /dev/null
  ncu -i gpurun_out/prof_${R}_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/sum_$R/sass_$v.csv 2>/dev/null
  python scripts/ncu_sass.py gpurun_out/sum_$R/sass_$v.csv 25 > gpurun_out/sum_$R/ncu_${R}_${v}_top_sass.txt
  rm -f gpurun_out/sum_$R/sass_$v.csv gpurun_out/prof_${R}_$v.ncu-rep
done
ls -la gpurun_out gpurun_out/sum_$R
