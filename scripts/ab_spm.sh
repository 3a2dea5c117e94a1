#!/bin/bash
# A/B of SPM kernel builds on the GPU box: spm tests on the base build, construct
# times (ab_time.py) and executed instructions of k_spm_lean per build.
#   LIBS="old" bash scripts/ab_spm.sh
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "spm" 2>&1 | tail -2
python scripts/ab_time.py base ${LIBS:-} --variants spm --iters 20
for lib in base ${LIBS:-}; do
  if [ "$lib" = base ]; then export ACS_LIB_VARIANT=; else export ACS_LIB_VARIANT=$lib; fi
  timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:k_spm_lean -s 2 -c 1 --csv \
    python scripts/colony_run.py --variant spm --iters 3 2>/dev/null | grep -E "inst_executed|duration" | awk -F'","' -v l=$lib '{print l, $(NF-2), $NF}'
done
