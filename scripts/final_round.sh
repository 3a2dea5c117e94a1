#!/bin/bash
# End-of-round pass on the GPU box: tests, smoke, headline bench + launch list
# + ncu captures, setup-path timing against the reference code, and the
# spm-sync quality leg.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
R=${ROUND:-r01f}
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/tests_$R.log; tail -2 gpurun_out/tests_$R.log
timeout 600 python __graft_entry__.py > gpurun_out/smoke_$R.log 2>&1; tail -1 gpurun_out/smoke_$R.log
ROUND=$R bash scripts/profile_round.sh
timeout 1200 python scripts/setup_timing.py --out gpurun_out/setup_timing_$R.json > gpurun_out/setup_timing_$R.log 2>&1
tail -8 gpurun_out/setup_timing_$R.log
if [ "${QUALITY:-1}" = "1" ]; then
  timeout 1500 python tools/quality.py --instances d198 pcb442 --variants spm-sync --seeds 30 --iterations 1000 \
    --out gpurun_out/q_spm_sync_$R.json
fi
