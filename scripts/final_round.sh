#!/bin/bash
# End-of-round pass on the GPU box: tests, smoke, headline bench + launch list
# + ncu captures (profile_round.sh), the reference arm, the two-rank bench path
# (ranks sharing the GPU), setup timing.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
R=${ROUND:-r02f}
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/tests_$R.log; tail -2 gpurun_out/tests_$R.log
timeout 600 python __graft_entry__.py > gpurun_out/smoke_$R.log 2>&1; tail -1 gpurun_out/smoke_$R.log
ROUND=$R bash scripts/profile_round_box.sh
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err
tail -c 800 gpurun_out/bench_ref_$R.json
bash scripts/multirank.sh
python scripts/create_timing.py --instance pr2392 > gpurun_out/create_$R.log 2>&1; cat gpurun_out/create_$R.log
