#!/bin/bash
# SURVEY 8(d) config 3 on the GPU box: equal-time quality (paper time limits)
# for pr1002 / nrw1379, m=256, k=4: GPU SPM and relaxed (Alt*) vs the CPU
# oracle SEQ (1 core) and RELAXED (all host cores).  SEEDS / OSEEDS runs each.
mkdir -p gpurun_out
S=${SEEDS:-5}
OS=${OSEEDS:-2}
for spec in "pr1002:26.39" "nrw1379:56.77"; do
  inst=${spec%%:*}; lim=${spec##*:}
  python tools/quality.py --instances $inst --variants spm relaxed --ants 256 --k 4 --time-limit-s $lim \
    --seeds $S --out gpurun_out/qt_gpu_$inst.json
  python tests/studies/oracle_quality.py run --instances $inst --mode seq --ants 256 --k 4 \
    --time-limit-s $lim --seeds $OS --out gpurun_out/qt_seq_$inst.json
  python tests/studies/oracle_quality.py run --instances $inst --mode relaxed --ants 256 --k 4 \
    --time-limit-s $lim --seeds $OS --out gpurun_out/qt_rel_$inst.json
  python tests/studies/oracle_quality.py compare gpurun_out/qt_gpu_$inst.json gpurun_out/qt_seq_$inst.json \
    gpurun_out/qt_rel_$inst.json --out gpurun_out/qt_cmp_$inst.json
done
