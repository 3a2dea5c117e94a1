#!/bin/bash
# Reproduce the paper's m-sweep / k-sweep tables on the GPU.  The paper fixes
# the BUDGET, not the iteration count: b = 1000 n solutions, so a colony of m
# ants runs b / m iterations.
#   PAPER.md:1170-1186  ACS-GPU-Alt (relaxed), m = 256, k in {1,2,4,8,16}, nrw1379 / pr2392
#   PAPER.md:1211-1240  ACS-GPU-SPM, m = 256, same k sweep (figure; k = 16: 3.72 / 4.66 %)
#   PAPER.md:1136-1146  ACS-GPU-Alt, k = 1, m in {128, 512, 1024}
set -u
mkdir -p gpurun_out
S=${SEEDS:-10}
S0=${SEED0:-0}
TAG=${TAG:-qb}
M=${ANTS:-256}
VARS=${VARS:-relaxed spm}
for spec in ${SPECS:-nrw1379:1379 pr2392:2392}; do
  inst=${spec%%:*}; n=${spec##*:}
  for k in ${KS:-1 2 4 8 16}; do
    python tools/quality.py --instances $inst --variants $VARS --ants $M --k $k --seeds $S --seed0 $S0 \
      --iterations $((1000 * n / M)) --out gpurun_out/${TAG}_${inst}_m${M}_k$k.json
  done
  for m in ${MS-128 512 1024}; do
    python tools/quality.py --instances $inst --variants relaxed --ants $m --k 1 --seeds $S --seed0 $S0 \
      --iterations $((1000 * n / m)) --out gpurun_out/${TAG}_${inst}_m${m}_k1.json
  done
done
