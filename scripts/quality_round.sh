#!/bin/bash
# 30-seed solution-quality study on the GPU (paper parameters, 1000 iterations, m = n, k = 1)
mkdir -p gpurun_out
R=${ROUND:-r01}
timeout 2400 python tools/quality.py --instances d198 pcb442 rat783 pr1002 nrw1379 pr2392 \
  --variants atomic relaxed spm --seeds 30 --iterations 1000 --out gpurun_out/quality_${R}.json \
  > gpurun_out/quality_${R}.log 2>&1
timeout 1200 python tools/quality.py --instances d198 pcb442 --variants deferred --seeds 30 --iterations 1000 \
  --out gpurun_out/quality_${R}_deferred.json >> gpurun_out/quality_${R}.log 2>&1
cat gpurun_out/quality_${R}.log
