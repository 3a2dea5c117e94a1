#!/bin/bash
ABS="lf lfany" VARIANTS="atomic relaxed" bash scripts/ab.sh
timeout 900 python tools/quality.py --instances a280 pcb442 rat783 --variants spm relaxed atomic --seeds 10 \
  --iterations 1000 --ants 256 --k 4 --out gpurun_out/quality_r01_m256k4.json 2>&1 | tail -12
