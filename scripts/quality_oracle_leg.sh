#!/bin/bash
# CPU oracle leg of the quality-vs-reference study (paper parameters, m = n,
# k = 1, 1000 iterations, seeds 0..S-1), one oracle mode per GPU variant:
#   atomic  -> RELAXED + consistent (no lost update)     relaxed -> RELAXED
#   spm     -> RELAXED + selective memory                 seq     -> SEQ (ACS-SEQ)
# The GPU leg is profiles/quality_r01_gpu*.json (tools/quality.py, same settings);
# scripts/quality_compare.py puts the two side by side with the rank-sum test.
# Runs on any host (the oracle is CPU code):  THREADS=6 bash scripts/quality_oracle_leg.sh
set -eu
OUT=${OUT:-profiles/quality_oracle_r01}
S=${SEEDS:-30}
T=${THREADS:-0}
mkdir -p $OUT
for inst in ${INSTANCES:-d198 pcb442 rat783}; do
  python tests/studies/oracle_quality.py run --instances $inst --mode relaxed --consistent --seeds $S \
    --threads $T --iterations 1000 --out $OUT/orc_atomic_$inst.json
  python tests/studies/oracle_quality.py run --instances $inst --mode relaxed --seeds $S \
    --threads $T --iterations 1000 --out $OUT/orc_relaxed_$inst.json
  python tests/studies/oracle_quality.py run --instances $inst --mode relaxed --memory selective --seeds $S \
    --threads $T --iterations 1000 --out $OUT/orc_spm_$inst.json
done
