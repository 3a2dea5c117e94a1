#!/bin/bash
# GPU leg of the quality-vs-oracle study at the ORACLE's concurrency: the
# relaxed variants with at most $W ants constructing at once
# (ACS_RESIDENT_ANTS), against tests/studies/oracle_quality.py RELAXED with
# $W threads (scripts/quality_oracle_leg.sh).  Same params: paper values,
# m = n, k = 1, 1000 iterations.
set -u
mkdir -p gpurun_out
W=${W:-6}
for spec in ${SPECS:-d198:30 pcb442:10}; do
  inst=${spec%%:*}; seeds=${spec##*:}
  ACS_RESIDENT_ANTS=$W timeout 3000 python tools/quality.py --instances $inst --variants atomic relaxed spm \
    --seeds $seeds --iterations 1000 --out gpurun_out/qc_w${W}_$inst.json
done
