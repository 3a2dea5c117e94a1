#!/bin/bash
# Quality tolerance vs the CPU oracle, per pheromone variant (north_star:
# "mean and best % over optimum across 30 seeds within a stated tolerance of
# the reference"): GPU variant and the oracle's matching mode, same settings
# (paper parameters, m = n, k = 1, 1000 iterations), rank-sum compared.
mkdir -p gpurun_out
for spec in "d198:30:30" "pcb442:30:${PCB_OSEEDS:-8}"; do
  inst=${spec%%:*}; rest=${spec#*:}; gs=${rest%%:*}; os=${rest##*:}
  python tools/quality.py --instances $inst --variants atomic relaxed spm deferred --seeds $gs \
    --iterations 1000 --out gpurun_out/qo_gpu_$inst.json
  python tests/studies/oracle_quality.py run --instances $inst --mode relaxed --consistent --seeds $os \
    --iterations 1000 --out gpurun_out/qo_orc_atomic_$inst.json
  python tests/studies/oracle_quality.py run --instances $inst --mode relaxed --seeds $os \
    --iterations 1000 --out gpurun_out/qo_orc_relaxed_$inst.json
  python tests/studies/oracle_quality.py run --instances $inst --mode relaxed --memory selective --seeds $os \
    --iterations 1000 --out gpurun_out/qo_orc_spm_$inst.json
done
