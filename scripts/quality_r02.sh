#!/bin/bash
# Round-2 quality parity legs on the GPU box (north_star tolerance):
#   PART=1: lost-update rates (instrumented build), full concurrency and W=128
#           residency (the paper's GK104: one 32-thread block per ant, ~128 in
#           flight), nrw1379 / pr2392, m = n, 1000 and 100 iterations, 30 seeds
#   PART=2: W=6 legs on pcb442 / rat783, 30 seeds (round 1 had 10)
set -u
O=gpurun_out/q02
mkdir -p $O
if [ "${PART:-1}" = "1" ]; then
  python scripts/lost_updates.py --instances pcb442 rat783 nrw1379 pr2392 --resident 0 128 6 --iterations 100 \
    --out $O/lost_updates.json
  for inst in nrw1379 pr2392; do
    ACS_RESIDENT_ANTS=0 python tools/quality.py --instances $inst --variants relaxed atomic spm --seeds 30 \
      --iterations 1000 --rng philox --out $O/q_${inst}_Wall_it1000.json
    ACS_RESIDENT_ANTS=128 python tools/quality.py --instances $inst --variants relaxed atomic spm --seeds 30 \
      --iterations 100 --rng philox --out $O/q_${inst}_W128_it100.json
    ACS_RESIDENT_ANTS=128 python tools/quality.py --instances $inst --variants relaxed atomic spm --seeds 30 \
      --iterations 1000 --rng philox --out $O/q_${inst}_W128_it1000.json
  done
fi
if [ "${PART:-1}" = "2" ]; then
  for inst in pcb442 rat783; do
    ACS_RESIDENT_ANTS=6 python tools/quality.py --instances $inst --variants atomic relaxed spm --seeds 30 \
      --iterations 1000 --rng philox --out $O/q_${inst}_W6_it1000.json
  done
fi
