#!/bin/bash
# Round-2 quality parity legs on the GPU box (north_star tolerance).
# Every (instance, variant, residency) leg writes its own JSON, so a leg cut by
# the call's time limit loses only itself.
#   LEGS="pr2392:relaxed:128:1000 ..."  instance:variant:resident ants (0 = all):iterations
set -u
O=gpurun_out/q02
mkdir -p $O
for leg in ${LEGS}; do
  IFS=: read -r inst v w it <<< "$leg"
  out=$O/q_${inst}_${v}_W${w}_it${it}.json
  [ -f "$out" ] && continue
  ACS_RESIDENT_ANTS=$w timeout 3000 python tools/quality.py --instances $inst --variants $v --seeds 30 \
    --iterations $it --rng philox --out $out
done
