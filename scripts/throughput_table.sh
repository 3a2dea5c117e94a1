#!/bin/bash
# Throughput of every variant on every TSPLIB config instance (m = n, k = 1),
# bench.py's own timing (L2 flushed, CUDA events, 20 steps after 3 warm-up).
mkdir -p gpurun_out/tput
for inst in ${INSTANCES:-d198 pcb442 rat783 pr1002 nrw1379 pr2392}; do
  for v in ${VARIANTS:-atomic relaxed spm deferred}; do
    timeout 300 python bench.py --instance $inst --variant $v --steps ${STEPS:-20} --warmup 3 \
      --no-cpu-baseline --no-variants --no-e2e > gpurun_out/tput/${inst}_$v.json 2> gpurun_out/tput/${inst}_$v.err
  done
done
python - <<'PY'
import json, glob, os
rows = []
for f in sorted(glob.glob("gpurun_out/tput/*.json")):
    try:
        d = json.load(open(f))
    except Exception:
        continue
    r = d["roofline"]
    rows.append((d["config"]["instance"], d["config"]["variant"], d["ms_per_step"], d["value"],
                 r["latency"]["frac"], r["latency"]["isolated_ant"]["frac_colony"], r["frac"]))
for x in rows:
    print("%-8s %-9s %8.3f ms/it %12.0f tours/s  floor frac %.2f  isolated-ant frac %.2f  l2 %.3f" % x)
PY
