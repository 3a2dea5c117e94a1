#!/bin/bash
# A/B timing of in-tree library builds: ABS="lf lfany" VARIANTS="atomic relaxed" bash scripts/ab.sh
for lib in base ${ABS:-}; do
  for v in ${VARIANTS:-atomic relaxed}; do
    if [ "$lib" = base ]; then export ACS_LIB_VARIANT=; else export ACS_LIB_VARIANT=$lib; fi
    timeout 300 python bench.py --variant $v --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e --no-variants ${BENCH_ARGS:-} \
      | python -c "import json,sys; d=json.load(sys.stdin); c=d.get('counters_per_step',{}); print('$lib', '$v', d['roofline']['construct_ms_per_launch'], d['ms_per_step'], 'fb', c.get('fallback_steps'), 'full', c.get('fallback_full'))"
  done
done
