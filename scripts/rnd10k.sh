#!/bin/bash
# rnd10k throughput per variant, m = n and m = 256
mkdir -p gpurun_out
for v in ${VARIANTS:-atomic relaxed spm deferred}; do
  for m in ${ANTS:-0 256}; do
    timeout 600 python bench.py --instance rnd10k --variant $v --ants $m --k ${K:-1} --steps ${STEPS:-5} --warmup 3 \
      --no-cpu-baseline --no-e2e --no-variants > gpurun_out/rnd_${v}_$m.json 2> gpurun_out/rnd_${v}_$m.err
    python -c "
import json,sys
try:
    d=json.load(open('gpurun_out/rnd_${v}_$m.json')); c=d['counters_per_step']
    print('$v m=$m', d['value'], 'tours/s', d['ms_per_step'], 'ms/it construct', d['roofline']['construct_ms_per_launch'], 'fb', c['fallback_steps'], 'full', c.get('fallback_full'), 'best', d['quality']['best_len'])
except Exception as e: print('$v $m failed', e, open('gpurun_out/rnd_${v}_$m.err').read()[-1500:])
"
  done
done
