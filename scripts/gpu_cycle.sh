#!/bin/bash
# One measure cycle on the GPU box (run under gpurun from the repo root):
#   TESTS=1     pytest -m gpu
#   VARIANTS    bench variants to time (default "atomic relaxed spm deferred")
#   PROF        kernel regex for one ncu --set full capture (empty = skip)
#   PROF_VARIANT bench variant used for the ncu capture (default atomic)
#   TAG         suffix of the output files
set -u
mkdir -p gpurun_out
TAG=${TAG:-run}
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/tests_$TAG.log
  tail -3 gpurun_out/tests_$TAG.log
fi
for v in ${VARIANTS:-atomic relaxed spm deferred}; do
  timeout 300 python bench.py --variant $v --steps ${STEPS:-5} --warmup 2 --no-cpu-baseline --no-e2e \
    > gpurun_out/b_${TAG}_$v.json 2> gpurun_out/b_${TAG}_$v.err
  python - <<EOF
import json
try:
    d = json.load(open('gpurun_out/b_${TAG}_$v.json'))
    print('$v', d['value'], 'tours/s', d['roofline']['construct_ms_per_launch'], 'ms/construct', d['ms_per_step'], 'ms/step', d['clocks'])
except Exception as e:
    print('$v failed', e, open('gpurun_out/b_${TAG}_$v.err').read()[-2000:])
EOF
done
if [ -n "${PROF:-}" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --variant ${PROF_VARIANT:-atomic} --steps 3 --warmup 1 \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$PROF" -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --variant ${PROF_VARIANT:-atomic} --steps 1 --warmup 1 \
    --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
  tail -2 gpurun_out/ncu_$TAG.log
fi
