#!/bin/bash
# A/B of the pruned-fallback slice batch (ACS_EXT_BATCH / ACS_EXT_BATCH_DEFER):
# construct ms per launch at pr2392, two alternating passes.
set -u
for pass in 1 2; do
  python scripts/ab_time.py base ${LIBS:-d6 e1} --variants atomic relaxed spm deferred --iters ${ITERS:-30}
done
