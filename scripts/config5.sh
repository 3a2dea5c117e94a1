#!/bin/bash
# SURVEY 8(d) config 5 on one GPU: rnd10k with k = 4 (m = n and 256), and the
# island path with 2 ranks sharing the GPU (host exchange every X iterations).
mkdir -p gpurun_out/cfg5
[ "${SKIP_K4:-0}" = "1" ] || K=4 bash scripts/rnd10k.sh > gpurun_out/cfg5/rnd10k_k4.log 2>&1; cat gpurun_out/cfg5/rnd10k_k4.log
mkdir -p gpurun_out/cfg5k4 && cp gpurun_out/rnd_*.json gpurun_out/cfg5k4/ 2>/dev/null
for X in 10 50; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29540 + X)) bench.py --gpus 2 --instance rnd10k --variant relaxed --steps 10 --warmup 3 \
    --exchange-every $X --no-cpu-baseline --no-variants > gpurun_out/cfg5/island2_x$X.json 2> gpurun_out/cfg5/island2_x$X.err
  python -c "
import json; d=json.load(open('gpurun_out/cfg5/island2_x$X.json')); print('X=$X', d['n_gpus'], d['value'], d['ms_per_step'], d['config']['exchange'], d['quality']['best_len'])"
done
