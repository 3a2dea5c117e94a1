#!/bin/bash
# Colonies of m = 256 (the paper's best-quality setting) use ~1.7 warps per SM,
# so several island colonies fit on ONE B200: 1, 2, 4, 8 ranks sharing the GPU
# (gloo + host exchange every 10 iterations), pr2392, relaxed and spm (k = 4).
mkdir -p gpurun_out/isl256
for v in relaxed spm; do
  for N in 1 2 4 8; do
    if [ $N = 1 ]; then
      timeout 600 python bench.py --variant $v --ants 256 --k 4 --steps 20 --warmup 3 --no-cpu-baseline \
        --no-variants --no-e2e > gpurun_out/isl256/${v}_n$N.json 2> gpurun_out/isl256/${v}_n$N.err
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $((29600 + N)) bench.py --gpus $N --variant $v --ants 256 --k 4 --steps 20 --warmup 3 \
        --exchange-every 10 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/isl256/${v}_n$N.json \
        2> gpurun_out/isl256/${v}_n$N.err
    fi
    python -c "
import json; d=json.load(open('gpurun_out/isl256/${v}_n$N.json')); print('$v', 'colonies=$N', round(d['value']), 'tours/s', d['ms_per_step'], 'ms/step')" || tail -3 gpurun_out/isl256/${v}_n$N.err
  done
done
