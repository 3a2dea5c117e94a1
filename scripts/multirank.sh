#!/bin/bash
# Multi-rank bench path on one GPU: 2 ranks share the device (gloo + host
# exchange); checks the max-over-ranks timing and the JSON line of rank 0.
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 --exchange-every 5 --no-cpu-baseline \
  --no-variants > gpurun_out/bench_2rank_shared.json 2> gpurun_out/bench_2rank_shared.err
echo "rc=$?"; tail -c 1500 gpurun_out/bench_2rank_shared.json; tail -3 gpurun_out/bench_2rank_shared.err
