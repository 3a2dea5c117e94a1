for v in atomic relaxed spm deferred; do timeout 300 python bench.py --variant $v --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_$v.json 2>gpurun_out/b_$v.err; python -c "import json,sys; d=json.load(open('gpurun_out/b_$v.json')); print(d['config']['variant'], d['value'], d['roofline']['construct_ms_per_launch'], d['clocks'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_atomic.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_construct_dense -s 1 -c 1 -o gpurun_out/prof_atomic python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
