set -u
mkdir -p gpurun_out/v2
timeout 900 python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_parity.py -x -q -k "rnd10k or no_eta or non_integer or headline or grid" > gpurun_out/v2/t_grid.log 2>&1; tail -3 gpurun_out/v2/t_grid.log
ACS_LIB_VARIANT=newdef timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_headline.py -x -q -k "sync or deferred or pr2392 or nrw1379 or config2 or rnd10k or d198 or update_period or philox or q0 or beta or tiny or att" > gpurun_out/v2/t_newdef.log 2>&1; tail -3 gpurun_out/v2/t_newdef.log
python scripts/ab_time.py base newdef --variants deferred --iters 5
python scripts/ab_time.py base lenpass --variants spm
python scripts/lost_updates.py --instances pcb442 rat783 nrw1379 pr2392 --resident 0 128 6 --iterations 100 --out gpurun_out/v2/lost_updates.json
python scripts/large_instances.py --sizes 10000 14051 --ants 256 0 --iters 3 --out gpurun_out/v2/large.json
ACS_NO_GRID=1 python scripts/large_instances.py --sizes 10000 14051 --ants 256 0 --iters 3 --variants relaxed --out gpurun_out/v2/large_nogrid.json
