set -u
mkdir -p gpurun_out/v4
ACS_LIB_VARIANT=lost python -c "
import sys; sys.path.insert(0,'.')
import paper_1605_02669_b200 as P
inst=P.load_instance('d198')
for m in (1, 2, 8):
    with P.Colony(inst, P.AcsParams(variant='relaxed', m=m, seed=1, rng='philox')) as col:
        col.iterate(5); c=col.counters(); print('m', m, 'writes', c['relaxed_writes'], 'lost', c['lost_updates'])
"
timeout 900 python -m pytest tests/test_gpu_parity_headline.py tests/test_gpu_parity.py -x -q -k "rnd10k or no_eta or non_integer or grid or sync or deferred" 2>&1 | tail -2
python scripts/lost_updates.py --instances pcb442 rat783 nrw1379 pr2392 --resident 0 128 6 --iterations 100 --out gpurun_out/v4/lost_updates.json
