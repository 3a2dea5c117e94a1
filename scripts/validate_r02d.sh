set -u
timeout 1200 python -m pytest tests/test_golden.py tests/test_gpu_instance.py tests/test_gpu_parity.py -x -q -k "not studies" 2>&1 | tail -2
python scripts/create_timing.py --instance pr2392
ACS_NN_GLOBAL=1 python scripts/create_timing.py --instance pr2392
python scripts/create_timing.py --instance rnd10000 --variant relaxed --reps 3
python scripts/ab_time.py base b32 --variants atomic relaxed spm
python scripts/ab_time.py base b32 --variants atomic relaxed spm
