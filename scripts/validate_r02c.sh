set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lean or single_ant or concurrent or fold" 2>&1 | tail -2
python scripts/ab_time.py base idx32 route1 both --variants atomic relaxed
python scripts/ab_time.py base idx32 route1 both --variants atomic relaxed
LEGS="nrw1379:spm:8:100" bash scripts/quality_r02.sh
