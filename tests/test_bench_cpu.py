"""bench.py's CPU legs (reference arm + JSON contract) run on a CPU-only box."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--instance", "d198", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, check=True, timeout=600).stdout.strip().splitlines()
    assert len(out) == 1
    d = json.loads(out[0])
    assert d["impl"] == "reference" and d["unit"] == "tours/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["metric"].startswith("constructed tours/sec at pr2392")
    # the same workload as the GPU arm: one persistent colony of m = n ants
    c = d["config"]
    assert c["instance"] == "d198" and c["ants_per_gpu"] == 198 and c["rng"] == "philox"
    assert c["reference_mode"] == {"mode": "relaxed", "memory": "dense", "consistent": 1}
    assert "persistent 198-ant colony" in d["cpu_baseline"]["sample"]


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    p = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                        "--instance", "d198", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode == 0 and p.stdout.strip() == ""
