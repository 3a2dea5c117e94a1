"""bench.py contract on the GPU: one short run must print ONE JSON line with
every key the driver and the judge read (value, e2e, roofline incl. the L2 and
issue sub-objects, clocks, gpu_launches, cpu_baseline)."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_json_line(gpu):
    out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-variants"],
                         cwd=REPO, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    # the construction working set is L2-resident: the L2 is the bound
    assert r["bound"] == "l2" and 0 < r["frac"] < 1 and r["peak"] > 0
    assert 0 < r["hbm"]["frac"] < 1
    assert r["algorithmic_bytes_per_launch"] == r["bytes_per_tour"] * 2392 + r["fallback_bytes_per_launch"]
    assert "issue" in r and 0 < r["issue"]["frac"] < 1
    lat = r["latency"]  # hardware floor from acs_gpu_l2_latency, measured in the run
    assert 0 < lat["l2_load_ns"] < lat["floor_ns_per_step"] < lat["achieved_ns_per_step"]
    assert 0 < lat["frac"] < 1
    assert d["config"]["workload"].startswith("pr2392")
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_same_config(gpu):
    """--impl reference runs the GPU arm's workload: the same config dict."""
    ours = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-variants",
                           "--no-e2e", "--no-cpu-baseline"], cwd=REPO, capture_output=True, text=True, timeout=600)
    ref = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                         cwd=REPO, capture_output=True, text=True, timeout=600)
    assert ours.returncode == 0 and ref.returncode == 0, (ours.stderr[-2000:], ref.stderr[-2000:])
    a = json.loads([x for x in ours.stdout.splitlines() if x.startswith("{")][0])
    b = json.loads([x for x in ref.stdout.splitlines() if x.startswith("{")][0])
    cb = dict(b["config"])
    cb.pop("reference_mode")
    assert a["config"] == cb
    assert a["metric"] == b["metric"] and a["unit"] == b["unit"]
