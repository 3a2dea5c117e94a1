"""bench-cli over the drop-in C++ API: solve / sweep / compare.
CPU: usage errors exit 2 before any device work.  GPU: row cardinality, CSV
columns, JSON round trip with parameter provenance, SEQ determinism
(acceptance 10), baseline rows unmarked, compare's paired report."""
import csv
import io
import json
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "build", "acs-bench")
D198 = os.path.join(REPO, "data", "tsplib", "d198.tsp.gz")
A280 = os.path.join(REPO, "data", "tsplib", "a280.tsp.gz")
OPTIMA = os.path.join(REPO, "data", "tsplib", "optima.txt.gz")
SPEC_COLS = "instance,n,mode,memory,ants,period,slots,rep,seed,best_len,err_pct,iters,total_ms," \
            "construct_ms_per_iter,hit_ratio".split(",")


def cli(*args, check=True):
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", REPO, "tools"], check=True)
    r = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    if check and r.returncode != 0:
        raise AssertionError(f"exit {r.returncode}: {r.stderr}")
    return r


@pytest.mark.parametrize("args", [[], ["bogus"], ["solve"], ["solve", "--instance", D198, "--mode", "nope"],
                                  ["solve", "--instance", D198, "--frobnicate", "1"],
                                  ["sweep", "--instance", D198],
                                  ["compare", "--instance", D198, "--a", "k=1", "--b", "k=4", "--reps", "3"]])
def test_usage_errors_exit_2(args):
    assert cli(*args, check=False).returncode == 2


def test_unreadable_instance_exits_1():
    assert cli("solve", "--instance", "/nonexistent.tsp", check=False).returncode == 1


@pytest.mark.gpu
def test_solve_csv_and_json_roundtrip(gpu):
    r = cli("solve", "--instance", D198, "--optima", OPTIMA, "--mode", "seq", "--ants", "20", "--iterations", "5",
            "--seed", "3", "--reps", "2")
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert len(rows) == 2 and all(c in rows[0] for c in SPEC_COLS)
    assert rows[0]["n"] == "198" and rows[1]["seed"] == "4" and float(rows[0]["err_pct"]) > 0
    j1 = cli("solve", "--instance", D198, "--optima", OPTIMA, "--mode", "seq", "--ants", "20", "--iterations", "5",
             "--seed", "3", "--format", "json").stdout
    j2 = cli("solve", "--instance", D198, "--optima", OPTIMA, "--mode", "seq", "--ants", "20", "--iterations", "5",
             "--seed", "3", "--format", "json").stdout
    d = json.loads(j1)
    # acceptance 10 (determinism): identical reports apart from wall-clock fields
    strip = lambda x: {k: v for k, v in x.items() if not k.endswith("_ms") and k not in ("trace_ms", "tours_per_s",
                                                                                         "construct_ms_per_iter")}
    assert strip(d) == strip(json.loads(j2))
    assert d["best_len"] == int(rows[0]["best_len"]) and len(d["best_tour"]) == 198
    assert sorted(d["best_tour"]) == list(range(198)) and d["params"]["seed"] == 3
    assert json.loads(json.dumps(d)) == d


@pytest.mark.gpu
def test_sweep_rows_and_marks(gpu, tmp_path):
    out = str(tmp_path / "sw")
    r = cli("sweep", "--instance", D198, "--optima", OPTIMA, "--mode", "relaxed", "--ants", "64",
            "--iterations", "10", "--reps", "3", "--sweep", "k=1,2,4", "--out", out)
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert len(rows) == 9  # 3 points x 3 reps
    assert {x["period"] for x in rows} == {"1", "2", "4"}
    assert all(x["mark"] == "" for x in rows if x["point"] == "k=1")  # baseline carries no mark
    js = json.load(open(out + ".json"))
    assert [p["point"] for p in js] == ["k=1", "k=2", "k=4"] and js[0]["p_vs_baseline"] is None
    assert all(0 < p["p_vs_baseline"] <= 1 for p in js[1:])
    assert open(out + ".csv").read() == r.stdout


@pytest.mark.gpu
def test_compare_paired_report(gpu):
    r = cli("compare", "--instance", A280, "--optima", OPTIMA, "--ants", "64", "--update-period", "4",
            "--time-limit-ms", "150", "--reps", "3", "--a", "memory=dense,consistent=0",
            "--b", "memory=selective")
    d = json.loads(r.stdout)
    assert d["A"]["runs"] == d["B"]["runs"] == 3 and 0 < d["p_value"] <= 1
    assert d["winner"] in ("A", "B", "none") and d["A"]["mean_iters"] > 0
    # without an optimum the errors are raw lengths
    r = cli("compare", "--instance", D198, "--ants", "8", "--mode", "seq", "--time-limit-ms", "30", "--reps", "3",
            "--a", "k=1", "--b", "k=1")
    d = json.loads(r.stdout)
    assert d["errors_are"].startswith("raw")
