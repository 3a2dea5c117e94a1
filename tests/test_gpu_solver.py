"""GPU solver surface: SPEC run() budget forms, RunReport fields, the C++
acs-bench CLI, island import/exchange (NCCL with one rank), the synthetic
10k-city instance, and the one-call C-ABI."""
import csv
import ctypes as C
import io
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from helpers import assert_permutations, to_acs

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_run_budget_forms(acs, gpu):
    I = O.load("d198")
    inst = to_acs(acs, I)
    inst.optimum = 15780
    r = acs.run(inst, acs.AcsParams(variant="atomic", iterations=7, seed=2))
    assert r.iterations == 7 and r.solutions == 7 * 198 and len(r.trace) == 7
    assert r.best_length == r.trace[-1] and (np.diff(r.trace) <= 0).all()
    assert r.error_pct == pytest.approx(100 * (r.best_length - 15780) / 15780)
    assert sorted(r.best_tour.tolist()) == list(range(198))
    r = acs.run(inst, acs.AcsParams(variant="relaxed", budget=198 * 5, seed=2))
    assert r.iterations == 5
    with pytest.raises(ValueError):
        acs.run(inst, acs.AcsParams(budget=199))
    r = acs.run(inst, acs.AcsParams(variant="spm", time_limit_s=0.3, seed=1))
    assert r.iterations >= 8 and r.hit_ratio() > 0.5
    # one timestamp per iteration, increasing, ending near the limit (coarse check, D14)
    assert len(r.trace_ms) == len(r.trace) == r.iterations
    assert (np.diff(r.trace_ms) > 0).all() and 250 < r.trace_ms[-1] < 1500


def test_cli_solve_csv(acs, gpu, tmp_path):
    subprocess.run(["make", "-s", "tools"], cwd=REPO, check=True)
    cat = tmp_path / "optima.txt"
    cat.write_text("d198 15780\n")
    out = subprocess.run([os.path.join(REPO, "build", "acs-bench"), "solve", "--instance",
                          os.path.join(REPO, "data", "tsplib", "d198.tsp.gz"), "--variant", "spm",
                          "--iterations", "20", "--reps", "2", "--seed", "3", "--optima", str(cat)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.DictReader(io.StringIO(out)))
    assert len(rows) == 2
    assert rows[0]["instance"] == "d198" and rows[0]["variant"] == "spm" and rows[0]["iters"] == "20"
    assert float(rows[0]["err_pct"]) >= 0 and 0 < float(rows[0]["hit_ratio"]) <= 1
    assert [r["seed"] for r in rows] == ["3", "4"]


def test_set_best_adopts_only_strictly_better(acs, gpu):
    I = O.load("pr2392")
    inst = to_acs(acs, I)
    with acs.Colony(inst, acs.AcsParams(variant="relaxed", seed=1, m=64)) as col:
        col.iterate(1)
        _, own = col.best()
        ident = np.arange(2392, dtype=np.uint32)  # file order is optimal: 378032
        col.set_best(ident, 378032)
        order, ln = col.best()
        assert ln == 378032 and (order == ident).all()
        col.set_best(np.roll(ident, 5)[::-1].copy(), 378032)  # tie: not adopted
        assert (col.best()[0] == ident).all()
        st = col.iterate(2)
        assert st["global_best_len"].tolist() == [378032, 378032]
        with pytest.raises(acs.AcsError):
            col.set_best(np.zeros(2392, np.uint32), 1)


def test_island_exchange_single_rank(acs, gpu):
    I = O.load("d198")
    inst = to_acs(acs, I)
    try:
        uid = acs.Colony.nccl_unique_id()
    except acs.AcsError as e:
        pytest.skip(f"NCCL not loadable here: {e}")
    with acs.Colony(inst, acs.AcsParams(variant="atomic", seed=3)) as col:
        col.island_init(uid, 1, 0)
        col.iterate(3)
        _, own = col.best()
        assert col.island_exchange() == own
        assert col.best()[1] == own


def test_rnd10k_tours_valid(acs, orc, gpu):
    I = O.rnd_instance()
    inst = to_acs(acs, I)
    for variant in ("atomic", "spm"):
        with acs.Colony(inst, acs.AcsParams(variant=variant, m=256, seed=1)) as col:
            st = col.iterate(2)
            routes, lens = col.routes()
        assert_permutations(routes, I.n)
        assert int(lens[7]) == orc.tour_length(I, routes[7])
        assert st["global_best_len"][-1] <= st["global_best_len"][0]


def test_one_call_run_matches_colony(acs, gpu):
    from paper_1605_02669_b200 import _native as N
    I = O.load("lin318")
    inst = to_acs(acs, I)
    p = acs.AcsParams(variant="seq", m=16, seed=4)
    order = np.empty(I.n, np.uint32)
    trace = np.empty(5, np.int64)
    ln = C.c_int64()
    d, cp = inst.desc(), p.to_c(I.n)
    N.check(N.lib().acs_gpu_run(C.byref(d), C.byref(cp), 5, 0, order.ctypes.data_as(C.c_void_p), C.byref(ln),
                                trace.ctypes.data_as(C.c_void_p)), "run")
    with acs.Colony(inst, p) as col:
        st = col.iterate(5)
        o2, l2 = col.best()
    assert trace.tolist() == st["global_best_len"].tolist() and ln.value == l2 and (order == o2).all()
