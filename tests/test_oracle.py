"""Pin the CPU oracle before trusting it (CPU only):
  * against SURVEY Appendix A golden hashes derived from the reference code,
  * against the reference's own code compiled from /root/reference (oracle/_ref)
    on every shipped instance and on random/tie-heavy inputs,
  * against the SPEC per-op known-answer examples (SPEC.md op examples,
    acceptance criteria 1-3, 10)."""
import ctypes as C
from collections import OrderedDict

import numpy as np
import pytest

import oracle as O
from helpers import GOLDEN, RND10K_CAND_FNV, RND10K_NN, TSPLIB, small_instance


@pytest.mark.parametrize("name", TSPLIB)
def test_oracle_golden_hashes(orc, name):
    I = O.load(name)
    dist_fnv, cand_fnv, nn, opt = GOLDEN[name]
    assert O.fnv1a64(orc.distance_table(I)) == dist_fnv
    assert O.fnv1a64(orc.candidates(I, 32)) == cand_fnv
    assert orc.nn_tour_length(I, 0) == nn
    assert O.optima()[name] == opt


def test_oracle_rnd10k_golden(orc):
    I = O.rnd_instance()
    assert (I.xs[0], I.ys[0]) == (120054.0, 324231.0)
    assert O.fnv1a64(orc.candidates(I, 32)) == RND10K_CAND_FNV


@pytest.mark.slow
def test_oracle_rnd10k_nn(orc):
    assert orc.nn_tour_length(O.rnd_instance(), 0) == RND10K_NN


def test_tour_length_kats(orc):
    assert orc.tour_length(O.load("pr2392"), np.arange(2392)) == 378032
    assert orc.tour_length(O.load("d198"), np.arange(198)) == 22498


@pytest.mark.parametrize("name", TSPLIB)
def test_oracle_vs_reference_code(orc, ref, name):
    I = O.load(name)
    ri, err = ref.parse(O.read_tsplib_text(name))
    assert err is None
    xs, ys = ri.coords()
    assert np.array_equal(xs, I.xs) and np.array_equal(ys, I.ys) and ri.type == I.type
    for cl in (1, 5, 32, 40):
        assert (orc.candidates(I, cl) == ri.candidates(cl)).all()
    for s in (0, I.n // 3, I.n - 1):
        assert orc.nn_tour_length(I, s) == ri.nn_tour_length(s)
    rng = np.random.default_rng(1)
    for _ in range(5):
        p = rng.permutation(I.n).astype(np.uint32)
        assert orc.tour_length(I, p) == ri.tour_length(p)


@pytest.mark.parametrize("typ", [O.EUC_2D, O.CEIL_2D, O.ATT])
@pytest.mark.parametrize("n", [3, 4, 10, 57])
def test_oracle_vs_reference_ties(orc, ref, typ, n):
    I = small_instance(n, seed=n + typ, scale=7, typ=typ)  # many duplicate points / ties
    ri = ref.make(I)
    assert (orc.distance_table(I) == ri.distance_table()).all()
    for cl in (1, 3, 32):
        assert (orc.candidates(I, cl) == ri.candidates(cl)).all()
    for s in range(min(n, 5)):
        assert orc.nn_tour_length(I, s) == ri.nn_tour_length(s)


def test_rng_survey_kats(orc):
    lib = orc.lib
    r = orc.rng_derive(42, 0, 0)
    assert f"{lib.orc_rng_next_u64(C.byref(r)):016x}" == "c986fd807e5b8ab5"
    assert f"{lib.orc_rng_next_u64(C.byref(r)):016x}" == "e071ea15f19664d1"
    assert lib.orc_rng_uniform01(C.byref(r)) == 0.44735932804098311
    r = orc.rng_derive(42, 1, 7)
    assert f"{lib.orc_rng_next_u64(C.byref(r)):016x}" == "1e41e6edf5d70818"
    assert lib.orc_rng_uniform_int(C.byref(r), 280) == 133
    r = orc.rng_seed(0)
    assert f"{lib.orc_rng_next_u64(C.byref(r)):016x}" == "99ec5f36cb75f2b4"
    assert lib.orc_rng_uniform01(C.byref(orc.rng_derive(1, 0, 0))) == 0.37699756613273605
    assert lib.orc_rng_uniform_int(C.byref(orc.rng_derive(1, 0, 0)), 198) == 74


@pytest.mark.parametrize("seed,it,ant,derive", [(0, 0, 0, 0), (42, 1, 7, 1), (2**64 - 1, 5, 2391, 1),
                                                 (123456789, 0, 0, 0)])
def test_rng_vs_reference_code(orc, ref, seed, it, ant, derive):
    rng = np.random.default_rng(seed % 1000)
    ops = rng.integers(0, 3, 2000).astype(np.int32)
    args = rng.integers(1, 1 << 62, 2000).astype(np.uint64)
    args[::5] = rng.integers(1, 9, len(args[::5]))
    want = ref.rng_script(seed, it, ant, derive, ops, args)
    r = orc.rng_derive(seed, it, ant) if derive else orc.rng_seed(seed)
    lib = orc.lib
    got = []
    for op, a in zip(ops, args):
        if op == 0:
            got.append(lib.orc_rng_next_u64(C.byref(r)))
        elif op == 1:
            got.append(int(np.float64(lib.orc_rng_uniform01(C.byref(r))).view(np.uint64)))
        else:
            got.append(lib.orc_rng_uniform_int(C.byref(r), int(a)))
    assert got == want.tolist()


# ---------------- SPEC op KATs (SPEC.md examples, acceptance 1) ----------------

def test_update_arithmetic_kats(orc):
    lib = orc.lib
    assert abs(lib.orc_local_update_value(0.5, 0.01, 0.1) - 0.496) <= 1e-12 * 0.496
    assert lib.orc_local_update_value(0.1, 0.01, 0.1) == pytest.approx(0.1, rel=1e-15)  # fixed point
    assert abs(lib.orc_global_update_value(0.5, 0.2, 100) - 0.402) <= 1e-12 * 0.402
    assert lib.orc_global_update_value(0.01, 0.2, 100) == pytest.approx(0.01, rel=1e-15)
    assert lib.orc_default_q0(1379) == pytest.approx(0.98550, abs=5e-6)
    assert lib.orc_default_q0(20) == 0.0 and lib.orc_default_q0(10) == 0.0
    assert lib.orc_score(0.1, 1.0, 3.0) == 0.1
    assert lib.orc_score(0.2, 0.5, 3.0) == 0.025
    assert lib.orc_score(0.7, 0.3, 0.0) == 0.7


def test_selection_kats(orc):
    lib = orc.lib
    f = lambda *w: np.asarray(w, np.float64)
    assert lib.orc_greedy_pick(f(0.025, 0.1), 2) == 1
    assert lib.orc_greedy_pick(f(0.3), 1) == 0
    assert lib.orc_greedy_pick(f(0.5, 0.5, 0.2), 3) == 0  # D7 tie -> earliest
    assert lib.orc_roulette_pick(f(1, 1, 2), 3, 0.6) == 2
    assert lib.orc_roulette_pick(f(0, 1, 2), 3, 0.0) == 1  # r=0 -> first positive weight
    assert lib.orc_roulette_pick(f(0, 0, 0), 3, 0.4) == 0  # all zero -> greedy tie rule
    assert lib.orc_select_best(np.asarray([10, 7, 9], np.int64), 3) == 1
    assert lib.orc_select_best(np.asarray([7, 7], np.int64), 2) == 0


def test_roulette_chi_square(orc):
    """acceptance 2: Eq.(2) probabilities by chi-square on 1e5 seeded draws."""
    from scipy.stats import chisquare
    lib = orc.lib
    r = orc.rng_seed(2016)
    for w in (np.asarray([1.0, 3.0]), np.random.default_rng(5).random(32)):
        counts = np.zeros(len(w))
        for _ in range(100000):
            counts[lib.orc_roulette_pick(w, len(w), lib.orc_rng_uniform01(C.byref(r)))] += 1
        assert chisquare(counts, w / w.sum() * counts.sum()).pvalue > 1e-3


class FifoMap:
    """SPEC derived oracle: map with per-key-set capacity s and FIFO eviction."""

    def __init__(self, s, tau_min):
        self.s, self.tau_min, self.rec = s, tau_min, {}

    def read(self, u, v):
        return self.rec.get(u, OrderedDict()).get(v, self.tau_min)

    def update(self, u, v, cm, ca):
        r = self.rec.setdefault(u, OrderedDict())
        if v in r:
            r[v] = cm * r[v] + ca
            return True
        if len(r) == self.s:
            r.popitem(last=False)
        r[v] = cm * self.tau_min + ca
        return False


@pytest.mark.parametrize("s", [1, 2, 4, 8])
def test_selective_store_vs_fifo_map(orc, s):
    """acceptance 3: 1e4 random single-threaded ops, 0 mismatches."""
    lib = orc.lib
    n, tau_min = 50, 0.1
    p = lib.orc_spm_new(n, s, tau_min)
    ref = FifoMap(s, tau_min)
    rng = np.random.default_rng(s)
    try:
        for _ in range(10000):
            u, v = rng.choice(n, 2, replace=False)
            if rng.random() < 0.4:
                assert lib.orc_spm_read(p, int(u), int(v)) == ref.read(int(u), int(v))
            else:
                cm, ca = (0.99, 0.001) if rng.random() < 0.8 else (0.8, 0.2 / rng.integers(50, 500))
                assert lib.orc_spm_update_record(p, int(u), int(v), cm, ca) == ref.update(int(u), int(v), cm, ca)
    finally:
        lib.orc_spm_free(p)


def test_selective_kats(orc):
    lib = orc.lib
    p = lib.orc_spm_new(5, 2, 0.1)
    for v in (1, 2, 3):  # s=2: inserts 1,2,3 -> {2,3}
        lib.orc_spm_update_record(p, 0, v, 0.99, 0.005)
    assert lib.orc_spm_read(p, 0, 1) == 0.1 and lib.orc_spm_read(p, 0, 2) != 0.1
    ids = np.zeros(10, np.uint32)
    tail = np.zeros(5, np.uint32)
    lib.orc_spm_dump(p, ids.ctypes.data_as(C.c_void_p), None, tail.ctypes.data_as(C.c_void_p))
    assert sorted(ids[:2].tolist()) == [2, 3] and tail[0] == 0
    lib.orc_spm_update_record(p, 0, 3, 0.99, 0.001)  # hit: tail untouched
    lib.orc_spm_dump(p, None, None, tail.ctypes.data_as(C.c_void_p))
    assert tail[0] == 0
    h, m = C.c_uint64(), C.c_uint64()
    lib.orc_spm_counts(p, C.byref(h), C.byref(m))
    assert (h.value, m.value) == (1, 3)
    lib.orc_spm_free(p)
    p = lib.orc_spm_new(3, 8, 0.1)  # D5: first insertion lands in slot 0
    lib.orc_spm_update_record(p, 1, 2, 0.99, 0.001)
    ids = np.zeros(24, np.uint32)
    lib.orc_spm_dump(p, ids.ctypes.data_as(C.c_void_p), None, None)
    assert ids[8] == 2
    lib.orc_spm_free(p)


# ---------------- engine properties (acceptance 10) ----------------

def test_engine_determinism_and_counts(orc):
    I = O.load("d198")
    a = orc.run(I, m=20, iterations=5, seed=3, mode=O.SEQ, want_tau=True)
    b = orc.run(I, m=20, iterations=5, seed=3, mode=O.SEQ, want_tau=True)
    assert (a["routes"] == b["routes"]).all() and np.array_equal(a["tau"], b["tau"])
    assert (np.diff(a["trace"]) <= 0).all()
    for mode in (O.SEQ, O.SYNC, O.RELAXED):
        r = orc.run(I, m=20, iterations=3, seed=1, mode=mode, threads=4)
        assert r["local_updates"] == 3 * 20 * 198  # k=1: n updates per tour
        assert (np.sort(r["routes"], axis=1) == np.arange(198)).all()
    r = orc.run(O.load("d198"), m=10, iterations=2, seed=1, mode=O.SEQ, k=4)
    assert r["local_updates"] == 2 * 10 * (198 // 4)


def test_relaxed_stress_validity(orc):
    """acceptance 4 (reduced): concurrent RELAXED tours are all permutations."""
    I = O.load("lin318")
    for memory in (O.DENSE, O.SELECTIVE):
        r = orc.run(I, m=318, iterations=3, seed=2, mode=O.RELAXED, memory=memory, threads=8,
                    want_spm=True)
        assert (np.sort(r["routes"], axis=1) == np.arange(318)).all()
        if memory == O.SELECTIVE:
            assert (r["spm_tail"] < 8).all()
            occ = r["spm_ids"] != 0xFFFFFFFF
            assert (r["spm_ids"][occ] < 318).all() and (r["spm_vals"] > 0).all()
