"""Tour-level parity of the sm_100a construction kernels against the CPU
oracle (SPEC restatement).  Deterministic variants must be BIT-EXACT:

  GPU ACS_VARIANT_SEQ      (k_construct_dense, one warp)  == oracle SEQ   / DENSE
  GPU ACS_VARIANT_DEFERRED (k_def_select/apply, all ants) == oracle SYNC  / DENSE
  GPU ACS_VARIANT_SPM_SEQ  (k_construct_spm, one warp)    == oracle SEQ   / SELECTIVE
  GPU ACS_VARIANT_SPM_SYNC (k_ssync_*, all ants, sorted ordered apply) == oracle SYNC / SELECTIVE

compared on: per-iteration L_gb trace, iteration-best length and ant, every
route and length of the last iteration, the final pheromone state (dense
matrix or selective records) and the step counters.
"""
import numpy as np
import pytest

import oracle as O
from helpers import assert_permutations, small_instance, to_acs

pytestmark = pytest.mark.gpu

GPU_OF = {("seq", O.DENSE): (O.SEQ, "seq"), ("sync", O.DENSE): (O.SYNC, "deferred"),
          ("seq", O.SELECTIVE): (O.SEQ, "spm-seq"), ("sync", O.SELECTIVE): (O.SYNC, "spm-sync")}
MODES = [("seq", O.DENSE), ("sync", O.DENSE), ("seq", O.SELECTIVE), ("sync", O.SELECTIVE)]


def pair(acs, orc, I, mode, memory, *, m, iters, seed=1, k=1, beta=3.0, q0=-1.0, cl=32, s=8,
         rng="xoshiro", alpha=0.2, rho=0.01):
    omode, variant = GPU_OF[(mode, memory)]
    p = acs.AcsParams(variant=variant, m=m, seed=seed, k=k, beta=beta, q0=q0, cl=cl, s=s, rng=rng,
                      alpha=alpha, rho=rho)
    with acs.Colony(to_acs(acs, I), p) as col:
        st = col.iterate(iters)
        routes, lens = col.routes()
        state = col.pheromone() if memory == O.DENSE else col.selective()
        cnt = col.counters()
        best = col.best()
    o = orc.run(I, m=m, iterations=iters, seed=seed, mode=omode, memory=memory, k=k, beta=beta,
                q0=q0, cl=cl, s=s, rng=O.PHILOX if rng == "philox" else O.XOSHIRO, alpha=alpha,
                rho=rho, want_tau=True, want_spm=True)
    return st, routes, lens, state, cnt, best, o


def check_exact(st, routes, lens, state, cnt, best, o, memory):
    assert st["global_best_len"].tolist() == o["trace"].tolist()
    assert st["iter_best_len"].tolist() == o["iter_best_len"].tolist()
    assert st["iter_best_ant"].tolist() == o["iter_best_ant"].tolist()
    assert (routes == o["routes"]).all()
    assert lens.tolist() == o["lengths"].tolist()
    assert best[1] == o["best_len"] and (best[0] == o["best_tour"]).all()
    if memory == O.DENSE:
        assert np.array_equal(state.view(np.uint64), o["tau"].view(np.uint64)), "pheromone bits differ"
    else:
        ids, vals, tail = state
        assert (ids == o["spm_ids"]).all() and (tail == o["spm_tail"]).all()
        assert np.array_equal(vals.view(np.uint64), o["spm_vals"].view(np.uint64))
        assert cnt["hits"] == o["hits"] and cnt["misses"] == o["misses"]
    assert cnt["fallback_steps"] == o["fallback_steps"]
    assert cnt["greedy_steps"] == o["greedy_steps"]
    assert cnt["roulette_steps"] == o["roulette_steps"]
    assert cnt["local_updates"] == o["local_updates"]


@pytest.mark.parametrize("mode,memory", MODES)
def test_d198_bit_exact(acs, orc, gpu, mode, memory):
    I = O.load("d198")
    r = pair(acs, orc, I, mode, memory, m=40, iters=6)
    check_exact(*r, memory)


@pytest.mark.parametrize("mode,memory", MODES)
@pytest.mark.parametrize("k", [2, 4])
def test_update_period_bit_exact(acs, orc, gpu, mode, memory, k):
    I = O.load("a280")
    r = pair(acs, orc, I, mode, memory, m=24, iters=4, k=k, seed=5)
    check_exact(*r, memory)


@pytest.mark.parametrize("mode,memory", MODES)
def test_philox_bit_exact(acs, orc, gpu, mode, memory):
    I = O.load("lin318")
    r = pair(acs, orc, I, mode, memory, m=16, iters=4, rng="philox", seed=9)
    check_exact(*r, memory)


@pytest.mark.parametrize("q0", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("mode,memory", [("seq", O.DENSE), ("sync", O.DENSE), ("sync", O.SELECTIVE)])
def test_q0_extremes_bit_exact(acs, orc, gpu, mode, memory, q0):
    # q0 = 0 -> every candidate step is a roulette draw (exercises the
    # sequential-prefix warp roulette), q0 = 1 -> always greedy
    I = small_instance(150, seed=4)
    r = pair(acs, orc, I, mode, memory, m=30, iters=3, q0=q0, seed=2)
    check_exact(*r, memory)


@pytest.mark.parametrize("beta,cl", [(0.0, 32), (1.0, 8), (2.0, 3), (5.0, 16)])
def test_beta_and_cl_bit_exact(acs, orc, gpu, beta, cl):
    I = small_instance(120, seed=8)
    for mode, memory in MODES:
        r = pair(acs, orc, I, mode, memory, m=20, iters=3, beta=beta, cl=cl, seed=3)
        check_exact(*r, memory)


@pytest.mark.parametrize("s", [1, 2, 4, 16])
def test_spm_slots_bit_exact(acs, orc, gpu, s):
    I = O.load("d198")
    r = pair(acs, orc, I, "seq", O.SELECTIVE, m=20, iters=4, s=s, seed=4)
    check_exact(*r, O.SELECTIVE)


@pytest.mark.parametrize("n", [3, 4, 5, 31, 33])
def test_tiny_and_ragged_instances(acs, orc, gpu, n):
    I = small_instance(n, seed=n, scale=20)
    for mode, memory in [("seq", O.DENSE), ("sync", O.DENSE), ("seq", O.SELECTIVE)]:
        r = pair(acs, orc, I, mode, memory, m=7, iters=3, seed=n)
        check_exact(*r, memory)


def test_att_and_duplicates(acs, orc, gpu):
    I = O.load("att532")
    r = pair(acs, orc, I, "sync", O.DENSE, m=12, iters=2)
    check_exact(*r, O.DENSE)
    xs = np.array([0, 0, 3, 3, 7, 7, 7, 2, 9, 1], np.float64)  # duplicate points: d = 0 -> eps = 1 (D1)
    ys = np.array([0, 0, 4, 4, 1, 1, 1, 8, 9, 5], np.float64)
    I = O.Coords("dups", O.EUC_2D, xs, ys)
    for mode, memory in [("seq", O.DENSE), ("sync", O.DENSE), ("seq", O.SELECTIVE)]:
        check_exact(*pair(acs, orc, I, mode, memory, m=10, iters=5), memory)


def test_sync_full_colony_pcb442(acs, orc, gpu):
    """m = n ants in lockstep: many ants update the same edges in one step."""
    I = O.load("pcb442")
    r = pair(acs, orc, I, "sync", O.DENSE, m=442, iters=2, seed=17)
    check_exact(*r, O.DENSE)
    cnt = r[4]
    # most fallback steps are settled by the pruned pass (hot list + next-nearest)
    assert 0 < cnt["fallback_full"] < cnt["fallback_steps"] // 2


@pytest.mark.parametrize("variant", ["atomic", "relaxed", "spm"])
@pytest.mark.parametrize("name", ["pcb442", "rat783"])
def test_concurrent_variants_valid(acs, orc, gpu, variant, name):
    """Non-deterministic variants: every tour a permutation, lengths equal the
    oracle's tour_length, L_gb monotone, update counts exact."""
    I = O.load(name)
    p = acs.AcsParams(variant=variant, seed=3)
    iters = 5
    with acs.Colony(to_acs(acs, I), p) as col:
        st = col.iterate(iters)
        routes, lens = col.routes()
        cnt = col.counters()
        best, blen = col.best()
        if variant == "spm":
            ids, vals, tail = col.selective()
    assert_permutations(routes, I.n)
    sample = range(0, I.n, 37)
    assert [int(lens[a]) for a in sample] == [orc.tour_length(I, routes[a]) for a in sample]
    g = st["global_best_len"]
    assert (np.diff(g) <= 0).all() and g[-1] == blen == orc.tour_length(I, best)
    assert st["iter_best_len"].tolist()[-1] == lens.min()
    assert cnt["local_updates"] == iters * I.n * I.n  # k=1: n updates per tour
    assert cnt["greedy_steps"] + cnt["roulette_steps"] + cnt["fallback_steps"] == iters * I.n * (I.n - 1)
    if variant == "spm":  # structural invariants of the records under races
        assert (tail < 8).all()
        occupied = ids != 0xFFFFFFFF
        assert (ids[occupied] < I.n).all()
        assert np.isfinite(vals).all() and (vals > 0).all()
        assert cnt["hits"] + cnt["misses"] == 2 * cnt["local_updates"] + 2 * I.n * iters


def test_atomic_single_ant_equals_seq(acs, orc, gpu):
    """With one ant there is no concurrency: the CAS variant must reproduce SEQ."""
    I = O.load("d198")
    p = acs.AcsParams(variant="atomic", m=1, seed=12)
    with acs.Colony(to_acs(acs, I), p) as col:
        st = col.iterate(8)
        tau = col.pheromone()
    o = orc.run(I, m=1, iterations=8, seed=12, mode=O.SEQ, want_tau=True)
    assert st["global_best_len"].tolist() == o["trace"].tolist()
    assert np.array_equal(tau.view(np.uint64), o["tau"].view(np.uint64))


@pytest.mark.parametrize("variant", ["atomic", "relaxed"])
@pytest.mark.parametrize("rng", ["xoshiro", "philox"])
@pytest.mark.parametrize("q0", [-1.0, 0.0, 0.7])
def test_lean_kernel_single_ant_equals_seq(acs, orc, gpu, variant, rng, q0):
    """k = 1 with 32-slot lists runs the lean tour kernel (k_tour_lean): with
    one ant it must reproduce SEQ bit for bit -- routes, trace, pheromone,
    step counters -- for both RNG engines, greedy, roulette and mixed steps."""
    I = O.load("d198")
    p = acs.AcsParams(variant=variant, m=1, seed=12, rng=rng, q0=q0)
    with acs.Colony(to_acs(acs, I), p) as col:
        st = col.iterate(6)
        tau = col.pheromone()
        routes, lens = col.routes()
        cnt = col.counters()
    o = orc.run(I, m=1, iterations=6, seed=12, mode=O.SEQ, want_tau=True, q0=q0,
                rng=O.PHILOX if rng == "philox" else O.XOSHIRO)
    assert st["global_best_len"].tolist() == o["trace"].tolist()
    assert (routes == o["routes"]).all() and lens.tolist() == o["lengths"].tolist()
    assert np.array_equal(tau.view(np.uint64), o["tau"].view(np.uint64))
    for k in ("fallback_steps", "greedy_steps", "roulette_steps", "local_updates"):
        assert cnt[k] == o[k], k


@pytest.mark.parametrize("rng", ["xoshiro", "philox"])
@pytest.mark.parametrize("q0", [-1.0, 0.0, 0.7])
@pytest.mark.parametrize("name", ["d198", "pcb442"])
def test_spm_lean_single_ant_equals_seq(acs, orc, gpu, rng, q0, name):
    """k = 1, 32-slot lists, s = 8 runs the lean SPM kernel (k_spm_lean): with
    one ant it must reproduce SEQ x SELECTIVE bit for bit -- the records
    (ids, values, tails), routes, trace and the hit / miss counts."""
    I = O.load(name)
    p = acs.AcsParams(variant="spm", m=1, seed=5, rng=rng, q0=q0)
    with acs.Colony(to_acs(acs, I), p) as col:
        st = col.iterate(5)
        ids, vals, tail = col.selective()
        routes, lens = col.routes()
        cnt = col.counters()
    o = orc.run(I, m=1, iterations=5, seed=5, mode=O.SEQ, memory=O.SELECTIVE, want_spm=True, q0=q0,
                rng=O.PHILOX if rng == "philox" else O.XOSHIRO)
    assert st["global_best_len"].tolist() == o["trace"].tolist()
    assert (routes == o["routes"]).all() and lens.tolist() == o["lengths"].tolist()
    assert (ids == o["spm_ids"]).all() and (tail == o["spm_tail"]).all()
    assert np.array_equal(vals.view(np.uint64), o["spm_vals"].view(np.uint64))
    for k in ("hits", "misses", "fallback_steps", "greedy_steps", "roulette_steps", "local_updates"):
        assert cnt[k] == o[k], k


@pytest.mark.parametrize("variant", ["atomic", "relaxed", "spm"])
@pytest.mark.parametrize("m", [2, 3, 7, 64])
def test_lean_kernel_small_colonies(acs, orc, gpu, variant, m):
    """Lean kernel with small even and odd colonies: valid tours, exact
    lengths (the per-lane length shares reduced at the tour end), exact
    update and step counts."""
    I = O.load("lin318")
    with acs.Colony(to_acs(acs, I), acs.AcsParams(variant=variant, m=m, seed=m, rng="philox")) as col:
        st = col.iterate(3)
        routes, lens = col.routes()
        cnt = col.counters()
    assert_permutations(routes, I.n)
    assert [int(x) for x in lens] == [orc.tour_length(I, r) for r in routes]
    assert cnt["local_updates"] == 3 * m * I.n
    assert cnt["greedy_steps"] + cnt["roulette_steps"] + cnt["fallback_steps"] == 3 * m * (I.n - 1)
    assert st["iter_best_len"].tolist()[-1] == lens.min()


@pytest.mark.parametrize("variant", ["relaxed", "atomic", "spm"])
def test_lean_kernel_single_ant_pr2392(acs, orc, gpu, variant):
    """The headline instance through the lean kernels (k_tour_lean for
    relaxed / atomic, k_spm_lean for spm), one ant: bit-exact SEQ (SEQ x
    SELECTIVE for spm) -- trace, routes, and the whole pheromone matrix or the
    selective records as bit patterns."""
    I = O.load("pr2392")
    p = acs.AcsParams(variant=variant, m=1, seed=3, rng="philox")
    spm = variant == "spm"
    with acs.Colony(to_acs(acs, I), p) as col:
        st = col.iterate(2)
        routes, lens = col.routes()
        if spm:
            ids, vals, tail = col.selective()
        else:
            tau = col.pheromone()
    o = orc.run(I, m=1, iterations=2, seed=3, mode=O.SEQ, rng=O.PHILOX,
                **({"memory": O.SELECTIVE, "want_spm": True} if spm else {"want_tau": True}))
    assert st["global_best_len"].tolist() == o["trace"].tolist()
    assert (routes == o["routes"]).all() and lens.tolist() == o["lengths"].tolist()
    if spm:
        assert (ids == o["spm_ids"]).all() and (tail == o["spm_tail"]).all()
        assert np.array_equal(vals.view(np.uint64), o["spm_vals"].view(np.uint64))
    else:
        assert np.array_equal(tau.view(np.uint64), o["tau"].view(np.uint64))


def test_sync_more_ants_than_resident_warps(acs, orc, gpu):
    """m > resident warps: the cooperative deferred kernel runs several ants
    per warp (state in shared memory) and must stay bit-exact."""
    I = O.load("d198")
    r = pair(acs, orc, I, "sync", O.DENSE, m=3500, iters=2, seed=21)
    check_exact(*r, O.DENSE)


@pytest.mark.parametrize("variant", ["atomic", "relaxed"])
def test_colony_larger_than_one_wave(acs, orc, gpu, variant):
    """m above the 96-register residency (20 ants per SM) launches the wide
    (72-register) build; tours stay valid and the update count exact."""
    I = O.load("d198")
    m = 3500
    with acs.Colony(to_acs(acs, I), acs.AcsParams(variant=variant, m=m, seed=8, rng="philox")) as col:
        st = col.iterate(2)
        routes, lens = col.routes()
        cnt = col.counters()
    assert_permutations(routes, I.n)
    assert [int(lens[a]) for a in range(0, m, 97)] == [orc.tour_length(I, routes[a]) for a in range(0, m, 97)]
    assert cnt["local_updates"] == 2 * m * I.n
    assert st["iter_best_len"].tolist()[-1] == lens.min()


@pytest.mark.parametrize("grid", [True, False])
@pytest.mark.parametrize("mode", ["sync", "seq"])
def test_no_eta_table_bit_exact(acs, orc, gpu, monkeypatch, mode, grid):
    """n > 4096: no eta^beta table.  A fallback the ext rows cannot settle
    walks rings of grid cells (grid) or runs the compacted scan over the
    unvisited nodes (ACS_NO_GRID; deferred: split over the warps of the CTA).
    q0 = 0.5 and few ants keep fallbacks frequent and late."""
    if grid:
        monkeypatch.delenv("ACS_NO_GRID", raising=False)
    else:
        monkeypatch.setenv("ACS_NO_GRID", "1")
    I = small_instance(4200, seed=3, scale=20000)
    r = pair(acs, orc, I, mode, O.DENSE, m=48 if mode == "sync" else 6, iters=2, seed=2, q0=0.5, k=2)
    check_exact(*r, O.DENSE)
    assert (r[4]["fallback_grid"] if grid else r[4]["fallback_full"]) > 0


def test_sync_cooperative_scan_bit_exact(acs, orc, gpu):
    """The deferred kernel's full scans split over many warps of a CTA (n = 1002:
    32 bitmask words, 8 slices) must equal the oracle's single scan."""
    I = O.load("pr1002")
    r = pair(acs, orc, I, "sync", O.DENSE, m=64, iters=2, seed=4, q0=0.3)
    check_exact(*r, O.DENSE)
    assert r[4]["fallback_full"] > 0


@pytest.mark.parametrize("slots", [1, 2, 16])
def test_spm_sync_slots_bit_exact(acs, orc, gpu, slots):
    """SYNC x SELECTIVE with other record sizes, m = n (every record sees
    convoys of inserts per step, applied in ant order)."""
    I = O.load("d198")
    r = pair(acs, orc, I, "sync", O.SELECTIVE, m=198, iters=3, seed=6, s=slots)
    check_exact(*r, O.SELECTIVE)


@pytest.mark.parametrize("name,m", [("d198", 198), ("pcb442", 442)])
def test_atomic_fold_matches_sequential_updates(acs, orc, gpu, name, m):
    """ATOMIC (CONSISTENT) after one iteration: every copy of edge {u, v} was
    bumped once per ant that traversed it, and the epilogue folds c pending
    updates into the base (k_fold_counts / trail_value): the affine rule
    itself for c <= 1, the closed form tau_min + c_l^c (b - tau_min) for
    c >= 2.  The folded matrix must equal f applied c times in sequence (c
    from the routes) within 1e-12 relative, and bit for bit where c <= 1.
    The global update then touches only the best tour's edges."""
    I = O.load(name)
    rho, alpha = 0.01, 0.2
    with acs.Colony(to_acs(acs, I), acs.AcsParams(variant="atomic", m=m, seed=4, rho=rho, alpha=alpha)) as col:
        col.iterate(1)
        tau = col.pheromone()
        routes, _ = col.routes()
        best, blen = col.best()
        tau0 = col.info.tau0
    n = I.n
    c = np.zeros((n, n), np.int64)
    for r in routes.astype(np.int64):
        u, v = r, np.roll(r, -1)
        np.add.at(c, (u, v), 1)
        np.add.at(c, (v, u), 1)
    c_orig = c.copy()
    # f^c(tau0), sequential, with the device's constants
    c_l, c_0 = 1.0 - rho, rho * tau0
    want = np.full((n, n), tau0)
    for _ in range(int(c.max())):
        step = c > 0
        want[step] = c_l * want[step] + c_0
        c[step] -= 1
    bu = best.astype(np.int64)
    gb = np.zeros((n, n), bool)
    gb[bu, np.roll(bu, -1)] = True
    gb[np.roll(bu, -1), bu] = True
    keep = ~gb
    rel = np.abs(tau[keep] - want[keep]) / want[keep]
    assert rel.max() < 1e-12, rel.max()
    low = keep & (c_orig <= 1)
    assert np.array_equal(tau[low].view(np.uint64), want[low].view(np.uint64))
    assert (c_orig[keep] >= 2).any()  # the closed form was exercised
    # the global update on the best tour's edges: tau' = (1 - alpha) tau_folded + alpha / L_gb
    c_d = alpha * (1.0 / blen)
    g = (1.0 - alpha) * want[gb] + c_d
    assert (np.abs(tau[gb] - g) / g).max() < 1e-12


@pytest.mark.parametrize("beta", [2.5, 0.7])
@pytest.mark.parametrize("mode,memory", MODES)
def test_non_integer_beta_bit_exact(acs, orc, gpu, beta, mode, memory):
    """a non-integral beta takes eta^beta from a table by integer
    distance built on the host with the C library's pow -- the oracle's own
    computation -- so the deterministic variants stay bit-exact."""
    I = O.load("d198")
    r = pair(acs, orc, I, mode, memory, m=24, iters=3, beta=beta, seed=6)
    check_exact(*r, memory)


def test_non_integer_beta_no_eta_table(acs, orc, gpu):
    """n > 4096 (no eta^beta matrix: the fallback computes distances on the fly)
    with a non-integral beta, through the distance table."""
    I = small_instance(4200, seed=5, scale=20000)
    r = pair(acs, orc, I, "seq", O.DENSE, m=3, iters=1, beta=1.5, seed=2, q0=0.5)
    check_exact(*r, O.DENSE)


def test_non_integer_beta_lean_kernel(acs, orc, gpu):
    """The lean kernel (k = 1, 32-slot lists) with beta = 2.5, one ant: SEQ."""
    I = O.load("pcb442")
    p = acs.AcsParams(variant="relaxed", m=1, seed=3, beta=2.5, rng="philox")
    with acs.Colony(to_acs(acs, I), p) as col:
        st = col.iterate(3)
        tau = col.pheromone()
    o = orc.run(I, m=1, iterations=3, seed=3, mode=O.SEQ, want_tau=True, beta=2.5, rng=O.PHILOX)
    assert st["global_best_len"].tolist() == o["trace"].tolist()
    assert np.array_equal(tau.view(np.uint64), o["tau"].view(np.uint64))


@pytest.mark.parametrize("m", [198, 9000])
def test_spm_sync_device_wide_sort(acs, orc, gpu, monkeypatch, m):
    """SYNC x SELECTIVE above one CTA's sort (m > 8192): the step's
    record operations are radix-sorted device-wide; forced for m = 198 too
    (ACS_SSYNC_WIDE).  Bit-exact with the oracle either way."""
    monkeypatch.setenv("ACS_SSYNC_WIDE", "1")
    I = O.load("d198")
    r = pair(acs, orc, I, "sync", O.SELECTIVE, m=m, iters=1 if m > 1000 else 3, seed=7)
    check_exact(*r, O.SELECTIVE)
