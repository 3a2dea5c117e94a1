"""Bit-exact parity at the BASELINE.json headline configurations.

The deterministic GPU variants against the CPU oracle (SPEC SYNC semantics,
SPEC.md:300-311) at full colony size on the instances BASELINE.json quotes:

  config 4  pr2392, m = n = 2392          deferred (xoshiro and Philox) == oracle SYNC
            nrw1379, m = n = 1379         deferred == oracle SYNC
  config 2  rat783, m = n = 783           spm-sync == oracle SYNC x SELECTIVE
            pcb442/rat783, m = n          deferred == oracle SYNC (both RNGs)
  config 5  rnd10k (no eta^beta table: on-the-fly eta, compacted full scan)
            seq, deferred and spm-seq, m = 64, 1 iteration

Each comparison covers the per-iteration L_gb trace, iteration-best length and
ant, every route and length of the last iteration, the whole pheromone matrix
(or every selective record) as bit patterns, and the step counters
(greedy / roulette / fallback / local updates, and hits / misses).
"""
import numpy as np
import pytest

import oracle as O
from helpers import to_acs
from test_gpu_parity import check_exact, pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rng", ["xoshiro", "philox"])
def test_pr2392_full_colony_deferred(acs, orc, gpu, rng):
    """BASELINE config 4: m = n = 2392 ants in lockstep, 2 iterations."""
    I = O.load("pr2392")
    r = pair(acs, orc, I, "sync", O.DENSE, m=2392, iters=2, seed=11, rng=rng)
    check_exact(*r, O.DENSE)
    cnt = r[4]
    assert cnt["local_updates"] == 2 * 2392 * 2392  # k = 1: n updates per tour
    assert cnt["fallback_steps"] > 0 and cnt["fallback_full"] > 0  # the cooperative full scan ran


def test_nrw1379_full_colony_deferred(acs, orc, gpu):
    I = O.load("nrw1379")
    r = pair(acs, orc, I, "sync", O.DENSE, m=1379, iters=2, seed=5)
    check_exact(*r, O.DENSE)


@pytest.mark.parametrize("name", ["pcb442", "rat783"])
@pytest.mark.parametrize("rng", ["xoshiro", "philox"])
def test_config2_full_colony_deferred(acs, orc, gpu, name, rng):
    I = O.load(name)
    r = pair(acs, orc, I, "sync", O.DENSE, m=I.n, iters=3, seed=23, rng=rng)
    check_exact(*r, O.DENSE)


def test_rat783_full_colony_spm_sync(acs, orc, gpu):
    """BASELINE config 2, selective memory: m = n = 783, record operations of
    every step applied in (record, ant, u/v) order."""
    I = O.load("rat783")
    r = pair(acs, orc, I, "sync", O.SELECTIVE, m=783, iters=2, seed=3)
    check_exact(*r, O.SELECTIVE)


@pytest.mark.parametrize("mode,memory", [("seq", O.DENSE), ("sync", O.DENSE), ("seq", O.SELECTIVE)])
def test_rnd10k_bit_exact(acs, orc, gpu, mode, memory):
    """BASELINE config 5 instance: n = 10000 > 4096, so no eta^beta table:
    eta^beta is computed from the coordinates, and the full-scan fallback is
    the compacted scan over unvisited nodes only."""
    I = O.rnd_instance(10000)
    r = pair(acs, orc, I, mode, memory, m=64, iters=1, seed=8)
    check_exact(*r, memory)
    # fallbacks past the ext rows: settled by the grid rings (or the compacted full scan)
    assert r[4]["fallback_grid"] + r[4]["fallback_full"] > 0


@pytest.mark.parametrize("variant", ["seq", "deferred"])
def test_rnd10k_grid_ring_fallback_equals_full_scan(acs, orc, gpu, monkeypatch, variant):
    """n > 4096: a fallback the ext rows cannot settle walks rings of grid
    cells before giving up to the full scan.  The grid walk must give the
    full scan's answer: the same tours and pheromone with and without it
    (ACS_NO_GRID), and the oracle's."""
    I = O.rnd_instance(10000)
    out = {}
    for grid in (True, False):
        if grid:
            monkeypatch.delenv("ACS_NO_GRID", raising=False)
        else:
            monkeypatch.setenv("ACS_NO_GRID", "1")
        p = acs.AcsParams(variant=variant, m=16, seed=4, q0=0.6)
        with acs.Colony(to_acs(acs, I), p) as col:
            st = col.iterate(1)
            routes, _ = col.routes()
            tau = col.pheromone()
            out[grid] = (st["global_best_len"].tolist(), routes, tau, col.counters())
    g, f = out[True], out[False]
    assert g[0] == f[0] and (g[1] == f[1]).all()
    assert np.array_equal(g[2].view(np.uint64), f[2].view(np.uint64))
    assert g[3]["fallback_grid"] > 0 and f[3]["fallback_grid"] == 0
    assert g[3]["fallback_full"] < f[3]["fallback_full"]
    o = orc.run(I, m=16, iterations=1, seed=4, mode=O.SYNC if variant == "deferred" else O.SEQ, q0=0.6,
                want_routes=True)
    assert (g[1] == o["routes"]).all()
