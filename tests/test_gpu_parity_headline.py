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
    assert r[4]["fallback_full"] > 0  # the compacted full scan was exercised
