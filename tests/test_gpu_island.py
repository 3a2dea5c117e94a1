"""Island model on a real GPU with more than one colony.

The driver's box has one GPU, so a multi-GPU curve cannot be measured here.
What these tests pin instead:

* the device exchange kernels (k_island_pack / k_island_mask / k_adopt_best)
  with several ranks: acs_gpu_island_exchange_local runs them for colonies of
  one process on one GPU, with the two NCCL all-reduces restated as device
  reductions -- adoption, ties to the lowest rank, strictly-better adoption,
  and the no-tour-yet sentinel;
* the NCCL path itself with one rank, called before the first iteration;
* the host exchange (island.exchange_host) between two processes that each
  own a real Colony on cuda:0, over gloo: world_size 2 with real colonies.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from helpers import to_acs

pytestmark = pytest.mark.gpu

LLONG_MAX = (1 << 63) - 1


def test_local_exchange_before_first_iteration(acs, gpu):
    inst = to_acs(acs, O.load("d198"))
    cols = [acs.Colony(inst, acs.AcsParams(variant="atomic", seed=s, m=32)) for s in (1, 2, 3)]
    try:
        assert acs.Colony.island_exchange_local(cols) == LLONG_MAX
        for c in cols:
            assert c.best()[1] == LLONG_MAX  # nothing adopted
        # colony 1 iterates, the others have no tour yet: everyone adopts colony 1's
        cols[1].iterate(2)
        order1, len1 = cols[1].best()
        assert acs.Colony.island_exchange_local(cols) == len1
        for c in cols:
            o, ln = c.best()
            assert ln == len1 and (o == order1).all()
        # and the adopted tour drives a normal iteration (positive pheromone)
        st = cols[0].iterate(2)
        assert 0 < st["global_best_len"][-1] <= len1
        assert (cols[0].pheromone() > 0).all()
    finally:
        for c in cols:
            c.close()


def test_local_exchange_picks_best_and_lowest_rank(acs, gpu):
    I = O.load("d198")
    inst = to_acs(acs, I)
    cols = [acs.Colony(inst, acs.AcsParams(variant=v, seed=s, m=48))
            for v, s in (("relaxed", 4), ("atomic", 5), ("spm", 6), ("relaxed", 7))]
    try:
        for i, c in enumerate(cols):
            c.iterate(1 + 2 * i)
        lens = [c.best()[1] for c in cols]
        w = int(np.argmin(lens))  # argmin: lowest index among equals
        wt = cols[w].best()[0]
        g = acs.Colony.island_exchange_local(cols)
        assert g == min(lens)
        for c in cols:
            o, ln = c.best()
            assert ln == g and (o == wt).all()
        # tie: ranks 2 and 3 get the same better length with different tours;
        # everyone else adopts rank 2's; ranks 2 and 3 keep their own (strict)
        ident = np.arange(I.n, dtype=np.uint32)
        rev = ident[::-1].copy()
        better = g - 1
        cols[2].set_best(ident, better)
        cols[3].set_best(rev, better)
        assert acs.Colony.island_exchange_local(cols) == better
        for i, c in enumerate(cols):
            o, ln = c.best()
            assert ln == better
            assert (o == (rev if i == 3 else ident)).all()
        # traces stay monotone after adoption
        for c in cols:
            st = c.iterate(3)
            gb = st["global_best_len"]
            assert (np.diff(gb) <= 0).all() and gb[0] <= better
    finally:
        for c in cols:
            c.close()


def test_local_exchange_argument_checks(acs, gpu):
    inst = to_acs(acs, O.load("d198"))
    other = to_acs(acs, O.load("a280"))
    with acs.Colony(inst, acs.AcsParams(seed=1, m=8)) as a, acs.Colony(other, acs.AcsParams(seed=1, m=8)) as b:
        with pytest.raises(acs.AcsError):
            acs.Colony.island_exchange_local([a, b])  # different instance sizes
        with pytest.raises(acs.AcsError):
            acs.Colony.island_exchange_local([a, a])  # duplicate colony
        assert acs.Colony.island_exchange_local([a]) == LLONG_MAX


def test_nccl_exchange_before_first_iteration(acs, gpu):
    """the LLONG_MAX sentinel must not be shifted into a winning key."""
    inst = to_acs(acs, O.load("d198"))
    try:
        uid = acs.Colony.nccl_unique_id()
    except acs.AcsError as e:
        pytest.skip(f"NCCL not loadable here: {e}")
    with acs.Colony(inst, acs.AcsParams(variant="atomic", seed=3, m=32)) as col:
        col.island_init(uid, 1, 0)
        assert col.island_exchange() == LLONG_MAX
        assert col.best()[1] == LLONG_MAX
        st = col.iterate(2)
        assert 0 < st["global_best_len"][-1] < LLONG_MAX
        assert (col.pheromone() > 0).all()
        assert col.island_exchange() == st["global_best_len"][-1]


def test_island_init_rank_limits(acs, gpu):
    inst = to_acs(acs, O.load("d198"))
    try:
        uid = acs.Colony.nccl_unique_id()
    except acs.AcsError as e:
        pytest.skip(f"NCCL not loadable here: {e}")
    with acs.Colony(inst, acs.AcsParams(seed=3, m=8)) as col:
        with pytest.raises(acs.AcsError):
            col.island_init(uid, 70000, 0)  # > 65536 ranks cannot be keyed
        with pytest.raises(acs.AcsError):
            col.island_init(uid, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_real_colonies_gloo(gpu, tmp_path):
    """world_size 2, each rank a real Colony on cuda:0, host exchange over gloo
    (two processes, as torchrun would start them: tests/island_worker.py)."""
    import json
    import subprocess
    import sys
    port = _free_port()
    here = os.path.dirname(os.path.abspath(__file__))
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(here, "island_worker.py"),
                                       str(tmp_path / f"r{r}.json")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=300)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    res = {r: json.load(open(tmp_path / f"r{r}.json")) for r in (0, 1)}
    own = [res[r]["own"] for r in (0, 1)]
    best = min(own)
    winner = int(np.argmin(own))
    for r in (0, 1):
        o = res[r]
        assert o["g"] == best and o["len"] == best
        assert o["tour"] == res[winner]["tour"]
        tr = o["trace"]
        assert all(b <= a for a, b in zip(tr, tr[1:])), "global-best trace must be monotone"
        assert tr[-1] <= best
    # tie at the exchange: equal lengths, each keeps its own tour (strict adoption)
    assert res[0]["tie_g"] == res[1]["tie_g"] == 1000
    assert res[0]["tie_tour0"] == 0 and res[1]["tie_tour0"] == 441
