"""GPU instance layer vs the oracle / golden vectors: distances, candidate
lists (K2), NN tour, tour-length eval (K6), device RNG streams.  Bit-exact."""
import numpy as np
import pytest

import oracle as O
from helpers import GOLDEN, RND10K_CAND_FNV, RND10K_NN, TSPLIB, small_instance, to_acs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", TSPLIB)
def test_distance_table_and_candidates_golden(acs, gpu, name):
    I = O.load(name)
    inst = to_acs(acs, I)
    dist_fnv, cand_fnv, nn, _ = GOLDEN[name]
    assert O.fnv1a64(inst.distance_table()) == dist_fnv
    c = acs.build_candidates(inst, 32)
    assert c.list_len == 32
    assert O.fnv1a64(c.flat) == cand_fnv
    assert acs.nn_tour_length(inst, 0) == nn


def test_rnd10k_candidates_and_nn(acs, gpu):
    I = O.rnd_instance()
    inst = to_acs(acs, I)
    assert O.fnv1a64(acs.build_candidates(inst, 32).flat) == RND10K_CAND_FNV
    assert acs.nn_tour_length(inst, 0) == RND10K_NN


@pytest.mark.parametrize("cl", [1, 2, 7, 16, 31, 32])
@pytest.mark.parametrize("name", ["rat783", "pcb442", "att532"])
def test_candidates_vs_oracle_cl(acs, orc, gpu, name, cl):
    I = O.load(name)
    got = acs.build_candidates(to_acs(acs, I), cl)
    want = orc.candidates(I, cl)
    assert got.list_len == want.shape[1]
    assert (got.flat.reshape(want.shape) == want).all()


@pytest.mark.parametrize("n,cl", [(3, 32), (4, 2), (10, 32), (33, 32), (64, 32), (100, 5)])
@pytest.mark.parametrize("typ", [O.EUC_2D, O.CEIL_2D, O.ATT])
def test_candidates_small_and_ragged(acs, orc, gpu, n, cl, typ):
    I = small_instance(n, seed=n, scale=50, typ=typ)  # heavy ties on a 50x50 grid
    got = acs.build_candidates(to_acs(acs, I), cl)
    want = orc.candidates(I, cl)
    assert (got.flat.reshape(want.shape) == want).all()
    assert (to_acs(acs, I).distance_table() == orc.distance_table(I)).all()


@pytest.mark.parametrize("name", ["d198", "a280", "att532", "rat783"])
def test_nn_tour_from_several_starts(acs, orc, gpu, name):
    I = O.load(name)
    inst = to_acs(acs, I)
    for start in (0, 1, I.n // 2, I.n - 1):
        assert acs.nn_tour_length(inst, start) == orc.nn_tour_length(I, start)


def test_duplicate_points_nn_and_candidates(acs, orc, gpu):
    xs = np.array([0, 0, 0, 5, 5, 9, 9, 9], np.float64)
    ys = np.array([0, 0, 0, 5, 5, 9, 9, 1], np.float64)
    I = O.Coords("dups", O.EUC_2D, xs, ys)
    inst = to_acs(acs, I)
    for s in range(I.n):
        assert acs.nn_tour_length(inst, s) == orc.nn_tour_length(I, s)
    assert (acs.build_candidates(inst, 32).flat.reshape(I.n, -1) == orc.candidates(I, 32)).all()


@pytest.mark.parametrize("name", ["pr2392", "d198", "att532"])
def test_tour_lengths_eval(acs, orc, gpu, name):
    I = O.load(name)
    inst = to_acs(acs, I)
    rng = np.random.default_rng(3)
    routes = np.stack([np.arange(I.n)] + [rng.permutation(I.n) for _ in range(17)]).astype(np.uint32)
    got = inst.tour_lengths(routes)
    want = [orc.tour_length(I, r) for r in routes]
    assert got.tolist() == want
    if name == "pr2392":
        assert got[0] == 378032  # file order is optimal
    if name == "d198":
        assert got[0] == 22498


def _rng_script(acs, kind, seed, it, ant, derive, ops, args):
    import ctypes as C
    from paper_1605_02669_b200 import _native as N
    ops = np.asarray(ops, np.int32)
    args = np.asarray(args, np.uint64)
    out = np.zeros(len(ops), np.uint64)
    N.check(N.lib().acs_gpu_rng_script(kind, seed, it, ant, derive, ops.ctypes.data_as(C.c_void_p),
                                       args.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                       len(ops), 0), "rng_script")
    return out


def test_device_rng_matches_reference_kats(acs, gpu):
    o = _rng_script(acs, 0, 42, 0, 0, 1, [0, 0, 1], [0, 0, 0])
    assert f"{int(o[0]):016x}" == "c986fd807e5b8ab5"
    assert f"{int(o[1]):016x}" == "e071ea15f19664d1"
    assert o[2:3].view(np.float64)[0] == 0.44735932804098311
    o = _rng_script(acs, 0, 42, 1, 7, 1, [0, 2], [0, 280])
    assert f"{int(o[0]):016x}" == "1e41e6edf5d70818" and int(o[1]) == 133
    o = _rng_script(acs, 0, 0, 0, 0, 0, [0], [0])
    assert f"{int(o[0]):016x}" == "99ec5f36cb75f2b4"


@pytest.mark.parametrize("kind", [O.XOSHIRO, O.PHILOX])
def test_device_rng_matches_oracle_stream(acs, orc, gpu, kind):
    import ctypes as C
    rng = np.random.default_rng(11)
    ops = rng.integers(0, 3, 3000).astype(np.int32)
    args = rng.integers(1, 1 << 40, 3000).astype(np.uint64)
    args[::7] = rng.integers(1, 5, len(args[::7]))
    for (seed, it, ant) in [(0, 0, 0), (7, 3, 5), (2**63 + 5, 999, 2391)]:
        got = _rng_script(acs, kind, seed, it, ant, 1, ops, args)
        r = orc.rng_derive(seed, it, ant, kind)
        lib = orc.lib
        want = []
        for op, a in zip(ops, args):
            if op == 0:
                want.append(lib.orc_rng_next_u64(C.byref(r)))
            elif op == 1:
                want.append(int(np.float64(lib.orc_rng_uniform01(C.byref(r))).view(np.uint64)))
            else:
                want.append(lib.orc_rng_uniform_int(C.byref(r), int(a)))
        assert got.tolist() == want
