"""Checks against tests/golden/reference_golden.json: values produced by the
REFERENCE's own code (oracle/_ref, compiled from /root/reference sources by
tests/golden/make_golden.py).  The fixture travels with the repo, so these run
where /root/reference does not exist (the GPU box).

CPU: the oracle restatement reproduces every fixture value.
GPU: the sm_100a setup kernels (K2 candidate lists, NN tour, tour lengths)
and the device RngStream reproduce them through the C-ABI.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

import oracle as O
from helpers import to_acs

GOLDEN = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                     "reference_golden.json")))
NAMES = sorted(GOLDEN["instances"])


def _orc_rng(orc, case):
    r = orc.rng_derive(case["seed"], case["iteration"], case["ant"]) if case["derive"] else orc.rng_seed(case["seed"])
    lib, out = orc.lib, []
    for op, a in zip(case["ops"], case["args"]):
        if op == 0:
            out.append(lib.orc_rng_next_u64(C.byref(r)))
        elif op == 1:
            out.append(int(np.float64(lib.orc_rng_uniform01(C.byref(r))).view(np.uint64)))
        else:
            out.append(lib.orc_rng_uniform_int(C.byref(r), int(a)))
    return [f"{v:016x}" for v in out]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_fixture(orc, name):
    g = GOLDEN["instances"][name]
    I = O.load(name)
    assert I.n == g["n"] and I.type == g["type"]
    if "dist_fnv" in g:
        assert O.fnv1a64(orc.distance_table(I)) == g["dist_fnv"]
    cand = orc.candidates(I, 32)
    assert O.fnv1a64(cand) == g["cand_fnv"]
    assert cand[0, :8].tolist() == g["cand0_head"]
    assert [orc.distance(I, 0, int(v)) for v in g["cand0_head"]] == g["cand0_dist"]
    assert [orc.nn_tour_length(I, s) for s in range(4)] == g["nn_len"]
    assert orc.tour_length(I, np.arange(I.n, dtype=np.uint32)) == g["identity_len"]


def test_oracle_rng_matches_reference_fixture(orc):
    for case in GOLDEN["rng"]:
        assert _orc_rng(orc, case) == case["out"], case


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_reference_fixture(acs, gpu, name):
    g = GOLDEN["instances"][name]
    I = O.load(name)
    inst = to_acs(acs, I)
    cand = acs.build_candidates(inst, 32)
    assert O.fnv1a64(cand.flat) == g["cand_fnv"]
    assert [acs.nn_tour_length(inst, s) for s in range(4)] == g["nn_len"]
    assert int(inst.tour_lengths(np.arange(I.n, dtype=np.uint32)[None, :])[0]) == g["identity_len"]
    if "dist_fnv" in g:
        assert O.fnv1a64(inst.distance_table()) == g["dist_fnv"]
    # tau0 of a colony (1 / (n L_nn(0)), SPEC D2) from its own setup NN tour
    with acs.Colony(inst, acs.AcsParams(variant="atomic", m=32, seed=1)) as col:
        assert col.info.tau0 == g["tau0"] and col.info.nn_len == g["nn_len"][0]


@pytest.mark.gpu
def test_gpu_rng_matches_reference_fixture(acs, gpu):
    from paper_1605_02669_b200 import _native as N
    for case in GOLDEN["rng"]:
        ops = np.asarray(case["ops"], np.int32)
        args = np.asarray(case["args"], np.uint64)
        out = np.zeros(len(ops), np.uint64)
        N.check(N.lib().acs_gpu_rng_script(0, case["seed"], case["iteration"], case["ant"], case["derive"],
                                           ops.ctypes.data_as(C.c_void_p), args.ctypes.data_as(C.c_void_p),
                                           out.ctypes.data_as(C.c_void_p), len(ops), 0), "rng_script")
        assert [f"{int(v):016x}" for v in out] == case["out"], case
