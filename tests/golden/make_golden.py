#!/usr/bin/env python
"""Generate tests/golden/reference_golden.json from the REFERENCE's own code.

Runs only where /root/reference exists: oracle/_ref/libacsref.so is compiled
(oracle/Makefile) from the unmodified reference sources
(proj/src/tsp_instance.cpp + proj/include/acs/*.hpp) plus an extern "C" shim.
The fixture is committed, so the GPU box (which has no /root/reference) and
the CPU suite check against it:

  * per TSPLIB instance (proj/data/*.tsp): FNV-1a-64 of the n x n distance
    table and of the cl = 32 candidate lists (tsp_instance.cpp:219-252), the
    first 8 candidates of node 0 with distances, nn_tour_length from starts
    0..3 (cpp:254-280), tau0 = 1/(n L_nn(0)), tour_length of the identity;
  * RngStream (rng.hpp:16-84) scripts: next_u64 / uniform01 bits /
    uniform_int outputs for derive(seed, it, ant) and RngStream(seed).

    python tests/golden/make_golden.py   # rewrites the fixture
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402

INSTANCES = ["d198", "a280", "lin318", "pcb442", "att532", "rat783", "pr1002", "nrw1379", "pr2392"]
RNG_CASES = [(42, 0, 0, 1), (42, 1, 7, 1), (0, 0, 0, 0), (1, 0, 0, 1), (20161017, 3, 2391, 1), (7, 999, 12, 1)]
RNG_OPS = [0, 0, 1, 2, 2, 1, 0, 2, 2, 2, 1, 0]
RNG_ARGS = [0, 0, 0, 280, 198, 0, 0, 2392, 1, 10000, 0, 0]


def main():
    if not O.Reference.available():
        sys.exit("oracle/_ref/libacsref.so missing: build it with `make -C oracle` where /root/reference exists")
    ref = O.Reference()
    out = {"source": "reference code (oracle/_ref/libacsref.so from /root/reference/proj/src/tsp_instance.cpp)",
           "instances": {}, "rng": []}
    for name in INSTANCES:
        text = O.read_tsplib_text(name)
        R, err = ref.parse(text)
        assert R is not None, err
        n = R.n
        rec = {"n": n, "type": R.type}
        if n <= 4096:
            rec["dist_fnv"] = O.fnv1a64(R.distance_table())
        cand = R.candidates(32)
        L = min(32, n - 1)
        rec["cand_fnv"] = O.fnv1a64(cand)
        head = cand.reshape(n, L)[0, :8]  # noqa: E501
        rec["cand0_head"] = [int(x) for x in head]
        rec["cand0_dist"] = [int(R.distance(0, int(x))) for x in head]
        rec["nn_len"] = [int(R.nn_tour_length(s)) for s in range(4)]
        rec["tau0"] = 1.0 / (n * rec["nn_len"][0])
        rec["identity_len"] = int(R.tour_length(np.arange(n, dtype=np.uint32)))
        out["instances"][name] = rec
        print(name, rec["cand_fnv"], rec["nn_len"][0])
    for seed, it, ant, derive in RNG_CASES:
        vals = ref.rng_script(seed, it, ant, derive, RNG_OPS, RNG_ARGS)
        out["rng"].append({"seed": seed, "iteration": it, "ant": ant, "derive": derive, "ops": RNG_OPS,
                           "args": RNG_ARGS, "out": [f"{int(v):016x}" for v in vals]})
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
