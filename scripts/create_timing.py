#!/usr/bin/env python
"""Wall time of acs_gpu_create (host coordinates H2D + every setup kernel:
distance / eta tables, top-k candidate lists, packed and next-nearest rows,
the NN tour for tau0) -- the setup share of bench.py's e2e leg.

    python scripts/create_timing.py --instance pr2392 --reps 10
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_02669_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--instance", default="pr2392")
ap.add_argument("--variant", default="atomic")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
inst = P.load_instance(a.instance)
p = P.AcsParams(variant=a.variant, seed=1, rng="philox")
P.Colony(inst, p).close()  # lazy module loading
ms = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    c = P.Colony(inst, p)
    ms.append((time.perf_counter() - t0) * 1e3)
    tau0 = c.info.tau0
    c.close()
print(f"{a.instance} {a.variant} create ms: median {statistics.median(ms):.3f} min {min(ms):.3f} tau0 {tau0!r}")
