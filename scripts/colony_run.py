#!/usr/bin/env python
"""Run one colony for a few iterations (a target for ncu captures):
    python scripts/colony_run.py --variant relaxed --ants 128 --iters 4 [--instance pr2392]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_02669_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="relaxed")
ap.add_argument("--ants", type=int, default=0)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--instance", default="pr2392")
ap.add_argument("--rng", default="auto")
a = ap.parse_args()
inst = P.load_instance(a.instance)
rng = a.rng if a.rng != "auto" else ("philox" if a.variant in ("atomic", "relaxed", "spm") else "xoshiro")
with P.Colony(inst, P.AcsParams(variant=a.variant, m=a.ants or inst.n, seed=1, rng=rng)) as col:
    for _ in range(a.iters):
        col.iterate(1)
        print(a.variant, col.last_timing())
