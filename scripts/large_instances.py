#!/usr/bin/env python
"""the large-instance path (the paper's SPM large-instance table
runs pcb3038 .. brd14051; no TSPLIB file above pr2392 is
shipped here, so the sizes are synthetic uniform-random EUC_2D instances of the
same n).  Per variant and colony size: construct ms per iteration (CUDA
events, median of --iters after 2 warm-up iterations), tours/s, device
memory of the context, fallback steps and full scans per iteration.

    python scripts/large_instances.py --sizes 3038 5915 10000 14051 --ants 256 0 --out x.json
"""
import argparse
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1605_02669_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", nargs="+", type=int, default=[14051])
    ap.add_argument("--variants", nargs="+", default=["spm", "relaxed", "atomic"])
    ap.add_argument("--ants", nargs="+", type=int, default=[256, 0], help="0 = m = n")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {"params": vars(a), "results": {}}
    for n in a.sizes:
        inst = P.load_instance(f"rnd{n}")
        for m in a.ants:
            for v in a.variants:
                p = P.AcsParams(variant=v, m=m or n, seed=1, rng="philox")
                with P.Colony(inst, p) as col:
                    col.iterate(2)
                    c0 = col.counters()
                    ms = []
                    for _ in range(a.iters):
                        col.iterate(1)
                        ms.append(col.last_timing()[1])
                    c1 = col.counters()
                    info = col.info
                    best = col.best()[1]
                it = a.iters
                t = statistics.median(ms)
                rec = {"n": n, "m": col.m, "construct_ms": round(t, 3), "tours_per_s": round(col.m / (t / 1e3), 1),
                       "device_bytes": int(info.device_bytes),
                       "fallback_steps_per_iter": round((c1["fallback_steps"] - c0["fallback_steps"]) / it, 1),
                       "fallback_full_per_iter": round((c1["fallback_full"] - c0["fallback_full"]) / it, 1),
                       "fallback_grid_per_iter": round((c1["fallback_grid"] - c0["fallback_grid"]) / it, 1),
                       "steps_per_iter": col.m * (n - 1), "best_len_after": int(best)}
                rec["fallback_full_share"] = round(rec["fallback_full_per_iter"] / max(rec["fallback_steps_per_iter"], 1), 4)
                res["results"][f"rnd{n}/m{col.m}/{v}"] = rec
                print(json.dumps({k: rec[k] for k in ("n", "m", "construct_ms", "tours_per_s", "device_bytes",
                                                      "fallback_steps_per_iter", "fallback_full_per_iter",
                                                      "fallback_grid_per_iter")}),
                      v, flush=True)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
