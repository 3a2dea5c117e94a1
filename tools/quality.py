#!/usr/bin/env python
"""Solution-quality study (BASELINE metric, second half): mean and best % over
the known optimum across seeds, per instance and pheromone-memory variant,
with the paper's parameters (beta=3, alpha=0.2, rho=0.01, q0=(n-20)/n, cl=32,
m=n, k=1) unless overridden.  Optionally compares a variant against the CPU
oracle with the paper's two-sided Wilcoxon rank-sum test.

    python tools/quality.py --instances d198 pcb442 --variants atomic relaxed spm \
        --seeds 30 --iterations 1000 --out profiles/quality_r01.json
    python tools/quality.py --instances d198 --variants atomic --oracle-mode seq --seeds 10
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402  (instances + optimum catalog; oracle engine only with --oracle-mode)
import paper_1605_02669_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", nargs="+", default=["d198", "pcb442", "rat783", "pr1002", "pr2392"])
    ap.add_argument("--variants", nargs="+", default=["atomic", "relaxed", "spm", "deferred"])
    ap.add_argument("--seeds", type=int, default=30)
    ap.add_argument("--iterations", type=int, default=1000)
    ap.add_argument("--ants", type=int, default=0)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--oracle-mode", choices=["seq", "sync", "relaxed"], default=None)
    ap.add_argument("--oracle-threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    opt = O.optima()
    res = {"params": vars(a), "results": {}}
    for name in a.instances:
        I = O.load(name)
        inst = P.TspInstance(I.name, I.type, I.xs.copy(), I.ys.copy(), opt.get(name))
        for v in a.variants:
            lens, secs = [], []
            for seed in range(a.seeds):
                p = P.AcsParams(variant=v, m=a.ants, k=a.k, seed=seed, iterations=a.iterations)
                t0 = time.perf_counter()
                r = P.run(inst, p)
                secs.append(time.perf_counter() - t0)
                lens.append(int(r.best_length))
            err = [100.0 * (x - opt[name]) / opt[name] for x in lens]
            res["results"][f"{name}/{v}"] = {
                "mean_pct": round(float(np.mean(err)), 3), "min_pct": round(float(np.min(err)), 3),
                "best_len": int(min(lens)), "mean_s_per_run": round(float(np.mean(secs)), 3),
                "lengths": lens}
            print(name, v, res["results"][f"{name}/{v}"]["mean_pct"], res["results"][f"{name}/{v}"]["min_pct"],
                  f"{np.mean(secs):.2f}s/run", flush=True)
            if a.oracle_mode:
                mode = {"seq": O.SEQ, "sync": O.SYNC, "relaxed": O.RELAXED}[a.oracle_mode]
                orc = O.Oracle()
                olens = [int(orc.run(I, m=a.ants or None, iterations=a.iterations, seed=s, mode=mode,
                                     threads=a.oracle_threads, k=a.k, want_routes=False)["best_len"])
                         for s in range(a.seeds)]
                from scipy.stats import ranksums
                oerr = [100.0 * (x - opt[name]) / opt[name] for x in olens]
                p_val = float(ranksums(err, oerr).pvalue)
                res["results"][f"{name}/oracle-{a.oracle_mode}"] = {
                    "mean_pct": round(float(np.mean(oerr)), 3), "min_pct": round(float(np.min(oerr)), 3),
                    "lengths": olens, f"ranksum_p_vs_{v}": p_val}
                print(name, f"oracle-{a.oracle_mode}", round(float(np.mean(oerr)), 3), f"p={p_val:.3f}", flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
