#!/usr/bin/env python
"""Solution-quality study on the GPU (BASELINE metric, second half): mean and
best % over the known optimum across seeds, per instance and pheromone-memory
variant, with the paper's parameters (beta=3, alpha=0.2, rho=0.01,
q0=(n-20)/n, cl=32, m=n, k=1) unless overridden.  Budget: a fixed iteration
count, or a wall-clock limit (--time-limit-s, the paper's equal-time
protocol) in which case the per-iteration (ms, L_gb) trace of every run is
kept for quality-vs-time curves.  Product API only;
the CPU oracle leg of a comparison is tests/studies/oracle_quality.py.

    python tools/quality.py --instances d198 pcb442 --variants atomic relaxed spm \
        --seeds 30 --iterations 1000 --out profiles/quality_r01.json
    python tools/quality.py --instances pr1002 --variants spm relaxed --ants 256 --k 4 \
        --time-limit-s 26.39 --seeds 5 --out profiles/quality_time_pr1002.json
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import paper_1605_02669_b200 as P  # noqa: E402


def checkpoints(trace_ms, trace, marks_ms):
    """L_gb reached by each time mark (None before the first iteration ends)."""
    out = []
    for t in marks_ms:
        k = int(np.searchsorted(np.asarray(trace_ms), t, side="right"))
        out.append(int(trace[k - 1]) if k else None)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", nargs="+", default=["d198", "pcb442", "rat783", "pr1002", "pr2392"])
    ap.add_argument("--variants", nargs="+", default=["atomic", "relaxed", "spm", "deferred"])
    ap.add_argument("--seeds", type=int, default=30)
    ap.add_argument("--seed0", type=int, default=0)
    ap.add_argument("--iterations", type=int, default=1000)
    ap.add_argument("--time-limit-s", type=float, default=0.0)
    ap.add_argument("--ants", type=int, default=0)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--slots", type=int, default=8)
    ap.add_argument("--rng", default="xoshiro", choices=["xoshiro", "philox"])
    ap.add_argument("--trace-points", type=int, default=200, help="trace samples kept per run (time mode)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {"params": dict(vars(a), resident_ants=os.environ.get("ACS_RESIDENT_ANTS")), "results": {}}
    for name in a.instances:
        inst = P.load_instance(name)
        opt = inst.optimum
        for v in a.variants:
            lens, secs, iters, traces = [], [], [], []
            for seed in range(a.seed0, a.seed0 + a.seeds):
                p = P.AcsParams(variant=v, m=a.ants, k=a.k, s=a.slots, seed=seed, rng=a.rng,
                                iterations=0 if a.time_limit_s else a.iterations, time_limit_s=a.time_limit_s)
                t0 = time.perf_counter()
                r = P.run(inst, p)
                secs.append(time.perf_counter() - t0)
                lens.append(int(r.best_length))
                iters.append(int(r.iterations))
                if a.time_limit_s:
                    idx = np.unique(np.linspace(0, len(r.trace) - 1, a.trace_points).astype(int))
                    traces.append({"ms": [round(float(r.trace_ms[i]), 2) for i in idx],
                                   "len": [int(r.trace[i]) for i in idx]})
            rec = {"best_len": int(min(lens)), "mean_len": float(np.mean(lens)),
                   "mean_s_per_run": round(float(np.mean(secs)), 3), "mean_iterations": float(np.mean(iters)),
                   "lengths": lens}
            if opt:
                err = [100.0 * (x - opt) / opt for x in lens]
                rec.update(mean_pct=round(float(np.mean(err)), 3), min_pct=round(float(np.min(err)), 3))
            if traces:
                marks = [a.time_limit_s * 1e3 * f for f in (0.01, 0.05, 0.1, 0.25, 0.5, 1.0)]
                rec["traces"] = traces
                rec["checkpoints_ms"] = marks
                rec["mean_len_at_checkpoints"] = [
                    float(np.mean([c for c in col if c is not None])) if any(c is not None for c in col) else None
                    for col in zip(*[checkpoints(t["ms"], t["len"], marks) for t in traces])]
            res["results"][f"{name}/{v}"] = rec
            print(name, v, rec.get("mean_pct"), rec.get("min_pct"), f"{np.mean(secs):.2f}s/run",
                  f"{np.mean(iters):.0f} it/run", flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
