#!/usr/bin/env python
"""CPU leg of the quality studies (test infrastructure: runs the oracle, the
SPEC restatement in oracle/, never the product).  Same JSON shape as
tools/quality.py so the two can be compared with the paper's rank-sum test:

    python tests/studies/oracle_quality.py run --instances pr1002 --mode relaxed --ants 256 --k 4 \
        --time-limit-s 26.39 --seeds 3 --threads 0 --out /tmp/oracle_pr1002.json
    python tests/studies/oracle_quality.py compare gpu.json oracle.json

Time-limited runs: the oracle has no wall-clock budget, so one iteration is
timed first and the run is given floor(limit / t_iter) iterations; the trace
timestamps are i * (loop_ms / iterations), i.e. uniform iteration cost.
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402

MODES = {"seq": O.SEQ, "sync": O.SYNC, "relaxed": O.RELAXED}


def run(a):
    orc = O.Oracle()
    threads = a.threads or os.cpu_count() or 1
    res = {"params": vars(a), "results": {}}
    opt_cat = O.optima()
    for name in a.instances:
        I = O.load(name)
        opt = opt_cat.get(name)
        kw = dict(m=a.ants or None, mode=MODES[a.mode], memory=O.SELECTIVE if a.memory == "selective" else O.DENSE,
                  consistent=1 if a.consistent else 0, threads=threads if a.mode != "seq" else 1, k=a.k, s=a.slots,
                  want_routes=False)
        iters = a.iterations
        if a.time_limit_s:
            orc.run(I, iterations=1, seed=10**6, **kw)  # warm-up (thread pool, page-in)
            probe = orc.run(I, iterations=3, seed=10**6 + 1, **kw)
            iters = max(1, int(a.time_limit_s * 1e3 / max(probe["loop_ms"] / 3, 1e-3)))
        lens, traces, secs = [], [], []
        for seed in range(a.seed0, a.seed0 + a.seeds):
            o = orc.run(I, iterations=iters, seed=seed, **kw)
            lens.append(int(o["best_len"]))
            secs.append(o["elapsed_ms"] / 1e3)
            if a.time_limit_s:
                per = o["loop_ms"] / iters
                idx = np.unique(np.linspace(0, iters - 1, a.trace_points).astype(int))
                traces.append({"ms": [round(float((i + 1) * per), 2) for i in idx],
                               "len": [int(o["trace"][i]) for i in idx]})
        key = f"{name}/oracle-{a.mode}{'-selective' if a.memory == 'selective' else ''}"
        rec = {"best_len": int(min(lens)), "mean_len": float(np.mean(lens)), "mean_s_per_run": float(np.mean(secs)),
               "mean_iterations": iters, "threads": kw["threads"], "lengths": lens}
        if opt:
            err = [100.0 * (x - opt) / opt for x in lens]
            rec.update(mean_pct=round(float(np.mean(err)), 3), min_pct=round(float(np.min(err)), 3))
        if traces:
            rec["traces"] = traces
        res["results"][key] = rec
        print(key, rec.get("mean_pct"), rec.get("min_pct"), f"{iters} it/run", flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


def compare(a):
    """Two-sided rank-sum p between every pair of results with the same instance."""
    from scipy.stats import mannwhitneyu
    recs = {}
    for path in a.files:
        recs.update(json.load(open(path))["results"])
    out = []
    keys = sorted(recs)
    for i, x in enumerate(keys):
        for y in keys[i + 1:]:
            if x.split("/")[0] != y.split("/")[0]:
                continue
            lx, ly = recs[x]["lengths"], recs[y]["lengths"]
            p = float(mannwhitneyu(lx, ly, alternative="two-sided").pvalue) if min(len(lx), len(ly)) >= 3 else None
            out.append({"a": x, "b": y, "mean_pct_a": recs[x].get("mean_pct"), "mean_pct_b": recs[y].get("mean_pct"),
                        "p": p})
            print(x, recs[x].get("mean_pct"), "vs", y, recs[y].get("mean_pct"), "p =", p)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--instances", nargs="+", required=True)
    r.add_argument("--mode", choices=list(MODES), default="seq")
    r.add_argument("--memory", choices=["dense", "selective"], default="dense")
    r.add_argument("--consistent", action="store_true")
    r.add_argument("--seeds", type=int, default=3)
    r.add_argument("--seed0", type=int, default=0)
    r.add_argument("--iterations", type=int, default=1000)
    r.add_argument("--time-limit-s", type=float, default=0.0)
    r.add_argument("--ants", type=int, default=0)
    r.add_argument("--k", type=int, default=1)
    r.add_argument("--slots", type=int, default=8)
    r.add_argument("--threads", type=int, default=0, help="0 = all host cores (ignored for seq)")
    r.add_argument("--trace-points", type=int, default=200)
    r.add_argument("--out", default=None)
    c = sub.add_parser("compare")
    c.add_argument("files", nargs="+")
    c.add_argument("--out", default=None)
    a = ap.parse_args()
    run(a) if a.cmd == "run" else compare(a)


if __name__ == "__main__":
    main()
