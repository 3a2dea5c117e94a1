#!/usr/bin/env python
"""A/B timing of kernel builds (make ab V=<name> DEFS=...): construct ms per
launch of the full colony (m = n) and of an isolated 128-ant colony, per
variant, median of ITERS launches after 3 warm-up iterations.

    python scripts/ab_time.py base lf1 lf2 --variants atomic relaxed --instance pr2392
(runs each library in its own process: ACS_LIB_VARIANT selects the .so)
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(instance, variants, iters):
    sys.path.insert(0, REPO)
    import paper_1605_02669_b200 as P
    inst = P.load_instance(instance)
    out = {}
    for v in variants:
        for m in (inst.n, 128):
            rng = "philox" if v in ("atomic", "relaxed", "spm") else "xoshiro"
            with P.Colony(inst, P.AcsParams(variant=v, m=m, seed=1, rng=rng)) as col:
                col.iterate(3)
                ms = []
                for _ in range(iters):
                    col.iterate(1)
                    ms.append(col.last_timing()[1])
                c = col.counters()
            out[f"{v}/{'full' if m == inst.n else 'iso'}"] = round(statistics.median(ms), 4)
            if m == inst.n:
                out[f"{v}/fb_full"] = c["fallback_full"]
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--variants", nargs="+", default=["atomic", "relaxed"])
    ap.add_argument("--instance", default="pr2392")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        return child(a.instance, a.variants, a.iters)
    for spec in a.libs:  # lib[:VAR=value,...] -- e.g. base:ACS_PAIR=0
        lib, _, extra = spec.partition(":")
        env = dict(os.environ, ACS_LIB_VARIANT="" if lib == "base" else lib)
        env.update(kv.split("=", 1) for kv in extra.split(",") if kv)
        r = subprocess.run([sys.executable, __file__, "x", "--child", "--instance", a.instance, "--iters", str(a.iters),
                            "--variants", *a.variants], env=env, capture_output=True, text=True, timeout=900)
        print(spec, r.stdout.strip() or r.stderr[-1500:], flush=True)


if __name__ == "__main__":
    main()
