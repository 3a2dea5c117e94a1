#!/usr/bin/env python
"""Lost-update rate of the RELAXED construction (ACS-GPU-Alt) against the
number of ants in flight (--variant spm: the share of selective-record
updates made from a stale copy of the record).  Needs the instrumented library
(make ab V=lost DEFS=-DACS_COUNT_LOST): every relaxed pheromone write is an
exchange, and a write whose old value differs from the value its update read
overwrote (lost) another ant's update.

    python scripts/lost_updates.py --instances pcb442 rat783 nrw1379 pr2392 --resident 0 128 6
(each residency in its own process: ACS_RESIDENT_ANTS is read once)
"""
import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(instances, iters, seed, variant):
    sys.path.insert(0, REPO)
    import paper_1605_02669_b200 as P
    out = {}
    for name in instances:
        inst = P.load_instance(name)
        with P.Colony(inst, P.AcsParams(variant=variant, seed=seed, rng="philox")) as col:
            st = col.iterate(iters)
            c = col.counters()
        opt = inst.optimum
        out[name] = {"relaxed_writes": c["relaxed_writes"], "lost_updates": c["lost_updates"],
                     "lost_rate": round(c["lost_updates"] / max(c["relaxed_writes"], 1), 6),
                     "best_pct": round(100.0 * (int(st["global_best_len"][-1]) - opt) / opt, 3),
                     "iterations": iters}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instances", nargs="+", default=["pcb442", "rat783", "nrw1379", "pr2392"])
    ap.add_argument("--resident", nargs="+", type=int, default=[0, 128, 6])
    ap.add_argument("--iterations", type=int, default=100)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--variant", default="relaxed", help="relaxed: lost trail updates; spm: stale record updates")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    if a.child:
        return child(a.instances, a.iterations, a.seed, a.variant)
    res = {"params": vars(a), "results": {}}
    for w in a.resident:
        env = dict(os.environ, ACS_LIB_VARIANT="lost", ACS_RESIDENT_ANTS=str(w))
        r = subprocess.run([sys.executable, __file__, "--child", "--instances", *a.instances, "--iterations",
                            str(a.iterations), "--seed", str(a.seed), "--variant", a.variant], env=env,
                           capture_output=True, text=True)
        if r.returncode:
            print(r.stderr[-2000:])
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        res["results"][f"W{w if w else 'all'}"] = d
        for name, x in d.items():
            print(f"W={w or 'all'} {name}: lost {x['lost_updates']} of {x['relaxed_writes']} writes "
                  f"({100 * x['lost_rate']:.3f}%), best {x['best_pct']}% after {x['iterations']} it", flush=True)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
