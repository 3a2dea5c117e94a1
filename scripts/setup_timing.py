#!/usr/bin/env python
"""SURVEY 8(d) CPU timing (i): the reference's own setup path vs the GPU.

For each instance: the REFERENCE code's build_candidates (cl = 32) and
nn_tour_length(0) (oracle/_ref/libacsref.so, compiled from
/root/reference/proj/src/tsp_instance.cpp; OpenMP inside build_candidates,
cpp:230) at 1 thread and at every host thread, against the sm_100a K2 top-k
kernel and the NN-tour kernel through the C-ABI (host buffers in/out, wall
time of the call, warm).  Results are checked equal (FNV of flat_, L_nn).

    python scripts/setup_timing.py [--out profiles/setup_timing_r01.json]
Run on the GPU box: oracle/_ref travels with the snapshot (git-ignored only).
"""
import argparse
import json
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

INSTANCES = ["d198", "pcb442", "rat783", "pr1002", "nrw1379", "pr2392", "rnd10k"]

CHILD = r"""
import json, sys, time
sys.path.insert(0, %r)
import oracle as O
ref = O.Reference()
out = {}
for name in %r:
    I = O.load(name) if name != "rnd10k" else O.rnd_instance()
    R = ref.make(I)
    R.candidates(32)  # warm (thread pool, page-in)
    t0 = time.perf_counter(); c = R.candidates(32); t1 = time.perf_counter()
    nn = R.nn_tour_length(0); t2 = time.perf_counter()
    out[name] = {"cand_ms": (t1 - t0) * 1e3, "nn_ms": (t2 - t1) * 1e3, "cand_fnv": O.fnv1a64(c), "nn": int(nn)}
print(json.dumps(out))
"""


def ref_times(threads):
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    r = subprocess.run([sys.executable, "-c", CHILD % (REPO, INSTANCES)], env=env, capture_output=True, text=True,
                       timeout=1800)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def gpu_times():
    import oracle as O
    import paper_1605_02669_b200 as P
    out = {}
    for name in INSTANCES:
        I = O.load(name) if name != "rnd10k" else O.rnd_instance()
        inst = P.TspInstance(I.name, I.type, I.xs.copy(), I.ys.copy())
        P.build_candidates(inst, 32)
        P.nn_tour_length(inst, 0)  # warm (module load)
        t0 = time.perf_counter(); c = P.build_candidates(inst, 32); t1 = time.perf_counter()
        nn = P.nn_tour_length(inst, 0); t2 = time.perf_counter()
        out[name] = {"cand_ms": (t1 - t0) * 1e3, "nn_ms": (t2 - t1) * 1e3, "cand_fnv": O.fnv1a64(c.flat),
                     "nn": int(nn)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ncpu = os.cpu_count() or 1
    r1, rn, g = ref_times(1), ref_times(ncpu), gpu_times()
    rows = {}
    for name in INSTANCES:
        assert r1[name]["cand_fnv"] == rn[name]["cand_fnv"] == g[name]["cand_fnv"], name
        assert r1[name]["nn"] == g[name]["nn"], name
        rows[name] = {"ref_1thr": r1[name], f"ref_{ncpu}thr": rn[name], "gpu": g[name]}
        print(f"{name:8s} candidates: ref 1 thr {r1[name]['cand_ms']:9.2f} ms, {ncpu} thr {rn[name]['cand_ms']:8.2f} ms,"
              f" GPU {g[name]['cand_ms']:7.2f} ms | NN tour: ref {r1[name]['nn_ms']:8.2f} ms, GPU {g[name]['nn_ms']:7.2f} ms")
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"host_threads": ncpu, "note": "GPU = C-ABI call wall time incl. H2D/D2H, warm; "
                       "acs_gpu_nn_tour_length is the stateless full-scan kernel (the colony setup uses the "
                       "candidate-list NN kernel)", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
