"""Per-iteration device time of one colony over a long run (does the
iteration cost drift as the pheromone converges?).
usage: python scripts/iter_profile.py [instance] [variant] [iterations]"""
import sys
import time

sys.path.insert(0, ".")
import paper_1605_02669_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "pr2392"
variant = sys.argv[2] if len(sys.argv) > 2 else "atomic"
K = int(sys.argv[3]) if len(sys.argv) > 3 else 200
inst = P.load_instance(name)
with P.Colony(inst, P.AcsParams(variant=variant, rng="philox" if variant in ("atomic", "relaxed") else "xoshiro")) as col:
    ms, cms, fb = [], [], []
    c_prev = col.counters()
    t0 = time.perf_counter()
    for i in range(K):
        col.iterate(1)
        tot, con = col.last_timing()
        c = col.counters()
        ms.append(tot)
        cms.append(con)
        fb.append((c["fallback_steps"] - c_prev["fallback_steps"], c["fallback_full"] - c_prev["fallback_full"]))
        c_prev = c
    wall = time.perf_counter() - t0
    for i in list(range(0, K, max(1, K // 20))) + [K - 1]:
        print(f"it {i:4d} total {ms[i]:7.3f} ms construct {cms[i]:7.3f} ms fallbacks {fb[i][0]:7d} full {fb[i][1]:6d}")
    print(f"{variant} {name}: {K} iterations, device sum {sum(ms):.1f} ms, wall {wall * 1e3:.1f} ms")
