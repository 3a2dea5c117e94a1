"""Several island colonies of m = 256 ants in ONE process on one B200, each
driven by its own host thread on its own stream (ctypes releases the GIL), so
their construction kernels run concurrently.  (Separate processes on one GPU
time-slice instead: scripts/islands_m256.sh.)  Colonies exchange the best tour
on the host every X iterations (acs_gpu_set_best).  Prints tours/s vs the
number of colonies.
usage: python scripts/colonies_threads.py [variant] [k] [iterations]"""
import sys
import threading
import time

sys.path.insert(0, ".")
import paper_1605_02669_b200 as P  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "relaxed"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 40
X = 10
inst = P.load_instance("pr2392")
for N in (1, 2, 4, 8, 16):
    cols = [P.Colony(inst, P.AcsParams(variant=variant, m=256, k=k, seed=c * 0x9E3779B97F4A7C15 % (1 << 63)))
            for c in range(N)]
    for c in cols:
        c.iterate(2)  # warm
    t0 = time.perf_counter()
    for r in range(iters // X):
        th = [threading.Thread(target=c.iterate, args=(X,)) for c in cols]
        for t in th:
            t.start()
        for t in th:
            t.join()
        best = min((c.best() for c in cols), key=lambda b: b[1])
        for c in cols:
            c.set_best(*best)
    dt = time.perf_counter() - t0
    print(f"{variant} k={k} colonies={N:2d}: {N * 256 * iters / dt:10.0f} tours/s, best {best[1]}", flush=True)
    for c in cols:
        c.close()
