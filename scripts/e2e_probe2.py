"""e2e variance probe: acs_gpu_run (create + K iterations + D2H + destroy)
repeated, with and without other contexts created in between."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1605_02669_b200 as P  # noqa: E402
from paper_1605_02669_b200 import _native as N  # noqa: E402

inst = P.load_instance("pr2392")
K = 100


def run(variant="atomic", rng="philox"):
    p = P.AcsParams(variant=variant, rng=rng).to_c(inst.n)
    d = inst.desc()
    order = np.empty(inst.n, np.uint32)
    trace = np.empty(K, np.int64)
    bl = C.c_int64()
    t0 = time.perf_counter()
    N.check(N.lib().acs_gpu_run(C.byref(d), C.byref(p), K, 0, order.ctypes.data_as(C.c_void_p), C.byref(bl),
                                trace.ctypes.data_as(C.c_void_p)), "run")
    return time.perf_counter() - t0


print("warm", round(run(), 4))
print("plain", [round(run(), 4) for _ in range(4)])
for v in ("relaxed", "spm", "deferred"):
    with P.Colony(inst, P.AcsParams(variant=v)) as col:
        col.iterate(3)
print("after other contexts", [round(run(), 4) for _ in range(4)])
with P.Colony(inst, P.AcsParams(variant="atomic", rng="philox")) as col:
    for r in range(3):
        t0 = time.perf_counter()
        col.iterate(K)
        print("colony iterate(100) wall", round(time.perf_counter() - t0, 4), "device", col.last_timing())
for r in range(6):
    t0 = time.perf_counter()
    col = P.Colony(inst, P.AcsParams(variant="atomic", rng="philox"))
    t1 = time.perf_counter()
    col.iterate(1)
    t2 = time.perf_counter()
    first = col.last_timing()[0]
    col.iterate(K - 1)
    t3 = time.perf_counter()
    rest = col.last_timing()[0]
    col.close()
    t4 = time.perf_counter()
    print(f"fresh colony {r}: create {t1 - t0:.4f} first-iter {t2 - t1:.4f} (dev {first:.2f} ms) "
          f"rest {t3 - t2:.4f} (dev {rest:.1f} ms) close {t4 - t3:.4f}")
