import sys, time, ctypes as C, numpy as np
sys.path.insert(0, '.')
import paper_1605_02669_b200 as P
from paper_1605_02669_b200 import _native as N
inst = P.load_instance('pr2392')
for K in (20, 20, 100, 1):
    p = P.AcsParams(variant='atomic', rng='philox').to_c(inst.n)
    d = inst.desc(); order = np.empty(inst.n, np.uint32); trace = np.empty(K, np.int64); bl = C.c_int64()
    t0 = time.perf_counter()
    N.check(N.lib().acs_gpu_run(C.byref(d), C.byref(p), K, 0, order.ctypes.data_as(C.c_void_p), C.byref(bl), trace.ctypes.data_as(C.c_void_p)), 'run')
    print(K, round(time.perf_counter() - t0, 4))
t0 = time.perf_counter(); col = P.Colony(inst, P.AcsParams(variant='atomic', rng='philox')); print('create', round(time.perf_counter()-t0,4))
t0 = time.perf_counter(); col.iterate(1); print('iter1', round(time.perf_counter()-t0,4))
t0 = time.perf_counter(); col.close(); print('destroy', round(time.perf_counter()-t0,4))
