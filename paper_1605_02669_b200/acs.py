"""Python mirror of the drop-in ACS interface (include/acs/*.hpp).

Names follow the reference (tsp_instance.hpp:14-96):
``TspInstance``, ``parse_tsplib``, ``load_tsplib_file``, ``build_candidates``,
``nn_tour_length``, ``AcsParams``, ``run`` -> ``RunReport``.  Every compute
call goes through the C-ABI into the sm_100a kernels; nothing here computes
a tour, a candidate list or a pheromone value on the CPU.
"""
from __future__ import annotations

import ctypes as C
import gzip
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N
from ._native import AcsError, ParseError  # noqa: F401  (re-export)

_TYPE_NAMES = {N.EUC_2D: "EUC_2D", N.CEIL_2D: "CEIL_2D", N.ATT: "ATT"}


def _f64(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class TspInstance:
    """Immutable symmetric TSP instance (reference TspInstance, hpp:30-59)."""
    name: str
    edge_weight_type: int
    xs: np.ndarray
    ys: np.ndarray
    optimum: Optional[int] = None

    def __post_init__(self):
        self.xs = np.ascontiguousarray(self.xs, np.float64)
        self.ys = np.ascontiguousarray(self.ys, np.float64)
        if len(self.xs) < 3:
            raise ParseError(f"instance needs at least 3 nodes, got {len(self.xs)}")
        if len(self.xs) != len(self.ys):
            raise ParseError("coordinate arrays differ in length")

    @property
    def dimension(self) -> int:
        return len(self.xs)

    n = dimension

    def desc(self) -> N.InstanceDesc:
        return N.InstanceDesc(self.dimension, self.edge_weight_type, _f64(self.xs), _f64(self.ys))

    def distance_table(self, device: int = 0) -> np.ndarray:
        out = np.empty((self.n, self.n), np.int32)
        d = self.desc()
        N.check(N.lib().acs_gpu_distance_table(C.byref(d), device, _ptr(out)), "distance_table")
        return out

    def tour_lengths(self, routes: np.ndarray, device: int = 0) -> np.ndarray:
        routes = np.ascontiguousarray(routes, np.uint32).reshape(-1, self.n)
        out = np.empty(routes.shape[0], np.int64)
        d = self.desc()
        N.check(N.lib().acs_gpu_tour_lengths(C.byref(d), _ptr(routes), routes.shape[0], device,
                                            _ptr(out)), "tour_lengths")
        return out

    def tour_length(self, order, device: int = 0) -> int:
        return int(self.tour_lengths(np.asarray(order, np.uint32)[None, :], device)[0])


def parse_tsplib(text: str) -> TspInstance:
    raw = text.encode()
    lib = N.lib()
    n, typ = C.c_uint32(0), C.c_uint32(0)
    name = C.create_string_buffer(1024)
    N.check(lib.acs_parse_tsplib(raw, len(raw), C.byref(n), C.byref(typ), None, None, 0, name, 1024),
            "parse_tsplib")
    xs = np.empty(n.value, np.float64)
    ys = np.empty(n.value, np.float64)
    N.check(lib.acs_parse_tsplib(raw, len(raw), C.byref(n), C.byref(typ), _ptr(xs), _ptr(ys),
                                 n.value, None, 0), "parse_tsplib")
    return TspInstance(name.value.decode(), typ.value, xs, ys)


def load_tsplib_file(path: str) -> TspInstance:
    opener = gzip.open if path.endswith(".gz") else open
    try:
        with opener(path, "rt") as f:
            text = f.read()
    except OSError:
        raise ParseError(f"cannot open instance file: {path}") from None
    return parse_tsplib(text)


# instance files shipped with the repo (gzipped TSPLIB + the optimum catalog)
DATA_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "tsplib")


def load_optimum_catalog_file(path: str) -> dict:
    """name -> optimal length (reference load_optimum_catalog_file, cpp:282-305)."""
    opener = gzip.open if path.endswith(".gz") else open
    out = {}
    try:
        with opener(path, "rt") as f:
            for line in f:
                fields = line.split("#", 1)[0].split()
                if len(fields) >= 2:
                    out[fields[0]] = int(fields[1])
    except OSError:
        raise RuntimeError(f"cannot open optimum catalog: {path}") from None
    return out


def optima() -> dict:
    return load_optimum_catalog_file(os.path.join(DATA_DIR, "optima.txt.gz"))


def random_uniform_instance(n: int, seed: int = 20161017, side: int = 1000000) -> TspInstance:
    """integer coordinates uniform in [0, side)^2 from the
    reference RngStream(seed).uniform_int(side), x then y per node."""
    xs = np.empty(n, np.float64)
    ys = np.empty(n, np.float64)
    N.check(N.lib().acs_random_instance(n, seed, side, _ptr(xs), _ptr(ys)), "random_instance")
    name = f"rnd{n // 1000}k" if n % 1000 == 0 else f"rnd{n}"
    return TspInstance(name, N.EUC_2D, xs, ys)


def load_instance(name: str) -> TspInstance:
    """A shipped TSPLIB instance by name (data/tsplib/<name>.tsp.gz), or a
    synthetic ``rnd<k>k`` / ``rnd<n>`` instance; the optimum is attached when
    the catalog has it."""
    if name.startswith("rnd") and name[3:].rstrip("k").isdigit():
        n = int(name[3:-1]) * 1000 if name.endswith("k") else int(name[3:])
        return random_uniform_instance(n)
    inst = load_tsplib_file(os.path.join(DATA_DIR, f"{name}.tsp.gz"))
    inst.optimum = optima().get(inst.name)
    return inst


@dataclass
class CandidateLists:
    cl: int
    list_len: int
    n: int
    flat: np.ndarray  # n * list_len uint32, row-major (reference flat_)

    def of(self, node: int) -> np.ndarray:
        return self.flat[node * self.list_len:(node + 1) * self.list_len]


def build_candidates(inst: TspInstance, cl: int, device: int = 0) -> CandidateLists:
    d = inst.desc()
    L = C.c_uint32(0)
    N.check(N.lib().acs_gpu_build_candidates(C.byref(d), cl, device, None, C.byref(L)), "build_candidates")
    flat = np.empty(inst.n * L.value, np.uint32)
    N.check(N.lib().acs_gpu_build_candidates(C.byref(d), cl, device, _ptr(flat), C.byref(L)),
            "build_candidates")
    return CandidateLists(cl, L.value, inst.n, flat)


def nn_tour_length(inst: TspInstance, start: int = 0, device: int = 0) -> int:
    d = inst.desc()
    out = C.c_int64(0)
    N.check(N.lib().acs_gpu_nn_tour_length(C.byref(d), start, device, C.byref(out)), "nn_tour_length")
    return out.value


def rank_sum_test(xs, ys) -> float:
    """Two-sided Wilcoxon rank-sum p-value (SPEC stats.rank_sum_test)."""
    a = np.ascontiguousarray(xs, np.float64)
    b = np.ascontiguousarray(ys, np.float64)
    p = C.c_double(0.0)
    N.check(N.lib().acs_rank_sum_test(_ptr(a), len(a), _ptr(b), len(b), C.byref(p)), "rank_sum_test")
    return p.value


def relative_error(length: int, optimum: int) -> float:
    """SPEC stats.relative_error."""
    if optimum <= 0:
        raise ValueError("relative_error: optimum must be > 0")
    return 100.0 * (length - optimum) / optimum


def default_q0(n: int) -> float:
    return 0.0 if n <= 20 else (n - 20) / n


@dataclass
class AcsParams:
    """SPEC AcsParams. alpha = GLOBAL, rho = LOCAL evaporation."""
    beta: float = 3.0
    alpha: float = 0.2
    rho: float = 0.01
    q0: float = -1.0
    cl: int = 32
    m: int = 0
    s: int = 8
    k: int = 1
    iterations: int = 1000
    budget: int = 0
    time_limit_s: float = 0.0
    variant: str = "atomic"
    rng: str = "xoshiro"
    seed: int = 0

    def to_c(self, n: int) -> N.Params:
        if self.variant not in N.VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}; one of {sorted(N.VARIANTS)}")
        return N.Params(self.beta, self.alpha, self.rho, self.q0, self.cl, self.m or n, self.s,
                        self.k, N.VARIANTS[self.variant],
                        N.RNG_PHILOX if self.rng == "philox" else N.RNG_XOSHIRO,
                        self.seed & 0xFFFFFFFFFFFFFFFF)


class Colony:
    """One ACS colony resident on one GPU (acs_gpu_ctx)."""

    def __init__(self, inst: TspInstance, params: AcsParams, device: int = 0):
        self.inst, self.params, self.device = inst, params, device
        self._lib = N.lib()
        self._h = C.c_void_p()
        d = inst.desc()
        p = params.to_c(inst.n)
        N.check(self._lib.acs_gpu_create(C.byref(d), C.byref(p), device, C.byref(self._h)), "acs_gpu_create")
        info = N.CtxInfo()
        N.check(self._lib.acs_gpu_info(self._h, C.byref(info)), "acs_gpu_info")
        self.info = info
        self.m = info.ants

    def close(self):
        if self._h:
            self._lib.acs_gpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def iterate(self, n_iter: int = 1) -> np.ndarray:
        st = (N.IterStats * n_iter)()
        N.check(self._lib.acs_gpu_iterate(self._h, n_iter, st), "acs_gpu_iterate")
        return np.array([(s.iter_best_len, s.iter_best_ant, s.improved, s.global_best_len) for s in st],
                        dtype=[("iter_best_len", "i8"), ("iter_best_ant", "u4"), ("improved", "u4"),
                               ("global_best_len", "i8")])

    def last_timing(self):
        t, c = C.c_float(), C.c_float()
        N.check(self._lib.acs_gpu_last_timing(self._h, C.byref(t), C.byref(c)), "last_timing")
        return t.value, c.value

    def best(self):
        order = np.empty(self.inst.n, np.uint32)
        ln = C.c_int64()
        N.check(self._lib.acs_gpu_get_best(self._h, _ptr(order), C.byref(ln)), "get_best")
        return order, ln.value

    def set_best(self, order, length: int):
        order = np.ascontiguousarray(order, np.uint32)
        N.check(self._lib.acs_gpu_set_best(self._h, _ptr(order), int(length)), "set_best")

    def routes(self):
        r = np.empty((self.m, self.inst.n), np.uint32)
        ln = np.empty(self.m, np.int64)
        N.check(self._lib.acs_gpu_get_routes(self._h, _ptr(r), _ptr(ln)), "get_routes")
        return r, ln

    def pheromone(self) -> np.ndarray:
        t = np.empty((self.inst.n, self.inst.n), np.float64)
        N.check(self._lib.acs_gpu_get_pheromone(self._h, _ptr(t)), "get_pheromone")
        return t

    def selective(self):
        S = self.info.slots
        ids = np.empty((self.inst.n, S), np.uint32)
        vals = np.empty((self.inst.n, S), np.float64)
        tail = np.empty(self.inst.n, np.uint32)
        N.check(self._lib.acs_gpu_get_selective(self._h, _ptr(ids), _ptr(vals), _ptr(tail)), "get_selective")
        return ids, vals, tail

    def candidates(self) -> np.ndarray:
        out = np.empty((self.inst.n, self.info.list_len), np.uint32)
        N.check(self._lib.acs_gpu_get_candidates(self._h, _ptr(out)), "get_candidates")
        return out

    def counters(self) -> dict:
        c = N.Counters()
        N.check(self._lib.acs_gpu_get_counters(self._h, C.byref(c)), "get_counters")
        return {k: getattr(c, k) for k, _ in N.Counters._fields_}

    # ---- island model ----
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        N.check(N.lib().acs_gpu_nccl_unique_id(buf), "nccl_unique_id")
        return buf.raw

    def island_init(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(uid, 128)
        N.check(self._lib.acs_gpu_island_init(self._h, buf, nranks, rank), "island_init")

    def island_exchange(self) -> int:
        out = C.c_int64()
        N.check(self._lib.acs_gpu_island_exchange(self._h, C.byref(out)), "island_exchange")
        return out.value

    @staticmethod
    def island_exchange_local(colonies) -> int:
        """Device-side exchange among colonies of this process on one GPU
        (colonies[i] plays rank i); returns the global best length."""
        arr = (C.c_void_p * len(colonies))(*[c._h.value for c in colonies])
        out = C.c_int64()
        N.check(N.lib().acs_gpu_island_exchange_local(arr, len(colonies), C.byref(out)),
                "island_exchange_local")
        return out.value


@dataclass
class RunReport:
    best_tour: np.ndarray
    best_length: int
    trace: np.ndarray
    trace_ms: list = field(default_factory=list)
    error_pct: Optional[float] = None
    total_ms: float = 0.0
    setup_ms: float = 0.0
    construct_ms_per_iter: float = 0.0
    iterations: int = 0
    solutions: int = 0
    counters: dict = field(default_factory=dict)
    params: Optional[AcsParams] = None

    def hit_ratio(self) -> float:
        h, m = self.counters.get("hits", 0), self.counters.get("misses", 0)
        if h + m == 0:
            raise ValueError("hit_ratio: no selective-memory update yet")
        return h / (h + m)


def run(inst: TspInstance, params: AcsParams, device: int = 0) -> RunReport:
    """SPEC run(inst, params) on the GPU; iteration / budget / time-limit forms."""
    t0 = time.perf_counter()
    with Colony(inst, params, device) as col:
        setup_ms = (time.perf_counter() - t0) * 1e3
        m = col.m
        iters = params.iterations
        if params.budget:
            if params.budget % m:
                raise ValueError("budget must be a multiple of the ant count")
            iters = params.budget // m
        trace, trace_ms, construct, done, chunk = [], [], 0.0, 0, 1
        last = (time.perf_counter() - t0) * 1e3
        while True:
            if params.time_limit_s > 0:
                if time.perf_counter() - t0 >= params.time_limit_s:
                    break
            else:
                if done >= iters:
                    break
                chunk = min(iters - done, 256)
            st = col.iterate(chunk)
            construct += col.last_timing()[1]
            trace.extend(st["global_best_len"].tolist())
            now = (time.perf_counter() - t0) * 1e3
            # per-iteration timestamps, interpolated inside a chunk
            trace_ms.extend(last + (now - last) * (i + 1) / chunk for i in range(chunk))
            if params.time_limit_s > 0:  # ~2 ms chunks: bounded overshoot, fine-grained trace
                chunk = int(min(64, max(1, 2.0 * chunk / max(now - last, 1e-3))))
            last = now
            done += len(st)
        order, length = col.best()
        rep = RunReport(order, length, np.asarray(trace, np.int64), trace_ms,
                        None if inst.optimum is None else 100.0 * (length - inst.optimum) / inst.optimum,
                        (time.perf_counter() - t0) * 1e3, setup_ms, construct / max(done, 1), done,
                        done * m, col.counters(), params)
    return rep
