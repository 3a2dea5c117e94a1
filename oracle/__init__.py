"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU oracle.

* ``Oracle``     -> oracle/liboracle.so, the C restatement (acs_oracle.c)
* ``Reference``  -> oracle/_ref/libacsref.so, the reference's own
  tsp_instance.cpp + rng.hpp compiled from /root/reference (present only where
  the reference was built; absent on a fresh GPU box unless shipped).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import gzip
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
DATA = os.path.join(REPO, "data", "tsplib")

EUC_2D, CEIL_2D, ATT = 0, 1, 2
SEQ, SYNC, RELAXED = 0, 1, 2
DENSE, SELECTIVE = 0, 1
XOSHIRO, PHILOX = 0, 1
_TYPES = {"EUC_2D": EUC_2D, "CEIL_2D": CEIL_2D, "ATT": ATT}

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


@dataclass
class Coords:
    """Plain instance record for the oracle (name, type, xs, ys)."""
    name: str
    type: int
    xs: np.ndarray
    ys: np.ndarray

    @property
    def n(self) -> int:
        return len(self.xs)


def read_tsplib_text(name: str) -> str:
    with gzip.open(os.path.join(DATA, f"{name}.tsp.gz"), "rt") as f:
        return f.read()


def parse_coords(text: str) -> Coords:
    """Minimal TSPLIB95 NODE_COORD reader for the oracle side (test helper)."""
    name, typ, xs, ys, in_coords = "", None, [], [], False
    for raw in text.splitlines():
        s = raw.strip()
        if not s:
            continue
        if s == "EOF":
            break
        if in_coords:
            parts = s.split()
            xs.append(float(parts[1]))
            ys.append(float(parts[2]))
            continue
        key, _, val = s.partition(":")
        key, val = key.strip(), val.strip()
        if key == "NAME":
            name = val
        elif key == "EDGE_WEIGHT_TYPE":
            typ = _TYPES[val]
        elif key.startswith("NODE_COORD_SECTION"):
            in_coords = True
    return Coords(name, typ, np.asarray(xs, np.float64), np.asarray(ys, np.float64))


def load(name: str) -> Coords:
    if name.startswith("rnd") and name[3:].rstrip("k").isdigit():
        return rnd_instance(int(name[3:-1]) * 1000 if name.endswith("k") else int(name[3:]))
    return parse_coords(read_tsplib_text(name))


def rnd_instance(n: int = 10000, seed: int = 20161017) -> Coords:
    """integer coords uniform in [0,1e6)^2 drawn by
    RngStream(seed).uniform_int(1e6), x then y per node."""
    o = Oracle()
    r = o.rng_seed(seed)
    xs = np.empty(n, np.float64)
    ys = np.empty(n, np.float64)
    for i in range(n):
        xs[i] = o.lib.orc_rng_uniform_int(C.byref(r), 1000000)
        ys[i] = o.lib.orc_rng_uniform_int(C.byref(r), 1000000)
    return Coords(f"rnd{n // 1000}k" if n % 1000 == 0 else f"rnd{n}", EUC_2D, xs, ys)


def optima() -> dict:
    out = {}
    with gzip.open(os.path.join(DATA, "optima.txt.gz"), "rt") as f:
        for line in f:
            line = line.split("#", 1)[0].split()
            if len(line) >= 2:
                out[line[0]] = int(line[1])
    return out


class _Rng(C.Structure):
    _fields_ = [("kind", C.c_int32), ("key", C.c_uint32 * 2), ("ctr_hi", C.c_uint32 * 3),
                ("draw", C.c_uint32), ("s", C.c_uint64 * 4)]


class OrcParams(C.Structure):
    _fields_ = [("beta", C.c_double), ("alpha", C.c_double), ("rho", C.c_double), ("q0", C.c_double),
                ("cl", C.c_uint32), ("m", C.c_uint32), ("s", C.c_uint32), ("k", C.c_uint32),
                ("iterations", C.c_uint64), ("seed", C.c_uint64),
                ("mode", C.c_int32), ("memory", C.c_int32), ("consistent", C.c_int32),
                ("rng", C.c_int32), ("threads", C.c_int32)]


class OrcReport(C.Structure):
    _fields_ = [("best_len", C.c_int64), ("best_tour", C.c_void_p), ("trace", C.c_void_p),
                ("iter_best_len", C.c_void_p), ("iter_best_ant", C.c_void_p),
                ("routes", C.c_void_p), ("lengths", C.c_void_p), ("tau", C.c_void_p),
                ("spm_ids", C.c_void_p), ("spm_vals", C.c_void_p), ("spm_tail", C.c_void_p),
                ("local_updates", C.c_uint64), ("hits", C.c_uint64), ("misses", C.c_uint64),
                ("fallback_steps", C.c_uint64), ("greedy_steps", C.c_uint64),
                ("roulette_steps", C.c_uint64), ("tau0", C.c_double), ("nn_len", C.c_int64),
                ("elapsed_ms", C.c_double), ("loop_ms", C.c_double), ("iter_ms", C.c_void_p)]


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class Oracle:
    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            path = os.path.join(HERE, "liboracle.so")
            if not os.path.exists(path):
                build()
            lib = C.CDLL(path)
            lib.orc_distance.restype = C.c_int32
            lib.orc_distance.argtypes = [C.c_int, _f64p, _f64p, C.c_uint32, C.c_uint32]
            lib.orc_distance_table.argtypes = [C.c_uint32, C.c_int, _f64p, _f64p, _i32p]
            lib.orc_build_candidates.restype = C.c_uint32
            lib.orc_build_candidates.argtypes = [C.c_uint32, C.c_int, _f64p, _f64p, C.c_uint32, _u32p]
            lib.orc_nn_tour_length.restype = C.c_int64
            lib.orc_nn_tour_length.argtypes = [C.c_uint32, C.c_int, _f64p, _f64p, C.c_uint32]
            lib.orc_tour_length.restype = C.c_int64
            lib.orc_tour_length.argtypes = [C.c_int, _f64p, _f64p, _u32p, C.c_uint32]
            lib.orc_rng_seed.argtypes = [C.POINTER(_Rng), C.c_uint64]
            lib.orc_rng_derive.argtypes = [C.POINTER(_Rng), C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]
            lib.orc_rng_next_u64.restype = C.c_uint64
            lib.orc_rng_next_u64.argtypes = [C.POINTER(_Rng)]
            lib.orc_rng_uniform01.restype = C.c_double
            lib.orc_rng_uniform01.argtypes = [C.POINTER(_Rng)]
            lib.orc_rng_uniform_int.restype = C.c_uint64
            lib.orc_rng_uniform_int.argtypes = [C.POINTER(_Rng), C.c_uint64]
            for fn in ("orc_default_q0",):
                getattr(lib, fn).restype = C.c_double
                getattr(lib, fn).argtypes = [C.c_uint32]
            lib.orc_tau0.restype = C.c_double
            lib.orc_tau0.argtypes = [C.c_uint32, C.c_int64]
            lib.orc_local_update_value.restype = C.c_double
            lib.orc_local_update_value.argtypes = [C.c_double, C.c_double, C.c_double]
            lib.orc_global_update_value.restype = C.c_double
            lib.orc_global_update_value.argtypes = [C.c_double, C.c_double, C.c_int64]
            lib.orc_eta_beta.restype = C.c_double
            lib.orc_eta_beta.argtypes = [C.c_int32, C.c_double]
            lib.orc_score.restype = C.c_double
            lib.orc_score.argtypes = [C.c_double, C.c_double, C.c_double]
            lib.orc_greedy_pick.restype = C.c_uint32
            lib.orc_greedy_pick.argtypes = [_f64p, C.c_uint32]
            lib.orc_roulette_pick.restype = C.c_uint32
            lib.orc_roulette_pick.argtypes = [_f64p, C.c_uint32, C.c_double]
            lib.orc_select_best.restype = C.c_uint32
            lib.orc_select_best.argtypes = [_i64p, C.c_uint32]
            lib.orc_spm_new.restype = C.c_void_p
            lib.orc_spm_new.argtypes = [C.c_uint32, C.c_uint32, C.c_double]
            lib.orc_spm_free.argtypes = [C.c_void_p]
            lib.orc_spm_read.restype = C.c_double
            lib.orc_spm_read.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
            lib.orc_spm_update_record.restype = C.c_int
            lib.orc_spm_update_record.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.c_double]
            lib.orc_spm_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
            lib.orc_spm_counts.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
            lib.orc_run.restype = C.c_int
            lib.orc_run.argtypes = [C.c_uint32, C.c_int, _f64p, _f64p, C.POINTER(OrcParams), C.POINTER(OrcReport)]
            Oracle._lib = lib
        self.lib = Oracle._lib

    # ---- instance ----
    def distance(self, I: Coords, u: int, v: int) -> int:
        return self.lib.orc_distance(I.type, I.xs, I.ys, u, v)

    def distance_table(self, I: Coords) -> np.ndarray:
        out = np.empty(I.n * I.n, np.int32)
        self.lib.orc_distance_table(I.n, I.type, I.xs, I.ys, out)
        return out.reshape(I.n, I.n)

    def candidates(self, I: Coords, cl: int) -> np.ndarray:
        L = min(cl, I.n - 1)
        out = np.empty(I.n * L, np.uint32)
        self.lib.orc_build_candidates(I.n, I.type, I.xs, I.ys, cl, out)
        return out.reshape(I.n, L)

    def nn_tour_length(self, I: Coords, start: int = 0) -> int:
        return self.lib.orc_nn_tour_length(I.n, I.type, I.xs, I.ys, start)

    def tour_length(self, I: Coords, order) -> int:
        order = np.ascontiguousarray(order, np.uint32)
        return self.lib.orc_tour_length(I.type, I.xs, I.ys, order, len(order))

    # ---- rng ----
    def rng_seed(self, seed: int) -> _Rng:
        r = _Rng()
        self.lib.orc_rng_seed(C.byref(r), seed)
        return r

    def rng_derive(self, seed: int, it: int, ant: int, kind: int = XOSHIRO) -> _Rng:
        r = _Rng()
        self.lib.orc_rng_derive(C.byref(r), kind, seed, it, ant)
        return r

    # ---- engine ----
    def run(self, I: Coords, *, m=None, iterations=10, seed=0, mode=SEQ, memory=DENSE,
            consistent=0, rng=XOSHIRO, threads=1, beta=3.0, alpha=0.2, rho=0.01, q0=-1.0,
            cl=32, s=8, k=1, want_tau=False, want_routes=True, want_spm=False) -> dict:
        n = I.n
        m = n if m is None else m
        p = OrcParams(beta, alpha, rho, q0, cl, m, s, k, iterations, seed, mode, memory,
                      consistent, rng, threads)
        out = dict(best_tour=np.zeros(n, np.uint32), trace=np.zeros(iterations, np.int64),
                   iter_best_len=np.zeros(iterations, np.int64),
                   iter_best_ant=np.zeros(iterations, np.uint32),
                   iter_ms=np.zeros(iterations, np.float64))
        if want_routes:
            out["routes"] = np.zeros((m, n), np.uint32)
            out["lengths"] = np.zeros(m, np.int64)
        if want_tau and memory == DENSE:
            out["tau"] = np.zeros((n, n), np.float64)
        if want_spm and memory == SELECTIVE:
            out["spm_ids"] = np.zeros((n, s), np.uint32)
            out["spm_vals"] = np.zeros((n, s), np.float64)
            out["spm_tail"] = np.zeros(n, np.uint32)
        rep = OrcReport()
        for key in ("best_tour", "trace", "iter_best_len", "iter_best_ant", "routes", "lengths",
                    "tau", "spm_ids", "spm_vals", "spm_tail", "iter_ms"):
            setattr(rep, key, _ptr(out.get(key)))
        rc = self.lib.orc_run(n, I.type, I.xs, I.ys, C.byref(p), C.byref(rep))
        if rc != 0:
            raise ValueError(f"orc_run rejected the parameters (rc={rc})")
        for key in ("best_len", "local_updates", "hits", "misses", "fallback_steps",
                    "greedy_steps", "roulette_steps", "tau0", "nn_len", "elapsed_ms", "loop_ms"):
            out[key] = getattr(rep, key)
        return out


class Reference:
    """The reference's own instance/RNG code (oracle/_ref/libacsref.so)."""
    _lib = None
    PATH = os.path.join(HERE, "_ref", "libacsref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self):
        if Reference._lib is None:
            lib = C.CDLL(self.PATH)
            lib.ref_parse.restype = C.c_void_p
            lib.ref_parse.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
            lib.ref_make.restype = C.c_void_p
            lib.ref_make.argtypes = [C.c_char_p, C.c_int, _f64p, _f64p, C.c_uint32, C.c_char_p, C.c_size_t]
            lib.ref_free.argtypes = [C.c_void_p]
            lib.ref_n.restype = C.c_uint32
            lib.ref_n.argtypes = [C.c_void_p]
            lib.ref_type.restype = C.c_int
            lib.ref_type.argtypes = [C.c_void_p]
            lib.ref_name.restype = C.c_size_t
            lib.ref_name.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
            lib.ref_coords.argtypes = [C.c_void_p, _f64p, _f64p]
            lib.ref_distance.restype = C.c_int32
            lib.ref_distance.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
            lib.ref_distance_table.argtypes = [C.c_void_p, _i32p]
            lib.ref_build_candidates.restype = C.c_uint32
            lib.ref_build_candidates.argtypes = [C.c_void_p, C.c_uint32, _u32p]
            lib.ref_nn_tour_length.restype = C.c_int64
            lib.ref_nn_tour_length.argtypes = [C.c_void_p, C.c_uint32]
            lib.ref_tour_length.restype = C.c_int64
            lib.ref_tour_length.argtypes = [C.c_void_p, _u32p, C.c_uint32]
            lib.ref_serialize.restype = C.c_size_t
            lib.ref_serialize.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
            lib.ref_catalog.restype = C.c_int
            lib.ref_catalog.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, _i64p, C.c_int]
            lib.ref_rng_script.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                           np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                           np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS"),
                                           np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS"), C.c_int]
            Reference._lib = lib
        self.lib = Reference._lib

    def parse(self, text: str):
        err = C.create_string_buffer(512)
        h = self.lib.ref_parse(text.encode(), err, 512)
        if not h:
            return None, err.value.decode()
        return RefInstance(self.lib, h), None

    def make(self, I: Coords):
        err = C.create_string_buffer(512)
        h = self.lib.ref_make(I.name.encode(), I.type, I.xs, I.ys, I.n, err, 512)
        if not h:
            raise ValueError(err.value.decode())
        return RefInstance(self.lib, h)

    def rng_script(self, seed, it, ant, derive, ops, args=None) -> np.ndarray:
        ops = np.asarray(ops, np.int32)
        args = np.zeros(len(ops), np.uint64) if args is None else np.asarray(args, np.uint64)
        out = np.zeros(len(ops), np.uint64)
        self.lib.ref_rng_script(seed, it, ant, int(derive), ops, args, out, len(ops))
        return out

    def catalog(self, text: str) -> dict:
        names = C.create_string_buffer(1 << 16)
        vals = np.zeros(4096, np.int64)
        k = self.lib.ref_catalog(text.encode(), names, 1 << 16, vals, 4096)
        keys = names.value.decode().split("\n")[:k]
        return dict(zip(keys, vals[:k].tolist()))


class RefInstance:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.ref_free(self.h)
        except Exception:
            pass

    @property
    def n(self):
        return self.lib.ref_n(self.h)

    @property
    def type(self):
        return self.lib.ref_type(self.h)

    @property
    def name(self):
        buf = C.create_string_buffer(4096)
        self.lib.ref_name(self.h, buf, 4096)
        return buf.value.decode()

    def coords(self):
        xs = np.empty(self.n, np.float64)
        ys = np.empty(self.n, np.float64)
        self.lib.ref_coords(self.h, xs, ys)
        return xs, ys

    def distance(self, u, v):
        return self.lib.ref_distance(self.h, u, v)

    def distance_table(self):
        out = np.empty(self.n * self.n, np.int32)
        self.lib.ref_distance_table(self.h, out)
        return out.reshape(self.n, self.n)

    def candidates(self, cl):
        L = min(cl, self.n - 1)
        out = np.empty(self.n * L, np.uint32)
        self.lib.ref_build_candidates(self.h, cl, out)
        return out.reshape(self.n, L)

    def nn_tour_length(self, start=0):
        return self.lib.ref_nn_tour_length(self.h, start)

    def tour_length(self, order):
        order = np.ascontiguousarray(order, np.uint32)
        return self.lib.ref_tour_length(self.h, order, len(order))

    def serialize(self) -> str:
        k = self.lib.ref_serialize(self.h, None, 0)
        buf = C.create_string_buffer(k + 1)
        self.lib.ref_serialize(self.h, buf, k + 1)
        return buf.value.decode()


def fnv1a64(arr: np.ndarray) -> str:
    """FNV-1a-64 over little-endian bytes."""
    lib = Oracle().lib
    lib.orc_fnv1a64.restype = C.c_uint64
    lib.orc_fnv1a64.argtypes = [C.c_void_p, C.c_uint64]
    a = np.ascontiguousarray(arr)
    return f"{lib.orc_fnv1a64(a.ctypes.data_as(C.c_void_p), a.nbytes):016x}"
