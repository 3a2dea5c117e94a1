"""ctypes binding of libacs_b200.so (include/acs_gpu.h).

This is the reference-facing boundary as a Python caller sees it: plain
pointers and sizes, integer status codes, thread-local error text.  The
library is built in-tree (``make`` / ``__graft_entry__.build()``); importing
this module without it raises immediately -- there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# ACS_LIB_VARIANT=<suffix> selects an in-tree A/B build libacs_b200_<suffix>.so
# (kernel experiments); the default is the product library.
_suffix = os.environ.get("ACS_LIB_VARIANT", "")
LIB_PATH = os.path.join(HERE, f"libacs_b200_{_suffix}.so" if _suffix else "libacs_b200.so")

ACS_OK, ACS_E_ARG, ACS_E_CUDA, ACS_E_NOMEM, ACS_E_NCCL, ACS_E_PARSE = 0, -1, -2, -3, -4, -5
EUC_2D, CEIL_2D, ATT = 0, 1, 2
VARIANT_ATOMIC, VARIANT_DEFERRED, VARIANT_RELAXED, VARIANT_SPM, VARIANT_SEQ, VARIANT_SPM_SEQ, VARIANT_SPM_SYNC = range(7)
RNG_XOSHIRO, RNG_PHILOX = 0, 1

VARIANTS = {"atomic": VARIANT_ATOMIC, "deferred": VARIANT_DEFERRED, "relaxed": VARIANT_RELAXED,
            "spm": VARIANT_SPM, "seq": VARIANT_SEQ, "spm-seq": VARIANT_SPM_SEQ, "spm-sync": VARIANT_SPM_SYNC}


class InstanceDesc(C.Structure):
    _fields_ = [("n", C.c_uint32), ("edge_weight_type", C.c_uint32),
                ("xs", C.POINTER(C.c_double)), ("ys", C.POINTER(C.c_double))]


class Params(C.Structure):
    _fields_ = [("beta", C.c_double), ("alpha", C.c_double), ("rho", C.c_double), ("q0", C.c_double),
                ("cl", C.c_uint32), ("ants", C.c_uint32), ("slots", C.c_uint32),
                ("update_period", C.c_uint32), ("variant", C.c_uint32), ("rng", C.c_uint32),
                ("seed", C.c_uint64)]


class IterStats(C.Structure):
    _fields_ = [("iter_best_len", C.c_int64), ("iter_best_ant", C.c_uint32),
                ("improved", C.c_uint32), ("global_best_len", C.c_int64)]


class Counters(C.Structure):
    _fields_ = [("local_updates", C.c_uint64), ("hits", C.c_uint64), ("misses", C.c_uint64),
                ("fallback_steps", C.c_uint64), ("greedy_steps", C.c_uint64),
                ("roulette_steps", C.c_uint64), ("cas_retries", C.c_uint64),
                ("iterations", C.c_uint64), ("fallback_elems", C.c_uint64),
                ("fallback_full", C.c_uint64), ("relaxed_writes", C.c_uint64), ("lost_updates", C.c_uint64),
                ("fallback_grid", C.c_uint64)]


class CtxInfo(C.Structure):
    _fields_ = [("n", C.c_uint32), ("ants", C.c_uint32), ("list_len", C.c_uint32),
                ("slots", C.c_uint32), ("q0", C.c_double), ("tau0", C.c_double),
                ("nn_len", C.c_int64), ("device_bytes", C.c_uint64)]


_P = C.c_void_p
_u32, _u64, _i32, _i64, _f64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double
_desc = C.POINTER(InstanceDesc)

# name -> (restype, argtypes); every symbol declared in include/acs_gpu.h
SIGNATURES = {
    "acs_gpu_last_error": (C.c_char_p, []),
    "acs_gpu_abi_version": (C.c_int, []),
    "acs_gpu_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "acs_parse_tsplib": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(_u32), C.POINTER(_u32), _P, _P,
                                   _u32, C.c_char_p, C.c_size_t]),
    "acs_random_instance": (C.c_int, [_u32, _u64, _u32, _P, _P]),
    "acs_gpu_l2_read_bandwidth": (C.c_int, [C.c_int, _u64, C.POINTER(_f64)]),
    "acs_gpu_l2_latency": (C.c_int, [C.c_int, _u64, C.POINTER(_f64), C.POINTER(_f64)]),
    "acs_rank_sum_test": (C.c_int, [_P, _u32, _P, _u32, C.POINTER(_f64)]),
    "acs_gpu_distance_table": (C.c_int, [_desc, C.c_int, _P]),
    "acs_gpu_build_candidates": (C.c_int, [_desc, _u32, C.c_int, _P, C.POINTER(_u32)]),
    "acs_gpu_nn_tour_length": (C.c_int, [_desc, _u32, C.c_int, C.POINTER(_i64)]),
    "acs_gpu_tour_lengths": (C.c_int, [_desc, _P, _u32, C.c_int, _P]),
    "acs_gpu_rng_script": (C.c_int, [_u32, _u64, _u64, _u64, C.c_int, _P, _P, _P, _u32, C.c_int]),
    "acs_gpu_spm_script": (C.c_int, [_u32, _u32, _f64, _f64, _f64, _f64, _P, _P, _u32, C.c_int, _P, _P,
                                     _P, _P, C.POINTER(_u64), C.POINTER(_u64)]),
    "acs_gpu_create": (C.c_int, [_desc, C.POINTER(Params), C.c_int, C.POINTER(_P)]),
    "acs_gpu_info": (C.c_int, [_P, C.POINTER(CtxInfo)]),
    "acs_gpu_iterate": (C.c_int, [_P, _u32, _P]),
    "acs_gpu_last_timing": (C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "acs_gpu_get_best": (C.c_int, [_P, _P, C.POINTER(_i64)]),
    "acs_gpu_set_best": (C.c_int, [_P, _P, _i64]),
    "acs_gpu_get_routes": (C.c_int, [_P, _P, _P]),
    "acs_gpu_get_pheromone": (C.c_int, [_P, _P]),
    "acs_gpu_get_selective": (C.c_int, [_P, _P, _P, _P]),
    "acs_gpu_get_candidates": (C.c_int, [_P, _P]),
    "acs_gpu_get_counters": (C.c_int, [_P, C.POINTER(Counters)]),
    "acs_gpu_destroy": (None, [_P]),
    "acs_gpu_run": (C.c_int, [_desc, C.POINTER(Params), _u64, C.c_int, _P, C.POINTER(_i64), _P]),
    "acs_gpu_nccl_unique_id": (C.c_int, [_P]),
    "acs_gpu_island_init": (C.c_int, [_P, _P, C.c_int, C.c_int]),
    "acs_gpu_island_exchange": (C.c_int, [_P, C.POINTER(_i64)]),
    "acs_gpu_island_exchange_local": (C.c_int, [_P, C.c_int, C.POINTER(_i64)]),
}


class AcsError(RuntimeError):
    def __init__(self, code: int, where: str, message: str):
        super().__init__(f"{where}: [{code}] {message}")
        self.code = code


class ParseError(ValueError):
    """TSPLIB parse failure naming the offending field (reference ParseError)."""


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(rc: int, where: str) -> None:
    if rc != ACS_OK:
        msg = (lib().acs_gpu_last_error() or b"").decode(errors="replace")
        if rc == ACS_E_PARSE:
            raise ParseError(msg)
        raise AcsError(rc, where, msg)


def l2_read_bandwidth(device: int = 0, nbytes: int = 64 << 20) -> float:
    """Measured L2 read GB/s over an L2-resident buffer (roofline denominator)."""
    g = C.c_double(0.0)
    check(lib().acs_gpu_l2_read_bandwidth(device, nbytes, C.byref(g)), "l2_read_bandwidth")
    return g.value


def l2_latency(device: int = 0, nbytes: int = 48 << 20):
    """(L2 load-to-use ns, minimal selection step ns) -- acs_gpu_l2_latency."""
    a, b = _f64(), _f64()
    check(lib().acs_gpu_l2_latency(device, nbytes, C.byref(a), C.byref(b)), "l2_latency")
    return a.value, b.value


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().acs_gpu_device_count(C.byref(n))
    return n.value if rc == ACS_OK else 0
