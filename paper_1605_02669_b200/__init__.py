"""B200-native Ant Colony System hot path (arXiv 1605.02669).

The product is ``libacs_b200.so`` (sm_100a kernels + C-ABI + C++ drop-in API,
sources in ``csrc/``, headers in ``include/``).  This package is the Python
caller of that C-ABI; see ``acs.py`` for the reference-named interface.
"""
from .acs import (AcsError, AcsParams, CandidateLists, Colony, ParseError, RunReport,  # noqa: F401
                  TspInstance, build_candidates, default_q0, load_instance, load_optimum_catalog_file,
                  load_tsplib_file, nn_tour_length, optima, parse_tsplib, random_uniform_instance, rank_sum_test,
                  relative_error, run)
from ._native import LIB_PATH, device_count, lib  # noqa: F401
from . import island  # noqa: F401
