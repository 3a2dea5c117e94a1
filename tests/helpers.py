"""Shared test helpers: instance conversion and oracle/GPU run pairs."""
import numpy as np

import oracle as O

TSPLIB = ["d198", "a280", "lin318", "pcb442", "att532", "rat783", "pr1002", "nrw1379", "pr2392"]

# SURVEY.md Appendix A, derived from the reference code (oracle/_ref) in this container
GOLDEN = {
    "d198": ("93787ab4725dbb01", "e08eb934a84b5227", 18240, 15780),
    "a280": ("7e8353c7f8fbe739", "ddaa130e683f8d23", 3157, 2579),
    "lin318": ("37dfb037dd3cd13d", "1c77b5789a791f2c", 54019, 42029),
    "pcb442": ("4c8c6f33dff81399", "43b5b6382839384e", 61979, 50778),
    "att532": ("ff63d766baf24b91", "c904b1fd112b483b", 35516, 27686),
    "rat783": ("6784d67407d6716d", "c37672e7df126e18", 11054, 8806),
    "pr1002": ("7169b51a7396590d", "4eb87cfe91c802c6", 331103, 259045),
    "nrw1379": ("f46eaf004ac372a5", "f95f007082dfb244", 68964, 56638),
    "pr2392": ("d059616565df4691", "ab4aeae1875974a6", 461170, 378032),
}
RND10K_CAND_FNV = "f1dbcc2e562e90b0"
RND10K_NN = 88691968


def to_acs(acs, I: O.Coords):
    return acs.TspInstance(I.name, I.type, I.xs.copy(), I.ys.copy())


def small_instance(n: int, seed: int = 1, scale: int = 1000, typ: int = O.EUC_2D) -> O.Coords:
    rng = np.random.default_rng(seed)
    xs = rng.integers(0, scale, n).astype(np.float64)
    ys = rng.integers(0, scale, n).astype(np.float64)
    return O.Coords(f"rnd{n}_{seed}", typ, xs, ys)


def assert_permutations(routes: np.ndarray, n: int):
    s = np.sort(routes, axis=1)
    assert (s == np.arange(n, dtype=s.dtype)[None, :]).all(), "a route is not a permutation"
