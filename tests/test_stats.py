"""SPEC stats module behind the C-ABI: relative_error KATs,
rank_sum_test KATs and properties, checked against scipy's Mann-Whitney U
(exact for small untied samples, asymptotic with tie + continuity correction
otherwise).  Host-only code: runs on the CPU."""
import numpy as np
import pytest
from scipy import stats as st


def test_relative_error_kats(acs):
    assert acs.relative_error(2579, 2579) == 0.0
    assert round(acs.relative_error(144529, 137694), 2) == 4.96
    assert acs.relative_error(102, 100) == pytest.approx(2.0)
    with pytest.raises(ValueError):
        acs.relative_error(10, 0)


def test_rank_sum_kats(acs):
    assert acs.rank_sum_test([1, 2, 3], [4, 5, 6]) == pytest.approx(0.1)
    assert acs.rank_sum_test([5, 6, 7, 8], [5, 6, 7, 8]) == 1.0
    assert acs.rank_sum_test([3, 3, 3], [3, 3, 3, 3]) == 1.0  # degenerate pooled sample
    with pytest.raises(Exception):
        acs.rank_sum_test([1, 2], [3, 4, 5])


def test_rank_sum_properties(acs):
    rng = np.random.default_rng(7)
    for _ in range(40):
        a = rng.integers(0, 20, rng.integers(3, 15)).astype(float)
        b = rng.integers(0, 20, rng.integers(3, 15)).astype(float)
        p = acs.rank_sum_test(a, b)
        assert 0 < p <= 1
        assert p == pytest.approx(acs.rank_sum_test(b, a), abs=1e-12)  # symmetry
        assert p == pytest.approx(acs.rank_sum_test(a + 17.5, b + 17.5), abs=1e-12)  # rank invariance


def test_rank_sum_exact_matches_scipy(acs):
    rng = np.random.default_rng(11)
    for _ in range(30):
        n1, n2 = rng.integers(3, 7), rng.integers(3, 7)
        if n1 + n2 > 12:
            continue
        v = rng.permutation(100)[: n1 + n2].astype(float)  # untied
        a, b = v[:n1], v[n1:]
        ref = st.mannwhitneyu(a, b, alternative="two-sided", method="exact").pvalue
        assert acs.rank_sum_test(a, b) == pytest.approx(ref, rel=1e-9)


def test_rank_sum_asymptotic_matches_scipy(acs):
    rng = np.random.default_rng(5)
    for _ in range(30):
        a = rng.integers(0, 12, rng.integers(7, 31)).astype(float)  # ties
        b = rng.integers(2, 14, rng.integers(7, 31)).astype(float)
        ref = st.mannwhitneyu(a, b, alternative="two-sided", method="asymptotic", use_continuity=True).pvalue
        assert acs.rank_sum_test(a, b) == pytest.approx(min(1.0, ref), rel=1e-9, abs=1e-12)


def test_rank_sum_approx_close_to_exact_8v8(acs):
    """random 8-vs-8 samples, approximation within 0.02 of exact."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        v = rng.permutation(1000)[:16].astype(float)
        exact = st.mannwhitneyu(v[:8], v[8:], alternative="two-sided", method="exact").pvalue
        assert abs(acs.rank_sum_test(v[:8], v[8:]) - exact) < 0.02
