"""Pins for the oracle's Ω generator (PAPER.md:163-168 Gaussian test vectors,
PAPER.md:437-440 uniform [-1,1]; counter layout = DESIGN.md reading Q7).

* the Philox4x32-10 integer stream is pinned bit-for-bit to cuRAND's own
  header (a library routine in the image), not to a retyped formula;
* the real-valued transform is pinned statistically: moments and a
  Kolmogorov–Smirnov test against scipy's normal / uniform CDFs.
"""
import numpy as np
import pytest
from scipy import stats

import oracle
from tests.helpers import curand_philox


def test_philox_matches_curand_header():
    rng = np.random.default_rng(7)
    rows = [(0, 0, 0, 0, 0, 0), (0xFFFFFFFF,) * 6, (1, 2, 3, 4, 5, 6)]
    rows += [tuple(int(v) for v in rng.integers(0, 2**32, 6)) for _ in range(200)]
    ref = curand_philox(rows)
    got = np.array([oracle.philox4x32_10(r[:4], r[4:]) for r in rows])
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("seed", [0, 1, 0x123456789ABCDEF])
def test_omega_counter_layout(seed):
    """Element e of Ω draws from Philox call p = e>>1, ctr = (p lo, p hi, 0, stream),
    key = seed halves (Q7): recover the two 53-bit uniforms of each call from the
    cuRAND words and check the uniform-distribution output reproduces them exactly."""
    rows, cols = 7, 5  # odd total: exercises the half-used last call
    U = oracle.omega(seed, rows, cols, dist=oracle.UNIFORM, stream=3)
    flat = U.reshape(-1)
    calls = (flat.size + 1) // 2
    words = curand_philox([(p, 0, 0, 3, seed & 0xFFFFFFFF, seed >> 32) for p in range(calls)])
    for p in range(calls):
        w = [int(x) for x in words[p]]
        a = ((w[0] << 32 | w[1]) >> 11) * 2.0**-53
        b = ((w[2] << 32 | w[3]) >> 11) * 2.0**-53
        assert flat[2 * p] == 2 * a - 1
        if 2 * p + 1 < flat.size:
            assert flat[2 * p + 1] == 2 * b - 1


def test_omega_deterministic_and_streams_differ():
    a = oracle.omega(5, 100, 12)
    b = oracle.omega(5, 100, 12)
    c = oracle.omega(5, 100, 12, stream=1)
    d = oracle.omega(6, 100, 12)
    assert np.array_equal(a, b)
    assert not np.allclose(a, c) and not np.allclose(a, d)


def test_gaussian_moments_and_ks():
    x = oracle.omega(0, 1000, 1000).reshape(-1)  # 1e6 draws
    n = x.size
    assert abs(x.mean()) < 5 / np.sqrt(n)
    assert abs(x.var() - 1) < 5 * np.sqrt(2 / n)
    assert abs(np.mean(x**4) - 3) < 5 * np.sqrt(96 / n)
    assert stats.kstest(x, "norm").pvalue > 1e-4
    # even and odd elements (cos / sin halves) are each standard normal and uncorrelated
    assert stats.kstest(x[0::2], "norm").pvalue > 1e-4
    assert stats.kstest(x[1::2], "norm").pvalue > 1e-4
    assert abs(np.corrcoef(x[0::2], x[1::2])[0, 1]) < 5 / np.sqrt(n / 2)


def test_uniform_range_and_moments():
    u = oracle.omega(3, 1000, 1000, dist=oracle.UNIFORM).reshape(-1)
    assert u.min() >= -1 and u.max() < 1
    assert abs(u.mean()) < 0.01
    assert abs(u.var() - 1 / 3) < 0.02
    assert stats.kstest(u, "uniform", args=(-1, 2)).pvalue > 1e-4
