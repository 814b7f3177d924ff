"""CPU checks of the algebraic identities the Fast-path narrow-phase kernels
rely on to issue fewer instructions than the reference's literal formulas
while staying bit-identical (ccdk_interval.cuh: CCDK_UNIFIED_SU,
CCDK_TWICE_MID).  Widening follows the reference (interval.hpp:36-49): one
ulp outward, |x| < 1e-250 flushed to +/-1e-250.  The GPU parity suite checks
the kernels themselves; these tests pin the arithmetic argument on many
random and adversarial operands."""
import numpy as np
import pytest

FLUSH = 1e-250


def up(x):
    x = np.asarray(x, dtype=np.float64)
    return np.where(np.abs(x) < FLUSH, FLUSH, np.nextafter(x, np.inf))


def dn(x):
    x = np.asarray(x, dtype=np.float64)
    return np.where(np.abs(x) < FLUSH, -FLUSH, np.nextafter(x, -np.inf))


def sub(a, b):  # interval a - b, outward widened
    return dn(a[0] - b[1]), up(a[1] - b[0])


def add(a, b):
    return dn(a[0] + b[0]), up(a[1] + b[1])


def scale(p, a):  # p in [0, 1]
    return dn(p * a[0]), up(p * a[1])


def operands(rng, n):
    """Doubles mixing O(1) values, exact zeros, flush-range tiny values and
    large magnitudes (up to the Fast path's 2^1000 bound / 64)."""
    kinds = rng.integers(0, 5, n)
    x = rng.standard_normal(n)
    x = np.where(kinds == 1, 0.0, x)
    x = np.where(kinds == 2, rng.standard_normal(n) * 1e-251, x)
    x = np.where(kinds == 3, rng.standard_normal(n) * 2.0 ** rng.integers(-900, 990, n), x)
    x = np.where(kinds == 4, rng.standard_normal(n) * 1e-249, x)
    return x


def interval(rng, n):
    a, b = operands(rng, n), operands(rng, n)
    return dn(np.minimum(a, b)), up(np.maximum(a, b))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_unified_u_term_equals_reference_add(seed):
    """EE: base + u*(p1 - p0) == base - u*(p0 - p1) bound for bound."""
    rng = np.random.default_rng(seed)
    n = 200_000
    at0, at1 = interval(rng, n), interval(rng, n)
    base = interval(rng, n)
    u = np.where(rng.random(n) < 0.2, rng.choice([0.0, 0.5, 1.0], n), rng.random(n))
    ref = add(base, scale(u, sub(at1, at0)))
    got = sub(base, scale(u, sub(at0, at1)))
    assert np.array_equal(ref[0].view(np.uint64), got[0].view(np.uint64))
    assert np.array_equal(ref[1].view(np.uint64), got[1].view(np.uint64))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_twice_midpoint_influences_are_exactly_doubled(seed):
    """|rn(lo_a + hi_a) - rn(lo_b + hi_b)| == 2 |m_a - m_b| with m = 0.5 (lo + hi)."""
    rng = np.random.default_rng(seed)
    n = 200_000
    fa, fb = interval(rng, n), interval(rng, n)
    ma, mb = 0.5 * (fa[0] + fa[1]), 0.5 * (fb[0] + fb[1])
    ref = np.abs(ma - mb)
    got = np.abs((fa[0] + fa[1]) - (fb[0] + fb[1]))
    assert np.array_equal((2.0 * ref).view(np.uint64), got.view(np.uint64))
    # the strict comparisons between dimensions are unchanged
    other = np.abs(ma[::-1] - mb)
    other2 = np.abs((fa[0][::-1] + fa[1][::-1]) - (fb[0] + fb[1]))
    assert np.array_equal(ref > other, got > other2)
