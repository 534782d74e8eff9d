"""Pins of the oracle's HR basis (Sec. 3, Eq. 2, lines 90-102) against things other than
the oracle itself: the paper's normalisation statement, sympy differentiation of Eq. 2, the
Beta-function integral, the paper's ReLU^2 formula (Eq. 1), SPEC's worked value, continuity
class, and finite differences."""
import math
import os

import numpy as np
import pytest
import sympy as sp

from oracle import hrkan_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_support_layout_examples():
    # (g=5,k=3,[-1,1]) -> 8 supports of width (k+1)h = 1.6
    s, e = O.make_supports(5, 3, -1.0, 1.0)
    assert len(s) == 8
    np.testing.assert_allclose(e - s, 1.6, rtol=0, atol=1e-15)
    # (g=1,k=1,[0,1]) -> [-1,1] and [0,2]
    s, e = O.make_supports(1, 1, 0.0, 1.0)
    np.testing.assert_array_equal(s, [-1.0, 0.0])
    np.testing.assert_array_equal(e, [1.0, 2.0])
    # the B-spline supports on the extended uniform knot vector cover [lo-kh, hi+kh]
    s, e = O.make_supports(8, 3, -1.0, 1.0)
    assert s[0] == pytest.approx(-1.75) and e[-1] == pytest.approx(1.75)
    with pytest.raises(ValueError):
        O.make_supports(0, 3, -1, 1)
    with pytest.raises(ValueError):
        O.make_supports(5, 3, 1, 1)


def test_worked_value_golden():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "basis_worked_value.txt")) if not l.startswith("#")]
    for s, e, m, x, d, val in rows:
        got = O.hr_basis(float(x), float(s), float(e), int(m), int(d))
        assert float(got) == float(val)


@pytest.mark.parametrize("m", range(1, 9))
def test_midpoint_normalisation(m):
    # P:94 "normalization constant for ensuring the height of each basis being 1"
    for G, k, lo, hi in [(5, 3, -1, 1), (10, 3, -1, 1), (16, 3, -1, 1), (7, 3, 0, 2.5)]:
        s, e = O.make_supports(G, k, lo, hi)
        v = O.hr_basis((s + e) / 2, s, e, m, 0)
        np.testing.assert_allclose(v, 1.0, rtol=0, atol=1e-12)
        # the midpoint is the maximum
        xs = np.linspace(s[0] - 1, e[-1] + 1, 4001)
        assert O.hr_basis(xs[:, None], s, e, m, 0).max() <= 1.0 + 1e-12


@pytest.mark.parametrize("d", range(4))
def test_compact_support_exact_zero(d):
    s, e = O.make_supports(5, 3, -1.0, 1.0)
    rng = np.random.default_rng(0)
    for n in range(len(s)):
        out = np.concatenate([rng.uniform(s[n] - 3, s[n], 50), rng.uniform(e[n], e[n] + 3, 50), [s[n], e[n]]])
        v = O.hr_basis(out, s[n], e[n], 4, d)
        assert np.all(v == 0.0)


@pytest.mark.parametrize("m", range(2, 9))
def test_derivatives_match_sympy(m):
    """Each closed-form derivative equals sympy's derivative of Eq. 2 (not a retyping: sympy
    differentiates the literal product ReLU(e-x)^m ReLU(x-s)^m c_m on the interior)."""
    x = sp.Symbol("x")
    s0, e0 = sp.Rational(-3, 5), sp.Rational(1, 1)
    expr = (e0 - x) ** m * (x - s0) ** m * (2 / (e0 - s0)) ** (2 * m)
    rng = np.random.default_rng(m)
    pts = rng.uniform(float(s0), float(e0), 7)
    for d in range(4):
        f = sp.lambdify(x, sp.diff(expr, x, d), "mpmath")
        for p in pts:
            ref = float(f(sp.Float(p, 30)))
            got = float(O.hr_basis(p, float(s0), float(e0), m, d))
            assert got == pytest.approx(ref, rel=1e-11, abs=1e-11 * max(1.0, abs(ref)))


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6])
def test_quadrature_beta_function(m):
    # int_s^e c (e-x)^m (x-s)^m dx = w * 2^{2m} (m!)^2 / (2m+1)!   (Beta(m+1, m+1) integral)
    s, e = -0.3, 0.9
    w = e - s
    ref = w * 2 ** (2 * m) * math.factorial(m) ** 2 / math.factorial(2 * m + 1)
    xs = np.linspace(s, e, 200001)
    v = O.hr_basis(xs, s, e, m, 0)
    got = np.trapezoid(v, xs)
    assert got == pytest.approx(ref, rel=1e-9)
    # the derivative integrates to zero (compact support)
    assert np.trapezoid(O.hr_basis(xs, s, e, m, 1), xs) == pytest.approx(0.0, abs=1e-9)


def test_m2_equals_relu_squared():
    # the "square of ReLU" basis is the HR basis with m = 2 (c = 16/(e-s)^4 = (2/(e-s))^4)
    s, e = O.make_supports(5, 3, -1.0, 1.0)
    xs = np.linspace(-2.5, 2.5, 1001)[:, None]
    np.testing.assert_allclose(O.hr_basis(xs, s, e, 2, 0), O.relu2_basis(xs, s, e), rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("m", [2, 3, 4, 5])
def test_continuity_class(m):
    """HR of order m is C^{m-1}: one-sided derivatives of order d <= m-1 vanish at the support
    ends (Fig. 3); the ReLU^2 (m=2) second derivative jumps to 32/(e-s)^2."""
    s, e = -1.0, 1.0
    w = e - s
    eps = 1e-6
    for d in range(0, min(m, 4)):
        for x in (s + eps, e - eps):
            v = O.hr_basis(x, s, e, m, d) * (w / 2) ** d
            assert abs(v) < 1e-3
    if m == 2:
        assert float(O.hr_basis(s + 1e-12, s, e, 2, 2)) == pytest.approx(32 / w ** 2, rel=1e-9)
        assert float(O.hr_basis(s, s, e, 2, 2)) == 0.0
    if m == 3:   # third derivative jumps by 48 (2/w)^3 (SURVEY §8(c) reading 2)
        assert float(O.hr_basis(s + 1e-12, s, e, 3, 3)) == pytest.approx(48 * (2 / w) ** 3, rel=1e-6)


@pytest.mark.parametrize("m", [2, 3, 4, 6])
def test_derivatives_central_fd(m):
    # analytic derivative vs central FD of the (d-1)-th derivative, rel < 1e-6,
    # step 1e-5 (e-s), 50 random interior points
    s, e = -0.2, 0.6
    h = 1e-5 * (e - s)
    rng = np.random.default_rng(10 + m)
    xs = rng.uniform(s + 0.01, e - 0.01, 50)
    for d in (1, 2, 3):
        if d >= 2 * m:
            continue
        fd = (O.hr_basis(xs + h, s, e, m, d - 1) - O.hr_basis(xs - h, s, e, m, d - 1)) / (2 * h)
        an = O.hr_basis(xs, s, e, m, d)
        scale = np.abs(an).max()
        np.testing.assert_allclose(fd, an, rtol=0, atol=1e-6 * scale)


def test_symmetry():
    s, e = O.make_supports(10, 3, -1.0, 1.0)
    mid = (s + e) / 2
    for dlt in (0.01, 0.1, 0.2):
        for d in range(4):
            a = O.hr_basis(mid + dlt, s, e, 4, d)
            b = O.hr_basis(mid - dlt, s, e, 4, d)
            np.testing.assert_allclose(a, (-1) ** d * b, rtol=1e-12, atol=1e-12)


def test_at_most_k_plus_1_active():
    # compact support on the uniform extended grid: at any x at most k+1 bases are non-zero
    for G, k in [(5, 3), (10, 3), (8, 3), (16, 3)]:
        s, e = O.make_supports(G, k, -1.0, 1.0)
        xs = np.random.default_rng(0).uniform(-2, 2, 2000)[:, None]
        nz = (O.hr_basis(xs, s, e, 4, 0) != 0).sum(axis=1)
        assert nz.max() <= k + 1
