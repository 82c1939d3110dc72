"""Pins for the oracle's 1D Matérn calculus and factor matrices (CPU only).

Each test ties oracle/matern.py / oracle/gram.py to something other than
itself: the literal Eq. 12 formula, numerical differentiation, adaptive
quadrature of the defining integrals, printed closed forms
(tests/golden/closed_forms.txt) and structural identities.
"""
import os

import mpmath as mp
import numpy as np
import pytest

from gpfvm_inputs import INTERVAL, POINT, Sites
from oracle.gram import factor_matrix
from oracle.matern import Matern1D, matern_direct

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "closed_forms.txt")


def _site(spec):
    parts = spec.split(":")
    if parts[0] == "pt":
        p = float(parts[1])
        return Sites(POINT, np.array([p]), np.array([p])), int(parts[2])
    a, b = float(parts[1]), float(parts[2])
    return Sites(INTERVAL, np.array([a]), np.array([b])), int(parts[3])


def _golden_rows():
    rows = []
    for line in open(GOLDEN):
        line = line.split("#")[0].strip()
        if not line:
            continue
        q, ell, var, f1, f2, val = line.split()
        rows.append((int(q), float(ell), float(var), f1, f2, float(val)))
    return rows


@pytest.mark.parametrize("row", _golden_rows())
def test_golden_closed_forms(row):
    q, ell, var, f1, f2, val = row
    s1, m1 = _site(f1)
    s2, m2 = _site(f2)
    got = factor_matrix((q, ell, var), s1, m1, s2, m2)[0, 0]
    assert abs(got - val) <= 1e-15 * max(1.0, abs(val))


@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_recurrence_matches_eq12_and_numerical_derivatives(q):
    """k^{(n)} from the product-rule recurrence == numerical derivatives of
    the literal Eq. 12 formula (mpmath.diff, high precision), off the diagonal
    and (for n <= 2q) at 0 from the right."""
    ell, var = 0.7, 1.3
    k = Matern1D(q, ell, var)
    f = lambda d: matern_direct(q, ell, var, d)
    for d in [0.05, 0.3, 1.1, 2.7]:
        assert abs(k.g(0, d) - f(d)) < mp.mpf(10) ** -35
        for n in range(1, 2 * q + 1):
            ref = mp.diff(f, mp.mpf(d), n)
            assert abs(k.g(n, d) - ref) <= mp.mpf(10) ** -20 * max(1, abs(ref)), (q, n, d)
            # parity g_n(-d) = (-1)^n g_n(d)
            assert abs(k.g(n, -d) - (-1) ** n * k.g(n, d)) < mp.mpf(10) ** -30


@pytest.mark.parametrize("q", [0, 1, 2, 3])
def test_antiderivatives_match_quadrature(q):
    k = Matern1D(q, 0.4, 1.0)
    for d in [-1.3, -0.2, 0.0, 0.15, 0.9]:
        K1 = mp.quad(lambda s: k.g(0, s), [0, d]) if d != 0 else mp.mpf(0)
        assert abs(k.g(-1, d) - K1) < mp.mpf(10) ** -25
        K2 = mp.quad(lambda s: k.g(-1, s), [0, d]) if d != 0 else mp.mpf(0)
        assert abs(k.g(-2, d) - K2) < mp.mpf(10) ** -25


def _quad_functional_pair(q, ell, var, s1, m1, s2, m2):
    """Brute-force value of L1 k L2' by adaptive quadrature of the defining
    integrals (split at the diagonal kink) and mpmath numerical derivatives of
    the literal Eq. 12 formula — no antiderivative or FTC used."""
    f = lambda d: matern_direct(q, ell, var, d)

    def dk(n, d):  # d^n/dd^n k(d), numerically, with the kink at 0 avoided
        if n == 0:
            return f(d)
        if abs(d) < mp.mpf(10) ** -30:
            return mp.diff(f, mp.mpf(10) ** -12, n) if n % 2 == 0 else mp.mpf(0)
        return mp.diff(f, d, n)

    def left(x2, m2_, fun):  # apply functional 1 in x1 to x1 -> fun(x1 - x2)
        if s1[0] == "pt":
            return fun(m1, s1[1] - x2)
        a, b = s1[1], s1[2]
        pts = [a, b] if not (a < x2 < b) else [a, x2, b]
        return mp.quad(lambda x1: fun(m1, x1 - x2), pts)

    def both():
        # d^m1/dx1^m1 d^m2/dx2^m2 k(x1-x2) = (-1)^m2 k^{(m1+m2)}(x1-x2)
        fun = lambda m, d: (-1) ** m2 * dk(m + m2, d)
        if s2[0] == "pt":
            return left(s2[1], m2, fun)
        a, b = s2[1], s2[2]
        inner = lambda x2: left(x2, m2, fun)
        cuts = sorted(set([a, b] + [c for c in s1[1:] if a < c < b]))
        return mp.quad(inner, cuts)

    with mp.workdps(30):
        return both()


CASES = [
    # q, ell, left site, m1, right site, m2
    (0, 1.0, ("iv", 0.0, 1.0), 0, ("pt", 0.0), 0),
    (2, 0.5, ("iv", 0.0, 1.0), 0, ("iv", 0.25, 0.75), 0),          # SPEC.md example (overlap)
    (2, 0.2, ("iv", 0.1, 0.3), 0, ("iv", 0.5, 0.6), 0),             # disjoint
    (2, 0.2, ("iv", 0.1, 0.3), 0, ("iv", 0.3, 0.45), 0),            # touching
    (3, 0.3, ("iv", 0.0, 0.2), 0, ("iv", 0.1, 0.4), 0),
    (1, 0.6, ("iv", 0.0, 0.3), 0, ("pt", 0.2), 0),                  # point inside interval
    (2, 0.5, ("pt", 0.1), 1, ("pt", 0.4), 1),
    (2, 0.5, ("pt", 0.1), 2, ("pt", 0.4), 0),
    (2, 0.4, ("iv", 0.0, 0.3), 1, ("iv", 0.5, 0.9), 0),             # FTC m=1 vs integral
    (2, 0.4, ("iv", 0.0, 0.3), 2, ("iv", 0.2, 0.9), 2),             # heat x-factor pair (2,2)
    (2, 0.4, ("iv", 0.0, 0.3), 0, ("iv", 0.1, 0.5), 2),
    (3, 0.25, ("iv", 0.0, 0.1), 2, ("iv", 0.3, 0.45), 2),           # wave t-factor pair (2,2)
    (3, 0.25, ("pt", 0.0), 1, ("iv", 0.05, 0.3), 2),                 # IC u_t against wave cell
]


def _to_sites(s):
    if s[0] == "pt":
        return Sites(POINT, np.array([s[1]]), np.array([s[1]]))
    return Sites(INTERVAL, np.array([s[1]]), np.array([s[2]]))


@pytest.mark.parametrize("case", CASES)
def test_factor_entries_match_bruteforce_quadrature(case):
    q, ell, s1, m1, s2, m2 = case
    got = factor_matrix((q, ell, 1.0), _to_sites(s1), m1, _to_sites(s2), m2)[0, 0]
    ref = float(_quad_functional_pair(q, ell, 1.0, s1, m1, s2, m2))
    assert abs(got - ref) <= 1e-10 * max(1e-3, abs(ref)), (got, ref)


def test_factor_symmetry_and_parity():
    """F^{m'm} = (F^{mm'})^T always; on identical site lists F^{mm'} is
    symmetric for m+m' even and skew for m+m' odd (R6)."""
    e = np.array([0.0, 0.1, 0.25, 0.3, 0.6, 1.0])
    S = Sites(INTERVAL, e[:-1], e[1:])
    for m, mm in [(0, 0), (0, 1), (1, 2), (0, 2), (2, 2), (1, 1)]:
        F = factor_matrix((2, 0.3, 1.0), S, m, S, mm)
        Ft = factor_matrix((2, 0.3, 1.0), S, mm, S, m)
        assert np.array_equal(Ft, F.T)
        sgn = 1 if (m + mm) % 2 == 0 else -1
        assert np.abs(F - sgn * F.T).max() <= 1e-16 * np.abs(F).max()


def test_order_limits_rejected():
    S = Sites(POINT, np.array([0.0]), np.array([0.0]))
    with pytest.raises(ValueError):
        factor_matrix((1, 1.0, 1.0), S, 2, S, 0)
