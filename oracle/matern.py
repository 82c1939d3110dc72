"""1D half-integer Matérn kernel calculus in high precision (oracle; test infrastructure only).

PAPER.md §3.1 (l.211-220), Eq. 12:
    k_{nu=q+1/2}(r) = exp(-sqrt(2q+1) r) p_q(sqrt(2q+1) r),     r = |x1-x2|/l
with p_q the order-q polynomial "with known coefficients" (Rasmussen &
Williams 2006, Eq. 4.16):
    p_q(s) = q!/(2q)! * sum_{i=0}^{q} (q+i)!/(i!(q-i)!) (2s)^(q-i).
"Application of the product rule shows that derivatives again have the form
of an exponential times a polynomial" (l.218) and "one can also derive
efficient closed-form integrals" (l.220): both are written out below.

Everything is evaluated with mpmath at ``DPS`` significant digits so that the
cancellation in the endpoint formulas (R2) does not limit the
oracle; values are rounded to fp64 by the caller.

Generalised order o of a 1D function of the lag d = x1 - x2:
    g_o(d) = k^{(o)}(d)        for o >= 0   (o-th derivative)
    g_{-1}(d) = K1(d) = int_0^d k                (odd antiderivative)
    g_{-2}(d) = K2(d) = int_0^d K1               (even second antiderivative)
with parity g_o(-d) = (-1)^o g_o(d).
"""
from __future__ import annotations

import math
from fractions import Fraction
from functools import lru_cache

import mpmath as mp

DPS = 40
mp.mp.dps = DPS


def pq_coefficients(q: int):
    """Exact coefficients c_k of p_q(s) = sum_k c_k s^k (Rasmussen & Williams Eq. 4.16)."""
    c = [Fraction(0)] * (q + 1)
    for i in range(q + 1):
        c[q - i] += Fraction(math.factorial(q), math.factorial(2 * q)) * \
            Fraction(math.factorial(q + i), math.factorial(i) * math.factorial(q - i)) * 2 ** (q - i)
    return c


def _mpf(v):
    if isinstance(v, Fraction):
        return mp.mpf(v.numerator) / v.denominator
    return mp.mpf(v)


class Matern1D:
    """k(d) = variance * exp(-lam |d|) * p_q(lam |d|),  lam = sqrt(2q+1)/lengthscale."""

    def __init__(self, q: int, lengthscale: float, variance: float = 1.0):
        if q < 0:
            raise ValueError("q must be >= 0")
        if not (lengthscale > 0 and variance > 0):
            raise ValueError("lengthscale and variance must be positive")
        with mp.workdps(DPS):
            self.q = q
            self.lam = mp.sqrt(2 * q + 1) / mp.mpf(lengthscale)
            var = mp.mpf(variance)
            pc = pq_coefficients(q)
            # polynomial in d (not s = lam d): a_k = var * c_k * lam^k
            a = [var * _mpf(pc[k]) * self.lam ** k for k in range(q + 1)]
            # k^{(n)}(d) = exp(-lam d) P_n(d) for d > 0; P_{n+1} = P_n' - lam P_n (product rule)
            self.der = [a]
            for _ in range(2 * q + 2):
                p = self.der[-1]
                dp = [mp.mpf(0)] * len(p)
                for k in range(1, len(p)):
                    dp[k - 1] += k * p[k]
                for k in range(len(p)):
                    dp[k] -= self.lam * p[k]
                self.der.append(dp)
            # int exp(-lam s) A(s) ds = -exp(-lam s) B(s):  lam b_k - (k+1) b_{k+1} = a_k
            self.B = self._anti(a)
            self.C = self._anti(self.B)
        self._cache = {}

    def _anti(self, a):
        n = len(a)
        b = [mp.mpf(0)] * n
        b[n - 1] = a[n - 1] / self.lam
        for k in range(n - 2, -1, -1):
            b[k] = (a[k] + (k + 1) * b[k + 1]) / self.lam
        return b

    @staticmethod
    def _poly(c, x):
        acc = mp.mpf(0)
        for coef in reversed(c):
            acc = acc * x + coef
        return acc

    def g(self, o: int, d) -> mp.mpf:
        """Generalised-order function g_o(d) (module docstring), exact in mpmath.

        ``d`` may be an mpf (exact lag) or a float.  Orders above 2q are
        rejected: k is only 2q times continuously differentiable at 0.
        """
        if o > 2 * self.q:
            raise ValueError(f"order {o} exceeds 2q = {2 * self.q} (kernel smoothness)")
        if o < -2:
            raise ValueError("orders below -2 are not needed")
        key = (o, d)
        hit = self._cache.get(key)
        if hit is not None:
            return hit
        with mp.workdps(DPS):
            d = mp.mpf(d)
            ad = abs(d)
            sgn = mp.sign(d)
            e = mp.exp(-self.lam * ad)
            if o >= 0:
                v = e * self._poly(self.der[o], ad)
                if o % 2 == 1:
                    v = v * sgn
            elif o == -1:
                v = sgn * (self.B[0] - e * self._poly(self.B, ad))
            else:
                v = self.B[0] * ad - self.C[0] + e * self._poly(self.C, ad)
        self._cache[key] = v
        return v

    def k(self, d) -> mp.mpf:
        return self.g(0, d)


@lru_cache(maxsize=None)
def kernel(q: int, lengthscale: float, variance: float) -> Matern1D:
    return Matern1D(q, lengthscale, variance)


def matern_direct(q: int, lengthscale: float, variance: float, d) -> mp.mpf:
    """Eq. 12 written out literally (used by the pins as the independent
    definition the recurrences above are checked against)."""
    with mp.workdps(max(DPS, mp.mp.dps)):
        s = mp.sqrt(2 * q + 1) * abs(mp.mpf(d)) / mp.mpf(lengthscale)
        p = sum(_mpf(c) * s ** k for k, c in enumerate(pq_coefficients(q)))
        return mp.mpf(variance) * mp.exp(-s) * p
