"""Functionals, factor matrices, dense Gram and Kronecker matvec (oracle; test infrastructure only).

PAPER.md references
  Eq. 10 (l.206-207): int_a^b D[u] = c_0 int_a^b u + sum_i c_{i+1} (u^{(i)}(b) - u^{(i)}(a))
      -> an interval functional of derivative order m is an antiderivative
         difference (m = 0) or an endpoint difference of u^{(m-1)} (m >= 1).
  l.170: point (collocation / IC / BC) functionals u^{(m)}(p).
  Eq. 15-16 (l.244-246): L_V k L'_V' = sum_{alpha,alpha'} c c' prod_i L_{[a_i,b_i];alpha_i} k^{(i)} L'_{[a'_i,b'_i];alpha'_i}
  Eq. 20 (l.316-318):   L_V k L'_V = sum c c' (x)_i L_{G_i} k^{(i)} L'_{G_i}   (Kronecker structure)
  Eq. 17-19 (l.257-277): multi-output prior with zero cross-covariances
      -> a term pair only contributes when both terms target the same output.
  l.109: G = L k L' + Sigma.

A 1D functional is expanded into weighted evaluations at points e with a
generalised order o (oracle/matern.py):
    point p, order m        -> [(p, +1)],             o = m
    interval [a,b], m = 0   -> [(b, +1), (a, -1)],    o = -1   (antiderivative)
    interval [a,b], m >= 1  -> [(b, +1), (a, -1)],    o = m-1  (Eq. 10)
and since d^o/dx1^o d^o'/dx2^o' k(x1 - x2) = (-1)^o' k^{(o+o')}(x1 - x2)
(negative orders = antiderivatives, the sign rule holds for them as well):
    (L1 k L2')  =  sum_{(e,w)} sum_{(e',w')}  w w' (-1)^o'  g_{o+o'}(e - e').
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import mpmath as mp
import numpy as np

from gpfvm_inputs import INTERVAL, POINT, Grid, Problem, Sites
from .matern import DPS, kernel


def expand(kind: int, lo: float, hi: float, m: int, q: int):
    """Endpoint expansion of one 1D functional (Eq. 10).  Returns (points, weights, o)."""
    if kind == POINT:
        if m > q:
            raise ValueError(f"point functional order {m} exceeds q={q} (sample paths are C^q)")
        return [mp.mpf(lo)], [1], m
    if kind != INTERVAL:
        raise ValueError("unknown site kind")
    if m - 1 > q:
        raise ValueError(f"interval functional order {m} exceeds q+1={q + 1}")
    return [mp.mpf(hi), mp.mpf(lo)], [1, -1], m - 1


def factor_matrix(kern_params: Tuple[int, float, float], left: Sites, m_left: int,
                  right: Sites, m_right: int) -> np.ndarray:
    """F[j, j'] = L_{left_j; m_left} k L'_{right_j'; m_right}   (Eq. 16), fp64-rounded.

    Evaluated in mpmath at DPS digits from exact fp64 endpoints; the lags
    e - e' are exact, so uniform grids hit the memo in ``Matern1D.g``.
    """
    q, ell, var = kern_params
    k = kernel(q, float(ell), float(var))
    L = [expand(left.kind, left.lo[j], left.hi[j], m_left, q) for j in range(left.n)]
    R = [expand(right.kind, right.lo[j], right.hi[j], m_right, q) for j in range(right.n)]
    F = np.empty((left.n, right.n))
    with mp.workdps(DPS):
        for j, (pl, wl, ol) in enumerate(L):
            for jj, (pr, wr, orr) in enumerate(R):
                s = mp.mpf(0)
                o = ol + orr
                for e, w in zip(pl, wl):
                    for e2, w2 in zip(pr, wr):
                        s += w * w2 * k.g(o, e - e2)
                if orr % 2:
                    s = -s
                F[j, jj] = float(s)
    return F


def _kp(problem: Problem, out: int, dim: int) -> Tuple[int, float, float]:
    kk = problem.kernels[out][dim]
    return (kk.q, kk.lengthscale, kk.variance)


def block_pair_terms(problem: Problem, I: int, J: int):
    """All Kronecker terms (coef, [F_0, ..., F_{d-1}]) of the Gram block (I, J), Eq. 15/20.

    Every term pair (tau in block I, tau' in block J) that targets the same
    output contributes c_tau c_tau' (x)_i F_i (Eq. 18-19: delta_{i1 i2}).
    No algebraic simplification is applied here.
    """
    bi, bj = problem.blocks[I], problem.blocks[J]
    out = []
    for t1 in bi.terms:
        for t2 in bj.terms:
            if t1.output != t2.output:
                continue
            fs = [factor_matrix(_kp(problem, t1.output, i), bi.sites[i], t1.order[i],
                                bj.sites[i], t2.order[i]) for i in range(problem.ndim)]
            out.append((t1.coeff * t2.coeff, fs))
    return out


def _kron_all(fs: Sequence[np.ndarray]) -> np.ndarray:
    M = np.ones((1, 1))
    for F in fs:
        M = np.kron(M, F)
    return M


def dense_gram(problem: Problem) -> np.ndarray:
    """G = L k L' + Sigma as a dense fp64 matrix (l.109 and Eq. 20)."""
    off = problem.offsets
    G = np.zeros((off[-1], off[-1]))
    for I in range(len(problem.blocks)):
        for J in range(len(problem.blocks)):
            for c, fs in block_pair_terms(problem, I, J):
                G[off[I]:off[I + 1], off[J]:off[J + 1]] += c * _kron_all(fs)
    G[np.diag_indices_from(G)] += noise_vector(problem)
    return G


def noise_vector(problem: Problem) -> np.ndarray:
    return np.concatenate([np.full(b.size, b.noise, dtype=np.float64) for b in problem.blocks])


class KroneckerGram:
    """Matrix-free G x via Kronecker structure (Eq. 20; "matrix-vector products
    with Kronecker products are cheap and only require access to the individual
    factors", l.320).  Plain: every term applied separately, one mode at a time."""

    def __init__(self, problem: Problem):
        self.problem = problem
        self.off = problem.offsets
        nb = len(problem.blocks)
        self.terms = {(I, J): block_pair_terms(problem, I, J) for I in range(nb) for J in range(nb)}
        self.noise = noise_vector(problem)

    @staticmethod
    def apply_kron(fs: Sequence[np.ndarray], x: np.ndarray, in_shape) -> np.ndarray:
        """((x)_i F_i) x for x flattened row-major with shape in_shape (dim 0 slowest)."""
        X = x.reshape(in_shape)
        for i, F in enumerate(fs):
            X = np.moveaxis(np.tensordot(F, X, axes=([1], [i])), 0, i)
        return X.reshape(-1)

    def matvec(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.ndim == 2:
            return np.stack([self.matvec(v) for v in x])
        blocks = self.problem.blocks
        y = self.noise * x
        for (I, J), lst in self.terms.items():
            xj = x[self.off[J]:self.off[J + 1]]
            for c, fs in lst:
                y[self.off[I]:self.off[I + 1]] += c * self.apply_kron(fs, xj, blocks[J].shape)
        return y


def cross_cov_terms(problem: Problem, grid: Grid, J: int):
    """Kronecker terms of the cross-covariance between u_out(grid points) and
    block J: (L_J k)(x) per Eq. 14 (l.244) with a point functional of order 0
    on the grid side."""
    bj = problem.blocks[J]
    out = []
    for t in bj.terms:
        if t.output != grid.output:
            continue
        fs = []
        for i in range(problem.ndim):
            p = np.asarray(grid.points[i], dtype=np.float64)
            gs = Sites(POINT, p, p)
            fs.append(factor_matrix(_kp(problem, t.output, i), gs, 0, bj.sites[i], t.order[i]))
        out.append((t.coeff, fs))
    return out


def dense_cross_cov(problem: Problem, grid: Grid) -> np.ndarray:
    """K_* (n_grid x N): rows = grid points (row-major, dim 0 slowest)."""
    cols = []
    ng = int(np.prod(grid.shape))
    for J in range(len(problem.blocks)):
        KJ = np.zeros((ng, problem.blocks[J].size))
        for c, fs in cross_cov_terms(problem, grid, J):
            KJ += c * _kron_all(fs)
        cols.append(KJ)
    return np.concatenate(cols, axis=1)


def prior_variance(problem: Problem, out: int = 0) -> float:
    """k(x, x) = prod_i variance_i (Eq. 13, stationary product kernel)."""
    v = 1.0
    for kk in problem.kernels[out]:
        v *= kk.variance
    return v
