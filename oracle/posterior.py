"""Posterior mean / variance on a tensor grid (oracle; test infrastructure only).

PAPER.md Eq. 5 (l.113):  m*(x) = m(x) + L k(x)^T G^+ (y - (L[m] + mu)),   zero prior mean
PAPER.md Eq. 6 (l.114):  k*(x1,x2) = k(x1,x2) - L k(x1)^T G^+ L k(x2)
IterGP combined posterior (§4.1, l.299-302): G^+ -> C_i = sum_j d_j d_j^T / eta_j.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sl

from gpfvm_inputs import Grid, Problem
from .gram import dense_cross_cov, prior_variance


def posterior_exact(problem: Problem, grid: Grid, G: np.ndarray, y: np.ndarray):
    """Exact mean and marginal variance via a dense Cholesky of G (§4 l.289)."""
    Ks = dense_cross_cov(problem, grid)
    L = np.linalg.cholesky(G)
    alpha = sl.cho_solve((L, True), y)
    mean = Ks @ alpha
    V = sl.solve_triangular(L, Ks.T, lower=True)
    var = prior_variance(problem, grid.output) - np.sum(V * V, axis=0)
    return mean, var, alpha


def posterior_from_weights(problem: Problem, grid: Grid, alpha: np.ndarray) -> np.ndarray:
    """m*(x) = K_* alpha."""
    return dense_cross_cov(problem, grid) @ alpha


def variance_itergp(problem: Problem, grid: Grid, directions, etas) -> np.ndarray:
    """Combined variance k(x,x) - sum_j (k_x^T d_j)^2 / eta_j (IterGP, C_0 = 0)."""
    Ks = dense_cross_cov(problem, grid)
    var = np.full(Ks.shape[0], prior_variance(problem, grid.output))
    for d, e in zip(directions, etas):
        var -= (Ks @ d) ** 2 / e
    return var


def variance_precond(problem: Problem, grid: Grid, precond_apply) -> np.ndarray:
    """k(x,x) - k_x^T P^{-1} k_x with the preconditioner as the inverse
    approximation (exact when P^{-1} = G^{-1})."""
    Ks = dense_cross_cov(problem, grid)
    var = np.full(Ks.shape[0], prior_variance(problem, grid.output))
    for i in range(Ks.shape[0]):
        var[i] -= Ks[i] @ precond_apply(Ks[i])
    return var
