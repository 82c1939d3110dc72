"""Solvers (oracle; test infrastructure only).

* ``cholesky_solve`` — the classic approach, §4 l.289-291:
  G = L L^T, then forward/backward substitution.
* ``FDPreconditioner`` / ``BlockLDLPreconditioner`` — the preconditioner the
  CUDA path uses, written out from its definition in DESIGN.md §5 (fast
  diagonalisation of the two-term Kronecker PDE block + exact Schur
  complement on the IC/BC observations, the latter generalising the paper's
  Cholesky deflation of §4.2, l.324-339).
* ``itergp_cg`` — IterGP with (preconditioned) CG actions and full
  reorthogonalisation, §4.1 l.295-302 ("IterGP generalizes CG ...
  produces a combined posterior"), §6 l.475 ("regular full
  reorthogonalization"), Wenger et al. 2022 Alg. 1 with C_0 = 0:
      s_i   = P^{-1} r_{i-1}                      (action, CG policy)
      z_i   = G s_i
      d_i   = s_i - C_{i-1} z_i                    (G-orthogonalise)
      eta_i = z_i^T d_i            (= d_i^T G d_i)
      C_i   = C_{i-1} + d_i d_i^T / eta_i
      x_i   = C_i y,   r_i = y - G x_i
  Directions d_i and eta_i are the "Krylov actions kept for the
  computational-uncertainty downdate".
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.linalg as sl

from gpfvm_inputs import Problem
from .gram import block_pair_terms


def cholesky_solve(G: np.ndarray, y: np.ndarray) -> np.ndarray:
    L = np.linalg.cholesky(G)
    return sl.cho_solve((L, True), y)


class FDPreconditioner:
    """Fast-diagonalisation inverse of a 2D non-deflated block.

    The block's diagonal Gram keeps, from Eq. 20's double sum, the two
    'diagonal' term pairs (tau, tau):
        G_PP ~= c_a A0 (x) A1 + c_b B0 (x) B1,   a = term with the larger time order,
    (for the heat operator the cross pairs cancel exactly, R6).
    With the generalised eigenproblems
        B0 V = A0 V Lam,  V^T A0 V = I;        A1 W = B1 W M,  W^T B1 W = I
    (V (x) W)^T G_PP (V (x) W) = c_a I (x) M + c_b Lam (x) I =: D, so
        P^{-1} = (V (x) W) D^{-1} (V (x) W)^T
    with the block noise folded in through its diagonal in the new basis.
    """

    def __init__(self, problem: Problem, P: int):
        blk = problem.blocks[P]
        if problem.ndim != 2 or len(blk.terms) != 2:
            raise NotImplementedError("FD preconditioner: 2D block with a two-term operator")
        ta, tb = blk.terms
        if ta.order[0] < tb.order[0]:
            ta, tb = tb, ta
        pairs = block_pair_terms(problem, P, P)
        # locate (ta,ta) and (tb,tb) among the pairs (order of block_pair_terms: t1 outer, t2 inner)
        idx = {}
        k = 0
        for t1 in blk.terms:
            for t2 in blk.terms:
                idx[(id(t1), id(t2))] = k
                k += 1
        ca, (A0, A1) = pairs[idx[(id(ta), id(ta))]]
        cb, (B0, B1) = pairs[idx[(id(tb), id(tb))]]
        lam, V = sl.eigh(B0, A0)
        mu, W = sl.eigh(A1, B1)
        self.V, self.W = V, W
        self.shape = blk.shape
        D = ca * mu[None, :] + cb * lam[:, None]
        if blk.noise:
            D = D + blk.noise * np.outer(np.sum(V * V, 0), np.sum(W * W, 0))
        self.D = D

    def apply(self, r: np.ndarray) -> np.ndarray:
        R = r.reshape(self.shape)
        Z = self.V.T @ R @ self.W
        Z = Z / self.D
        return (self.V @ Z @ self.W.T).reshape(-1)


class BlockLDLPreconditioner:
    """P^{-1} for G = [[G_bb, G_bp], [G_pb, G_pp]] (b = deflated IC/BC blocks,
    p = the FD block), DESIGN.md §5.2:
        Y = FD(G_pb),  S = G_bb - G_pb^T Y  (Cholesky, shifted only on failure),
        P^{-1} r = [z_b; z_p],  z_p0 = FD r_p,  z_b = S^{-1}(r_b - G_pb^T z_p0),
                               z_p = z_p0 - Y z_b.
    With an exact FD this is exactly G^{-1} (block LDL^T factorisation)."""

    def __init__(self, problem: Problem, G: np.ndarray):
        blocks = problem.blocks
        off = problem.offsets
        nd = [i for i, b in enumerate(blocks) if not b.deflate]
        if len(nd) != 1:
            raise NotImplementedError("exactly one non-deflated block supported")
        P = nd[0]
        self.pidx = np.arange(off[P], off[P + 1])
        self.bidx = np.concatenate([np.arange(off[i], off[i + 1]) for i, b in enumerate(blocks)
                                    if b.deflate] + [np.zeros(0, dtype=int)]).astype(int)
        self.fd = FDPreconditioner(problem, P)
        Gpb = G[np.ix_(self.pidx, self.bidx)]
        Gbb = G[np.ix_(self.bidx, self.bidx)]
        self.Gpb = Gpb
        if len(self.bidx):
            self.Y = np.stack([self.fd.apply(Gpb[:, i]) for i in range(Gpb.shape[1])], 1)
            S = Gbb - Gpb.T @ self.Y
            S = 0.5 * (S + S.T)
            shift = 0.0
            dmax = float(np.max(np.diag(S)))
            while True:
                try:
                    self.L = np.linalg.cholesky(S + shift * np.eye(len(S)))
                    break
                except np.linalg.LinAlgError:
                    shift = 1e-14 * dmax if shift == 0.0 else shift * 10.0
            self.shift = shift
        self.n = G.shape[0]

    def apply(self, r: np.ndarray) -> np.ndarray:
        z = np.zeros(self.n)
        zp0 = self.fd.apply(r[self.pidx])
        if len(self.bidx):
            zb = sl.cho_solve((self.L, True), r[self.bidx] - self.Gpb.T @ zp0)
            z[self.bidx] = zb
            z[self.pidx] = zp0 - self.Y @ zb
        else:
            z[self.pidx] = zp0
        return z


@dataclass
class IterGPTrace:
    x: np.ndarray
    directions: List[np.ndarray] = field(default_factory=list)
    etas: List[float] = field(default_factory=list)
    residual_norms: List[float] = field(default_factory=list)
    iterations: int = 0
    converged: bool = False


def itergp_cg(matvec, y: np.ndarray, precond=None, rtol: float = 1e-8, max_iter: int = 1000) -> IterGPTrace:
    """IterGP with CG actions, full reorthogonalisation (module docstring)."""
    y = np.asarray(y, dtype=np.float64)
    n = y.shape[0]
    x = np.zeros(n)
    r = y.copy()
    ny = np.linalg.norm(y)
    tr = IterGPTrace(x=x)
    Gd: List[np.ndarray] = []
    tr.residual_norms.append(np.linalg.norm(r) / ny if ny > 0 else 0.0)
    if ny == 0.0:
        tr.converged = True
        return tr
    for it in range(max_iter):
        if np.linalg.norm(r) <= rtol * ny:
            tr.converged = True
            break
        s = precond(r) if precond is not None else r.copy()
        z = matvec(s)
        d = s.copy()
        gd = z.copy()
        for dj, gdj, ej in zip(tr.directions, Gd, tr.etas):
            c = (dj @ z) / ej
            d -= c * dj
            gd -= c * gdj
        eta = float(z @ d)
        if not eta > 0:
            break
        a = float(d @ r) / eta
        x = x + a * d
        r = r - a * gd
        tr.directions.append(d)
        Gd.append(gd)
        tr.etas.append(eta)
        tr.iterations = it + 1
        tr.residual_norms.append(np.linalg.norm(r) / ny)
    else:
        tr.converged = bool(np.linalg.norm(r) <= rtol * ny)
    tr.x = x
    return tr
