"""Time-mode sharded GP-FVM operator and solver (north_star multi-GPU row,
DESIGN.md §7).

The PDE observation tensor (n0 time cells x spatial cells) is split along the
time mode into W contiguous slabs, one per rank.  For a Kronecker sum
``G x = sum_p (F0_p (x) F1_p (x) ...) x`` (Eq. 20):

  1. every rank contracts its slab with the spatial factors, writing one
     (slab x spatial-chunk) block per destination rank and term (no packing:
     the factor rows of the destination's chunk are used directly);
  2. ``all_to_all`` re-partitions to "all times x one spatial chunk";
  3. one GEMM contracts the time mode for all terms at once (the term sum is
     the K-concatenation: A_big[m, (src, p, t)] = c_p F0_p[m, src*nt + t]);
  4. ``all_to_all`` back, and a permute kernel restores the slab layout.
CG inner products are local partial dots + ``all_reduce``.  Communication per
matvec: (P + 1) N 8 bytes.

All arithmetic goes through a ``LocalOps`` backend.  ``GpuOps`` calls the
library kernels (gpfvm_kron_matvec, gpfvm_gemm, gpfvm_permute,
gpfvm_dot_many, gpfvm_axpy_many, gpfvm_sygv); the CPU backend used by the
gloo tests lives in ``tests/`` (test infrastructure).  torch.distributed only
moves bytes (NCCL over NVLink on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence

import torch
import torch.distributed as dist

from . import _lib as L


class GpuOps:
    """Library-kernel implementations of the local operations (CUDA tensors)."""

    def __init__(self, device):
        self.lib = L.load()
        self.device = torch.device(device)

    def _s(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def empty(self, *shape):
        return torch.empty(*shape, dtype=torch.float64, device=self.device)

    def zeros(self, *shape):
        return torch.zeros(*shape, dtype=torch.float64, device=self.device)   # memset (plumbing)

    def kron(self, in_shape, out_shape, coefs, factors, x, y, nrhs, beta=0.0):
        d = len(in_shape)
        ins = (C.c_int * d)(*in_shape)
        outs = (C.c_int * d)(*out_shape)
        cf = (C.c_double * len(coefs))(*coefs)
        fp = (C.c_void_p * (len(coefs) * d))(*[f.data_ptr() for term in factors for f in term])
        nin = 1
        nout = 1
        for a, b in zip(in_shape, out_shape):
            nin *= a
            nout *= b
        L.check(self.lib.gpfvm_kron_matvec(d, ins, outs, len(coefs), cf, fp, self._p(x), nin, self._p(y), nout,
                                           int(nrhs), float(beta), self._s()))

    def gemm(self, A, B, Cm, alpha=1.0, beta=0.0):
        M, K = A.shape
        K2, N = B.shape
        assert K == K2 and Cm.shape == (M, N)
        L.check(self.lib.gpfvm_gemm(M, N, K, float(alpha), self._p(A), A.stride(0), self._p(B), B.stride(0),
                                    float(beta), self._p(Cm), Cm.stride(0), self._s()))

    def permute(self, src, shape, perm):
        d = len(shape)
        out = self.empty([shape[p] for p in perm])
        L.check(self.lib.gpfvm_permute(d, (C.c_int * d)(*shape), (C.c_int * d)(*perm), self._p(src),
                                       self._p(out), self._s()))
        return out

    def dots(self, X, v):
        """[X_j . v for j] as a tensor (local partial dots)."""
        k = X.shape[0]
        out = self.empty(k)
        L.check(self.lib.gpfvm_dot_many(self._p(X), X.stride(0), self._p(v), v.numel(), k, self._p(out), self._s()))
        return out

    def axpy(self, y, X, coef, sign=1.0):
        k = X.shape[0]
        L.check(self.lib.gpfvm_axpy_many(self._p(y), self._p(X), X.stride(0), self._p(coef), float(sign), y.numel(),
                                         k, self._s()))

    def vmul(self, x, d):
        L.check(self.lib.gpfvm_vmul(self._p(x), self._p(d), x.numel(), self._s()))
        return x

    def transpose(self, A):
        return self.permute(A, list(A.shape), [1, 0])

    def fd_setup(self, ca, A0, A1, cb, B0, B1, noise):
        n0, n1 = A0.shape[0], A1.shape[0]
        V = self.empty(n0, n0)
        Wm = self.empty(n1, n1)
        Dinv = self.empty(n0, n1)
        L.check(self.lib.gpfvm_fd_setup(n0, n1, self._p(A0), self._p(A1), self._p(B0), self._p(B1), float(ca),
                                        float(cb), float(noise), self._p(V), self._p(Wm), self._p(Dinv), self._s()))
        return V, Wm, Dinv

    def sygv(self, A, B):
        n = A.shape[0]
        V = self.empty(n, n)
        w = self.empty(n)
        L.check(self.lib.gpfvm_sygv(n, self._p(A), self._p(B), self._p(V), self._p(w), self._s()))
        return V, w


@dataclass
class ShardedKron:
    """y = sum_p c_p ((x)_i F_{p,i}) x with x, y sharded along dim 0."""

    ops: object
    shape: Sequence[int]                 # (n0, n1, ...) square operator
    coefs: List[float]
    factors: List[List[torch.Tensor]]    # full factors, factors[p][i] : n_i x n_i
    group: object = None
    rank: int = 0
    world: int = 1
    A_big: torch.Tensor = field(init=False, default=None)

    def __post_init__(self):
        n0 = self.shape[0]
        W = self.world
        if n0 % W or self.shape[1] % W:
            raise ValueError(f"time ({n0}) and first spatial ({self.shape[1]}) sizes must be divisible by {W}")
        self.nt = n0 // W
        self.rest = 1
        for s in self.shape[1:]:
            self.rest *= s
        self.c1 = self.shape[1] // W
        self.cw = self.rest // W
        P = len(self.coefs)
        # A_big[m, (src, p, t)] = c_p F0_p[m, src*nt + t]
        F0 = self.ops.empty(P, n0, n0)
        for p in range(P):
            F0[p].copy_(self.factors[p][0])     # device copy (plumbing); c_p is applied in step 1
        self.A_big = self.ops.permute(F0.reshape(P, n0, W, self.nt), [P, n0, W, self.nt], [1, 2, 0, 3]).reshape(
            n0, W * P * self.nt)

    def matvec(self, x_local):
        P, W, nt, cw = len(self.coefs), self.world, self.nt, self.cw
        spatial = list(self.shape[1:])
        # one spatial Kronecker product per term over all destination chunks
        # (P library calls instead of W * P), then one permutation into the
        # all-to-all send layout [dest chunk][term][local time][chunk]
        full = self.ops.empty(P, nt, self.rest)
        for p in range(P):
            fac = [self.factors[p][1]] + list(self.factors[p][2:])
            self.ops.kron(spatial, spatial, [self.coefs[p]], [fac], x_local, full[p], nrhs=nt)
        send = self.ops.permute(full, [P, nt, W, cw], [2, 0, 1, 3])
        recv = _all_to_all(send, self.group, W)
        yspace = self.ops.empty(self.shape[0], cw)
        self.ops.gemm(self.A_big, recv.reshape(W * P * nt, cw), yspace)
        back = _all_to_all(yspace.reshape(W, nt, cw), self.group, W)
        return self.ops.permute(back, [W, nt, cw], [1, 0, 2]).reshape(-1)


def _all_to_all(t, group, W):
    if W == 1:
        return t
    out = torch.empty_like(t)
    dist.all_to_all_single(out.view(-1), t.contiguous().view(-1), group=group)
    return out


def allreduce_(t, group, W):
    if W > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


@dataclass
class ShardedFD:
    """Sharded fast-diagonalisation inverse of the 2D heat
    PDE block  c_a A0(x)A1 + c_b B0(x)B1:  (V(x)W) D^{-1} (V(x)W)^T."""

    ops: object
    fwd: ShardedKron      # applies V^T (x) W^T
    bwd: ShardedKron      # applies V (x) W
    dinv_local: torch.Tensor

    def apply(self, r_local):
        z = self.fwd.matvec(r_local)
        self.ops.vmul(z, self.dinv_local)
        return self.bwd.matvec(z)


def build_fd(ops, shape, ca, A0, A1, cb, B0, B1, noise, group, rank, world):
    V, Wm, Dinv = ops.fd_setup(ca, A0, A1, cb, B0, B1, noise)
    n0, n1 = shape
    nt = n0 // world
    dinv_local = Dinv[rank * nt:(rank + 1) * nt].reshape(-1).contiguous()
    fwd = ShardedKron(ops, shape, [1.0], [[ops.transpose(V), ops.transpose(Wm)]], group, rank, world)
    bwd = ShardedKron(ops, shape, [1.0], [[V, Wm]], group, rank, world)
    return ShardedFD(ops, fwd, bwd, dinv_local)


def heat_pde_operator(ops, factors, kappa, group=None, rank=0, world=1, noise=0.0):
    """Sharded PDE-block operator and FD preconditioner of the heat problem
    (terms T11(x)X00 + kappa^2 T00(x)X22 after the R6 cancellation).
    ``factors``: dict with keys T00, T11, X00, X22 (full matrices on the ops device)."""
    n0, n1 = factors["T00"].shape[0], factors["X00"].shape[0]
    A = ShardedKron(ops, (n0, n1), [1.0, kappa * kappa],
                    [[factors["T11"], factors["X00"]], [factors["T00"], factors["X22"]]], group, rank, world)
    fd = build_fd(ops, (n0, n1), 1.0, factors["T11"], factors["X00"], kappa * kappa, factors["T00"],
                  factors["X22"], noise, group, rank, world)
    return A, fd


@dataclass
class PCGResult:
    x: torch.Tensor
    iterations: int
    rel_residual: float
    converged: bool
    residual_norms: list


def sharded_pcg(ops, A: ShardedKron, y_local, precond=None, rtol=1e-8, max_iter=200, group=None, world=1):
    """IterGP/PCG with full reorthogonalisation (R7) on sharded vectors."""
    n = y_local.numel()
    x = ops.zeros(n)
    r = ops.empty(n)
    r.copy_(y_local)
    ny = float(allreduce_(ops.dots(r.reshape(1, -1), r), group, world)[0]) ** 0.5
    D = ops.empty(max_iter + 1, n)
    GD = ops.empty(max_iter + 1, n)
    etas = []
    norms = [1.0]
    k = 0
    nr = ny
    converged = ny == 0.0
    while not converged and k < max_iter:
        if nr <= rtol * ny:
            converged = True
            break
        if precond is not None:
            s = precond.apply(r)
        else:
            s = ops.empty(n)
            s.copy_(r)
        z = A.matvec(s)
        D[k].copy_(s)
        GD[k].copy_(z)
        if k > 0:
            c = allreduce_(ops.dots(D[:k], z), group, world).cpu()          # k scalars
            c = torch.tensor([float(c[j]) / etas[j] for j in range(k)], dtype=torch.float64).to(z.device)
            ops.axpy(D[k], D[:k], c, -1.0)
            ops.axpy(GD[k], GD[:k], c, -1.0)
        two = ops.empty(2)
        two[0:1].copy_(ops.dots(D[k].reshape(1, -1), GD[k]))
        two[1:2].copy_(ops.dots(D[k].reshape(1, -1), r))
        two = allreduce_(two, group, world).cpu()
        eta, dr = float(two[0]), float(two[1])
        if not eta > 0:
            break
        a = dr / eta
        coef = torch.tensor([a], dtype=r.dtype, device=r.device)
        ops.axpy(x, D[k:k + 1], coef, 1.0)
        ops.axpy(r, GD[k:k + 1], coef, -1.0)
        etas.append(eta)
        k += 1
        nr = float(allreduce_(ops.dots(r.reshape(1, -1), r), group, world)[0]) ** 0.5
        norms.append(nr / ny)
    converged = converged or nr <= rtol * ny
    return PCGResult(x, k, nr / ny if ny else 0.0, converged, norms)


def block_kron_terms(problem, J, device=0):
    """Kronecker terms (coefficients, full 1D factors on the GPU) of the diagonal
    Gram block (J, J), with the exact R6 cancellation of term pairs (the same
    rule the library applies internally), factors from gpfvm_factor_matrix."""
    from .api import factor_matrix
    blk = problem.blocks[J]
    d = problem.ndim
    coefs, facs = [], []
    cache = {}
    for a, t1 in enumerate(blk.terms):
        for b, t2 in enumerate(blk.terms):
            if t1.output != t2.output or b < a:
                continue
            c = t1.coeff * t2.coeff
            if a != b:
                if sum(t1.order[i] + t2.order[i] for i in range(d)) % 2:
                    continue
                c *= 2.0
            fs = []
            for i in range(d):
                key = (t1.output, i, t1.order[i], t2.order[i])
                if key not in cache:
                    k = problem.kernels[t1.output][i]
                    cache[key] = factor_matrix(k, blk.sites[i], t1.order[i], blk.sites[i], t2.order[i], device)
                fs.append(cache[key])
            coefs.append(c)
            facs.append(fs)
    return coefs, facs
