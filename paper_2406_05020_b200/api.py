"""Thin Python binding of the C ABI (include/gpfvm.h): argument marshalling only.

Every GP-FVM computation runs inside libgpfvm.so.  Arrays may be torch CUDA
tensors (device pointers, the fast path; the current torch stream is passed
to the library) or numpy arrays (host pointers; the library stages them).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from . import _lib as L

try:  # torch is plumbing only (device memory / streams)
    import torch
except Exception:  # pragma: no cover
    torch = None


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _stream_of(x) -> C.c_void_p:
    if _is_torch(x) and x.is_cuda:
        return C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
    return C.c_void_p(0)


def _ptr(x, min_numel: int = 0, name: str = "array"):
    """Raw pointer of an fp64 C-contiguous torch tensor or numpy array holding
    at least min_numel elements (the library reads/writes through it)."""
    if _is_torch(x):
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError(f"{name}: fp64 contiguous tensors only")
        if x.numel() < min_numel:
            raise ValueError(f"{name}: {x.numel()} elements, need {min_numel}")
        return C.c_void_p(x.data_ptr())
    if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags["C_CONTIGUOUS"]):
        raise ValueError(f"{name}: fp64 C-contiguous numpy arrays only")
    if x.size < min_numel:
        raise ValueError(f"{name}: {x.size} elements, need {min_numel}")
    return C.c_void_p(x.ctypes.data)


def version() -> str:
    return L.load().gpfvm_version().decode()


def launch_count() -> int:
    return int(L.load().gpfvm_launch_count())


def _sites(s, keep):
    lo = np.ascontiguousarray(s.lo, dtype=np.float64)
    hi = np.ascontiguousarray(s.hi, dtype=np.float64)
    keep += [lo, hi]
    return L.Sites1D(int(s.kind), int(lo.shape[0]), _dptr(lo), _dptr(hi))


def factor_matrix(kernel, left, m_left: int, right, m_right: int, device: int = 0):
    """gpfvm_factor_matrix into a new torch CUDA tensor (left.n x right.n)."""
    lib = L.load()
    keep = []
    k = L.Kernel1D(int(kernel.q), float(kernel.lengthscale), float(kernel.variance))
    out = torch.empty((left.n, right.n), dtype=torch.float64, device=f"cuda:{device}")
    sl, sr = _sites(left, keep), _sites(right, keep)
    L.check(lib.gpfvm_factor_matrix(C.byref(k), C.byref(sl), int(m_left), C.byref(sr), int(m_right),
                                    C.c_void_p(out.data_ptr()), right.n, _stream_of(out)))
    return out


class GpfvmProblem:
    """Owns one gpfvm_problem handle built from a gpfvm_inputs.Problem."""

    def __init__(self, problem, device: int = 0):
        self.lib = L.load()
        self.problem = problem
        self.device = device
        keep = []
        d = problem.ndim
        kern = (L.Kernel1D * (problem.n_outputs * d))()
        for o in range(problem.n_outputs):
            for i in range(d):
                kk = problem.kernels[o][i]
                kern[o * d + i] = L.Kernel1D(int(kk.q), float(kk.lengthscale), float(kk.variance))
        blocks = (L.Block * len(problem.blocks))()
        for b, blk in enumerate(problem.blocks):
            B = blocks[b]
            for i in range(d):
                B.sites[i] = _sites(blk.sites[i], keep)
            B.n_terms = len(blk.terms)
            for t, term in enumerate(blk.terms):
                B.terms[t].coeff = float(term.coeff)
                for i in range(d):
                    B.terms[t].order[i] = int(term.order[i])
                B.terms[t].output = int(term.output)
            B.noise = float(blk.noise)
            B.deflate = int(bool(blk.deflate))
        desc = L.ProblemDesc(d, problem.n_outputs, kern, len(problem.blocks), blocks)
        h = C.c_void_p()
        L.check(self.lib.gpfvm_problem_create(C.byref(desc), int(device), C.byref(h)))
        self.handle = h
        self.N = int(self.lib.gpfvm_problem_size(h))

    def close(self):
        if getattr(self, "handle", None):
            self.lib.gpfvm_problem_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- §8 row 1
    def gpfvm_assemble_factors(self, stream: Optional[int] = None):
        s = C.c_void_p(stream if stream is not None else
                       (torch.cuda.current_stream(self.device).cuda_stream if torch is not None else 0))
        L.check(self.lib.gpfvm_assemble_factors(self.handle, s))

    # ---- §8 row 2
    def gpfvm_gram_matvec(self, x, out=None):
        two_d = x.ndim == 2
        nrhs = x.shape[0] if two_d else 1
        if out is None:
            out = torch.empty_like(x) if _is_torch(x) else np.empty_like(x)
        if (x.shape[-1] if x.ndim else 0) != self.N:
            raise ValueError(f"x: last dimension {x.shape[-1] if x.ndim else 0}, expected N = {self.N}")
        L.check(self.lib.gpfvm_gram_matvec(self.handle, _ptr(x, nrhs * self.N, "x"), _ptr(out, nrhs * self.N, "out"),
                                           int(nrhs), int(self.N), _stream_of(x)))
        return out

    # ---- §8 row 3
    def gpfvm_solve(self, y, rtol: float = 1e-8, max_iter: int = 1000, precond: int = L.PRECOND_BLOCK_FD,
                    out=None, reorth_window: int = 0, keep_actions: bool = True) -> Tuple[object, dict]:
        if out is None:
            out = torch.empty_like(y) if _is_torch(y) else np.empty_like(y)
        opts = L.SolveOpts(float(rtol), int(max_iter), int(precond), int(reorth_window), int(bool(keep_actions)))
        if y.ndim == 2:  # several right-hand sides (rows): gpfvm_solve_many, device tensors
            nrhs = int(y.shape[0])
            if not (_is_torch(y) and y.is_cuda and _is_torch(out) and out.is_cuda):
                raise ValueError("several right-hand sides: CUDA tensors only")
            if y.shape[-1] != self.N:
                raise ValueError(f"y: last dimension {y.shape[-1]}, expected N = {self.N}")
            reps = (L.SolveReport * nrhs)()
            L.check(self.lib.gpfvm_solve_many(self.handle, _ptr(y, nrhs * self.N, "y"), _ptr(out, nrhs * self.N, "out"),
                                              nrhs, int(self.N), C.byref(opts), reps, _stream_of(y)))
            return out, [{f: getattr(r, f) for f, _ in L.SolveReport._fields_} for r in reps]
        rep = L.SolveReport()
        L.check(self.lib.gpfvm_solve(self.handle, _ptr(y, self.N, "y"), _ptr(out, self.N, "out"), C.byref(opts),
                                     C.byref(rep), _stream_of(y)))
        return out, {f: getattr(rep, f) for f, _ in L.SolveReport._fields_}

    # ---- §8 row 4
    def gpfvm_predict(self, grid, alpha, cov_mode: int = L.COV_ITERGP, want_mean: bool = True,
                      want_var: bool = True, mean=None, var=None):
        d = self.problem.ndim
        pts = [np.ascontiguousarray(p, dtype=np.float64) for p in grid.points]
        g = L.Grid()
        for i in range(d):
            g.n[i] = int(pts[i].shape[0])
            g.pts[i] = _dptr(pts[i])
        g.output = int(grid.output)
        ng = int(np.prod([p.shape[0] for p in pts]))
        if _is_torch(alpha):
            if want_mean and mean is None:
                mean = torch.empty(ng, dtype=torch.float64, device=alpha.device)
            if want_var and var is None:
                var = torch.empty(ng, dtype=torch.float64, device=alpha.device)
        else:
            if want_mean and mean is None:
                mean = np.empty(ng)
            if want_var and var is None:
                var = np.empty(ng)
        L.check(self.lib.gpfvm_predict(self.handle, C.byref(g), _ptr(alpha, self.N, "alpha"),
                                       _ptr(mean, ng, "mean") if want_mean else C.c_void_p(0),
                                       _ptr(var, ng, "var") if want_var else C.c_void_p(0), int(cov_mode),
                                       _stream_of(alpha)))
        return mean, var

    def matvec_flops(self) -> float:
        return float(self.lib.gpfvm_matvec_flops(self.handle))

    def matvec_flops_unsplit(self) -> float:
        return float(self.lib.gpfvm_matvec_flops_unsplit(self.handle))
