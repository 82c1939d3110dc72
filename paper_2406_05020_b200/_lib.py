"""ctypes declarations of include/gpfvm.h (argument marshalling only).

The shared library ``libgpfvm.so`` is built in-tree by ``build.py`` /
``__graft_entry__.build()``.  Loading fails loudly when it is missing: there
is no CPU fallback for any GP-FVM computation in this package.
"""
from __future__ import annotations

import ctypes as C
import os

MAX_DIMS = 4
MAX_TERMS = 16

SITE_POINT = 0
SITE_INTERVAL = 1
PRECOND_NONE, PRECOND_BLOCK_FD = 0, 2
COV_ITERGP, COV_PRECOND = 0, 1

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgpfvm.so")


class Kernel1D(C.Structure):
    _fields_ = [("q", C.c_int), ("lengthscale", C.c_double), ("variance", C.c_double)]


class Sites1D(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int), ("lo", C.POINTER(C.c_double)), ("hi", C.POINTER(C.c_double))]


class Term(C.Structure):
    _fields_ = [("coeff", C.c_double), ("order", C.c_int * MAX_DIMS), ("output", C.c_int)]


class Block(C.Structure):
    _fields_ = [("sites", Sites1D * MAX_DIMS), ("n_terms", C.c_int), ("terms", Term * MAX_TERMS),
                ("noise", C.c_double), ("deflate", C.c_int)]


class ProblemDesc(C.Structure):
    _fields_ = [("ndim", C.c_int), ("n_outputs", C.c_int), ("kernels", C.POINTER(Kernel1D)),
                ("n_blocks", C.c_int), ("blocks", C.POINTER(Block))]


class SolveOpts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iter", C.c_int), ("precond", C.c_int), ("reorth_window", C.c_int),
                ("keep_actions", C.c_int)]


class SolveReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("rel_residual", C.c_double),
                ("true_rel_residual", C.c_double), ("precond_shift", C.c_double),
                ("setup_ms", C.c_double), ("iterate_ms", C.c_double), ("breakdown", C.c_int)]


class Grid(C.Structure):
    _fields_ = [("n", C.c_int * MAX_DIMS), ("pts", C.POINTER(C.c_double) * MAX_DIMS), ("output", C.c_int)]


EXPORTS = {
    "gpfvm_last_error": (C.c_char_p, []),
    "gpfvm_version": (C.c_char_p, []),
    "gpfvm_problem_create": (C.c_int, [C.POINTER(ProblemDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "gpfvm_problem_destroy": (C.c_int, [C.c_void_p]),
    "gpfvm_problem_size": (C.c_int64, [C.c_void_p]),
    "gpfvm_assemble_factors": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gpfvm_factor_matrix": (C.c_int, [C.POINTER(Kernel1D), C.POINTER(Sites1D), C.c_int, C.POINTER(Sites1D),
                                      C.c_int, C.c_void_p, C.c_int64, C.c_void_p]),
    "gpfvm_gram_matvec": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_void_p]),
    "gpfvm_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(SolveOpts),
                              C.POINTER(SolveReport), C.c_void_p]),
    "gpfvm_solve_many": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.POINTER(SolveOpts),
                                   C.POINTER(SolveReport), C.c_void_p]),
    "gpfvm_predict": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                C.c_void_p]),
    "gpfvm_kron_matvec": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_void_p), C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int,
                                    C.c_double, C.c_void_p]),
    "gpfvm_probe_fp64_peak": (C.c_int, [C.POINTER(C.c_double), C.c_void_p]),
    "gpfvm_gemm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                             C.c_double, C.c_void_p, C.c_int64, C.c_void_p]),
    "gpfvm_permute": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    "gpfvm_sygv": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_dot_many": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]),
    "gpfvm_axpy_many": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_double, C.c_int64, C.c_int,
                                  C.c_void_p]),
    "gpfvm_fd_setup": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                 C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_vmul": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "gpfvm_shard_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.c_void_p]),
    "gpfvm_shard_destroy": (C.c_int, [C.c_void_p]),
    "gpfvm_shard_local_size": (C.c_int64, [C.c_void_p]),
    "gpfvm_shard_layout": (C.c_int, [C.c_void_p] + [C.POINTER(C.c_int64)] * 4),
    "gpfvm_shard_counts": (C.c_int, [C.c_void_p, C.c_int] + [C.POINTER(C.c_int64)] * 4),
    "gpfvm_shard_apply_begin": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_shard_apply_mid": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_shard_apply_end": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_shard_precond_scale": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_shard_plan_counts": (C.c_int, [C.c_void_p, C.c_int, C.c_int] + [C.POINTER(C.c_int64)] * 5),
    "gpfvm_shard_predict_mean": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_shard_gather_local": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_iter_init": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]),
    "gpfvm_iter_coefs": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_iter_update_local": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                          C.c_void_p, C.c_void_p]),
    "gpfvm_iter_update_final": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_iter_step_local": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                        C.c_void_p, C.c_void_p]),
    "gpfvm_iter_step_final": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "gpfvm_launch_count": (C.c_int64, []),
    "gpfvm_matvec_flops": (C.c_double, [C.c_void_p]),
    "gpfvm_matvec_flops_unsplit": (C.c_double, [C.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libgpfvm.so and declare every exported symbol; raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libgpfvm.so not built ({path}); run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class GpfvmError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc != 0:
        msg = load().gpfvm_last_error().decode(errors="replace")
        raise GpfvmError(f"gpfvm error {rc}: {msg}")
