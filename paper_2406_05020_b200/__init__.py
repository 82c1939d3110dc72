"""B200-native GP-FVM hot path (arxiv 2406.05020): FP64 CUDA kernels for sm_100a
behind the C ABI of include/gpfvm.h, with a thin ctypes binding.

    from paper_2406_05020_b200 import GpfvmProblem
    p = GpfvmProblem(problem)            # gpfvm_inputs.Problem description
    p.gpfvm_assemble_factors()
    y = p.gpfvm_gram_matvec(x)           # torch CUDA tensors (fp64)
    alpha, rep = p.gpfvm_solve(rhs)
    mean, var = p.gpfvm_predict(grid, alpha)
"""
from .api import GpfvmProblem, factor_matrix, launch_count, version  # noqa: F401
