"""In-tree build of libgpfvm.so for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
def cutlass_include():
    """Vendored CUTLASS/CuTe header tree (flashinfer's copy in this image), or None."""
    import glob
    for pat in ["/opt/prime-rl/.venv/lib/python3*/site-packages/flashinfer/data/cutlass/include",
                os.path.join(os.path.dirname(os.__file__), "site-packages", "flashinfer", "data", "cutlass", "include")]:
        for d in glob.glob(pat):
            if os.path.exists(os.path.join(d, "cutlass", "gemm", "device", "gemm_batched.h")):
                return d
    return None


SOURCES = ["pool.cu", "assemble.cu", "gemm.cu", "kron.cu", "lowrank.cu", "bjfd.cu", "linalg.cu", "vecops.cu", "problem.cu", "solve.cu", "predict.cu", "extras.cu", "cutlass_gemm.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-shared",
         "-Xcompiler", "-fPIC"]


def build(force: bool = False, verbose: bool = False) -> str:
    out = os.path.join(HERE, "libgpfvm.so")
    srcs = [os.path.join(HERE, "csrc", s) for s in SOURCES]
    hdrs = [os.path.join(HERE, "csrc", h) for h in os.listdir(os.path.join(HERE, "csrc")) if h.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(os.path.dirname(HERE), "include", "gpfvm.h"))
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(f) <= t for f in srcs + hdrs):
            return out
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    extra = []
    inc = cutlass_include()
    if inc:
        extra = ["-DGPFVM_WITH_CUTLASS", "-I" + inc, "--expt-relaxed-constexpr", "-Xcudafe", "--diag_suppress=20013"]
    cmd = [nvcc] + FLAGS + extra + ["-o", out] + srcs
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
