"""In-tree build of libgpfvm.so for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["pool.cu", "assemble.cu", "gemm.cu", "kron.cu", "lowrank.cu", "funcpass.cu", "bjfd.cu", "linalg.cu", "vecops.cu", "problem.cu", "solve.cu", "predict.cu", "extras.cu", "gemm_tma.cu", "shard.cu"]
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
    # one nvcc per translation unit, in parallel, then one link
    objdir = os.path.join(os.path.dirname(HERE), "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]
    jobs = []
    for src in srcs:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc] + cflags + ["-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd))
        jobs.append((obj, subprocess.Popen(cmd)))
    failed = [obj for obj, p in jobs if p.wait() != 0]
    if failed:
        raise RuntimeError("nvcc failed for " + ", ".join(os.path.basename(f) for f in failed))
    link = [nvcc] + FLAGS + ["-o", out] + [obj for obj, _ in jobs]
    if verbose:
        print(" ".join(link))
    subprocess.run(link, check=True)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
