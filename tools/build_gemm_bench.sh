#!/bin/sh
# Builds tools/gemm_bench (library GEMM paths on the mode-product shapes).
set -e
cd "$(dirname "$0")/.."
C=paper_2406_05020_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/gemm_bench tools/gemm_bench.cu \
  $C/gemm.cu $C/gemm_tma.cu $C/pool.cu
