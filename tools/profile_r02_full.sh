#!/bin/bash
# ncu --set full of the config-1 matvec's two mode-product GEMMs (the dominant
# kernels), after the same command exited 0 without ncu.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/matvec_once.py config1 128 > gpurun_out/mv_full_plain.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:dgemm_tma_kernel -c 2 \
    -o gpurun_out/r02_matvec_tma_full python tools/matvec_once.py config1 128 > gpurun_out/ncu_full.log 2>&1
