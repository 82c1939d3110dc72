#!/bin/bash
# GPU-box profiling pass, round 2 final plans (run under gpurun): per-config
# matvec DRAM traffic and per-kernel plan summaries, the ncu launch list of the
# default bench command, and ncu --set full of the config-1 parity-split GEMMs.
# Every ncu command runs after the same command exited 0 without ncu.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/profile_r02.sh
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launch_bench.json 2> gpurun_out/launch_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-sharded --no-e2e > gpurun_out/ncu_bench.log 2>&1
python tools/matvec_once.py config1 128 > gpurun_out/mv_full_plain.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"dgemm_tma_kernel|parity" -c 4 \
    -o gpurun_out/r02h_matvec_parity_full python tools/matvec_once.py config1 128 > gpurun_out/ncu_full.log 2>&1
