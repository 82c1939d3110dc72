#!/bin/bash
# GPU-box profiling pass of the final round-2 plans (run under gpurun).  Every
# ncu command runs after the same command exited 0 without ncu.
#  1. per-config matvec: every kernel's duration and DRAM bytes (-> profiles/r02_plan_*.txt, r02_traffic.json)
#  2. ncu launch list of the default bench command (-> profiles/r02j_bench_launches.txt)
#  3. ncu --set full: config-1 matvec kernels (parity transforms, functional pass, the two GEMMs),
#     config-3 3D parity kernels (fwd3, inv3 with fused mode updates, stage GEMMs)
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/profile_plans.sh config1:128 config2:4 config3:4 config4:4
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-sharded --no-e2e > gpurun_out/launch_bench.json 2> gpurun_out/launch_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-sharded --no-e2e > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"dgemm_tma_kernel|parity|func_pass" -c 6 \
    -o gpurun_out/r02j_config1_full python tools/matvec_once.py config1 128 > gpurun_out/ncu_full1.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"parity" -c 2 \
    -o gpurun_out/r02j_config3_parity_full python tools/matvec_once.py config3 4 > gpurun_out/ncu_full3.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"dgemm_tma_kernel" -c 40 \
    -o gpurun_out/r02j_config3_gemm_full python tools/matvec_once.py config3 4 > gpurun_out/ncu_full3g.log 2>&1
