#!/bin/bash
# GPU-box profiling pass of round 2 (run under gpurun): per-config matvec DRAM
# traffic (tools/ncu_traffic.py -> profiles/r02_traffic.json) and the ncu
# launch list of one bench step.  Every ncu command runs after the same
# command exited 0 without ncu.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for cfg in "config1 128" "config2 4" "config3 4" "config4 4"; do
  set -- $cfg
  python tools/matvec_once.py $1 $2 > gpurun_out/mv_$1.log 2>&1
  ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/traffic_$1.csv \
      python tools/matvec_once.py $1 $2 > gpurun_out/ncu_$1.log 2>&1
  python tools/ncu_traffic.py $1 $2 gpurun_out/traffic_$1.csv
done
cp profiles/r02_traffic.json gpurun_out/r02_traffic.json
