#!/bin/bash
# per-config matvec plan profile (durations + DRAM bytes of every kernel of one matvec)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for cfg in "$@"; do
  set -- $cfg
  name=${cfg%%:*}; R=${cfg##*:}
  python tools/matvec_once.py $name $R > gpurun_out/mv_$name.log 2>&1 || { echo "plain run failed for $name"; continue; }
  ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/traffic_$name.csv \
      python tools/matvec_once.py $name $R > gpurun_out/ncu_$name.log 2>&1
done
