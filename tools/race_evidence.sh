#!/bin/bash
# Evidence for DESIGN.md 4.4 (run under gpurun): the two-stream reproducer built
# from the shipped gemm_tma.cu (with the proxy fence) and from a copy with the
# fence line removed, several CTAs per SM (-DGPFVM_TMA_SHARED_SMS); then the
# library's stress / repeat tools on every config.  Output: gpurun_out/race_evidence.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/nofence
C=paper_2406_05020_b200/csrc
OUT=gpurun_out/race_evidence.txt
: > $OUT
grep -v 'fence.proxy.async.shared::cta;' $C/gemm_tma.cu > /tmp/nofence/gemm_tma.cu
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DGPFVM_TMA_SHARED_SMS -I $C -I include"
$NV -o /tmp/race_fence tools/gemm_race.cu $C/gemm.cu $C/gemm_tma.cu $C/pool.cu || exit 1
$NV -o /tmp/race_nofence tools/gemm_race.cu $C/gemm.cu /tmp/nofence/gemm_tma.cu $C/pool.cu || exit 1
echo "# tools/gemm_race (mode 0: cp.async GEMM on the second stream), 400 repetitions per line" >> $OUT
for v in 1 6 7 8 9; do
  echo "variant $v without the fence: $(GPFVM_TMA_VARIANT=$v /tmp/race_nofence 0 400 | tail -1)" >> $OUT
  echo "variant $v with the fence:    $(GPFVM_TMA_VARIANT=$v /tmp/race_fence 0 400 | tail -1)" >> $OUT
done
echo "# library, shipped configuration: every call against the oracle's Kronecker matvec (1e-12 of max|ref|)" >> $OUT
python tools/stress_matvec.py config4:2:100 config3:2:50 config2:4:100 config1:128:100 >> $OUT 2>&1
echo "# library: bitwise repeats" >> $OUT
python tools/repeat_matvec.py config4:2:200 config3:2:100 config2:4:200 config1:32:200 >> $OUT 2>&1
cat $OUT
