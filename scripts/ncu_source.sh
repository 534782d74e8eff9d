#!/bin/bash
# Source-level (SASS) stall attribution of the tensor-core kernels of one workload:
#   bash scripts/ncu_source.sh TAG CFG [N]  -> gpurun_out/r2/TAG/src_<CFG>_<kernel>.csv (+ raw metrics)
set -u
TAG=$1; CFG=$2; N=${3:-32768}
OUT=gpurun_out/r2/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_(fwd|wgrad|dgrad)_tc" -c 3 -f -o /tmp/src_$CFG python scripts/prof_step.py $CFG $N 1 > $OUT/src_$CFG.log 2>&1
ncu -i /tmp/src_$CFG.ncu-rep --page raw --csv > $OUT/src_${CFG}_raw.csv 2>/dev/null
for k in fwd wgrad dgrad; do
  ncu -i /tmp/src_$CFG.ncu-rep --page source --csv --print-source cuda,sass -k "regex:k_${k}_tc" > $OUT/src_${CFG}_$k.csv 2>/dev/null
done
ls -la $OUT
