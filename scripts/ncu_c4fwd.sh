#!/bin/bash
# ncu --set full (kernel replay) of C4's tensor-core kernels, one kernel class at a time, on the hang-guard build
# (a barrier-phase hang under replay traps with a message instead of hanging)
set -u
TAG=$1; OUT=gpurun_out/r2/$TAG; mkdir -p $OUT
for k in wgrad dgrad fwd; do
  HRKAN_LIB=paper_2409_14248_b200/_lib/variants/hg/libhrkan.so timeout 600 ncu --set full --clock-control none -k "regex:k_${k}_tc" -c 1 -f -o /tmp/ncu_C4_$k python scripts/prof_step.py C4 32768 1 > $OUT/ncu_C4_$k.log 2>&1
  echo "$k rc=$?" >> $OUT/ncu_C4_status.txt
  ncu -i /tmp/ncu_C4_$k.ncu-rep --page raw --csv > $OUT/ncu_C4_${k}_raw.csv 2>/dev/null
done
cat $OUT/ncu_C4_status.txt
