#!/bin/bash
# ncu --set full of the C4 tensor-core kernels with application replay (kernel replay of k_fwd_tc hung under ncu)
set -u
TAG=$1; OUT=gpurun_out/r2/$TAG; mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --replay-mode application -k "regex:k_(fwd|wgrad|dgrad)_tc|k_split|k_last|k_fwd_first|k_wgrad_first" -c 12 -f -o /tmp/ncu_C4 python scripts/prof_step.py C4 32768 1 > $OUT/ncu_C4.log 2>&1
ncu -i /tmp/ncu_C4.ncu-rep --page raw --csv > $OUT/ncu_C4_raw.csv 2>/dev/null
ncu -i /tmp/ncu_C4.ncu-rep --page details --csv > $OUT/ncu_C4_details.csv 2>/dev/null
tail -3 $OUT/ncu_C4.log
