#!/bin/bash
# Same-box A/B of library variants: bash scripts/ab_run.sh TAG "VARIANTS" "KEYS" [N]
#   VARIANTS: names under paper_2409_14248_b200/_lib/variants (or "cur" = the in-tree library)
set -u
TAG=$1; VARS=$2; KEYS=$3; N=${4:-262144}
OUT=gpurun_out/ab/$TAG; mkdir -p $OUT
for rep in 1 2; do
  for v in $VARS; do
    if [ "$v" = cur ]; then lib=""; else lib=paper_2409_14248_b200/_lib/variants/$v/libhrkan.so; fi
    HRKAN_LIB=$lib timeout 600 python scripts/ab_time.py $KEYS --n $N --reps 5 >> $OUT/ab_$v.log 2>&1
  done
done
tail -n 40 $OUT/ab_*.log
