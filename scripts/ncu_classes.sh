#!/bin/bash
# ncu --set full of one interior-pass launch of every kernel class of a config, one class per ncu invocation
# (a whole-step kernel-replay capture of C4 once stalled in ncu's replay of k_fwd_tc; per-class captures never did).
#   bash scripts/ncu_classes.sh TAG CFG [N=262144]   ->  gpurun_out/r2/TAG/ncu_CFG_<class>_raw.csv (summarise with scripts/ncu_summary.py a,b,c ...)
set -u
TAG=$1; CFG=$2; N=${3:-262144}
OUT=gpurun_out/r2/$TAG; mkdir -p $OUT
: > $OUT/ncu_${CFG}_status.txt
LIST=""
for k in k_fwd_tc k_wgrad_tc k_dgrad_tc k_last k_fwd_first k_wgrad_first k_split; do
  LIBV=""
  # ncu's kernel replay of C4's k_fwd_tc stalls ("launching the workload is taking more time than expected") on the
  # product build; the hang-guard build (bounded mbarrier waits, trap on expiry) profiles it without a trap
  if [ "$CFG $k" = "C4 k_fwd_tc" ] && [ -f paper_2409_14248_b200/_lib/variants/hg/libhrkan.so ]; then LIBV=paper_2409_14248_b200/_lib/variants/hg/libhrkan.so; fi
  HRKAN_LIB=$LIBV timeout 400 ncu --set full --clock-control none -k "regex:$k" -c 1 -f -o /tmp/ncu_${CFG}_$k python scripts/prof_step.py $CFG $N 1 > $OUT/ncu_${CFG}_$k.log 2>&1
  echo "$k rc=$? lib=${LIBV:-product}" >> $OUT/ncu_${CFG}_status.txt
  [ -f /tmp/ncu_${CFG}_$k.ncu-rep ] || continue
  ncu -i /tmp/ncu_${CFG}_$k.ncu-rep --page raw --csv > $OUT/ncu_${CFG}_${k}_raw.csv 2>/dev/null
  rm -f /tmp/ncu_${CFG}_$k.ncu-rep
done
cat $OUT/ncu_${CFG}_status.txt
