#!/bin/bash
# Source-level (SASS) ncu capture of the kernels matching a regex in one loss+grad step of a workload:
#   bash scripts/ncu_ksrc.sh TAG CFG REGEX [N]  -> gpurun_out/r2/TAG/ksrc_<CFG>_raw.csv, ksrc_<CFG>_<i>.csv
set -u
TAG=$1; CFG=$2; RX=$3; N=${4:-32768}
OUT=gpurun_out/r2/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$RX" -c 4 -f -o /tmp/ksrc_$CFG python scripts/prof_step.py $CFG $N 1 > $OUT/ksrc_$CFG.log 2>&1
ncu -i /tmp/ksrc_$CFG.ncu-rep --page raw --csv > $OUT/ksrc_${CFG}_raw.csv 2>/dev/null
ncu -i /tmp/ksrc_$CFG.ncu-rep --page details --csv > $OUT/ksrc_${CFG}_details.csv 2>/dev/null
for k in $(ncu -i /tmp/ksrc_$CFG.ncu-rep --page raw --csv 2>/dev/null | tail -n +3 | cut -d, -f5 | grep -o 'k_[a-z_0-9]*' | sort -u); do
  ncu -i /tmp/ksrc_$CFG.ncu-rep --page source --csv --print-source sass -k "regex:$k" > $OUT/ksrc_${CFG}_$k.csv 2>/dev/null
done
ls -la $OUT
