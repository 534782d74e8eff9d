#!/bin/bash
# Round-2 measurement session: bench lines, ncu captures (one GPU).  Usage: bash scripts/r2_measure.sh TAG ITEMS...
#   C3 / C4 / C5 / K6 ...   bench.py line (STEPS, WARMUP)
#   ncu_<cfg>               ncu --set full of the three tensor-core kernels (report kept in /tmp; raw CSV copied)
#   launches_<cfg>          ncu launch list (gpu__time_duration) of a short bench run
set -u
TAG=$1; shift
OUT=gpurun_out/r2/$TAG
mkdir -p $OUT
for c in "$@"; do
  case $c in
    ncu_*)
      k=${c#ncu_}
      timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_(fwd|wgrad|dgrad)_tc|k_split|k_last|k_fwd_first|k_wgrad_first" -c 24 -f -o /tmp/ncu_$k python scripts/prof_step.py $k ${NCU_N:-32768} 1 > $OUT/ncu_$k.log 2>&1
      ncu -i /tmp/ncu_$k.ncu-rep --page raw --csv > $OUT/ncu_${k}_raw.csv 2>/dev/null
      ncu -i /tmp/ncu_$k.ncu-rep --page details --csv > $OUT/ncu_${k}_details.csv 2>/dev/null
      ;;
    launches_*)
      k=${c#launches_}
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_$k.csv python bench.py --config $k --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --prof-steps 1 > $OUT/launches_$k.log 2>&1
      ;;
    *)
      timeout 1200 python bench.py --config $c --steps ${STEPS:-10} --warmup ${WARMUP:-3} > $OUT/bench_$c.json 2> $OUT/bench_$c.err
      ;;
  esac
done
du -sh $OUT
