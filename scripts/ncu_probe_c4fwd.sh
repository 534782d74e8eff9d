mkdir -p gpurun_out/r2/s4m
for sec in SpeedOfLight WarpStateStats SourceCounters InstructionStats MemoryWorkloadAnalysis Occupancy SchedulerStats ComputeWorkloadAnalysis LaunchStats PmSampling; do
  s=$(date +%s)
  timeout 120 ncu --section $sec --clock-control none -k "regex:k_fwd_tc" -c 1 -f -o /tmp/probe_$sec python scripts/prof_step.py C4 32768 1 > gpurun_out/r2/s4m/$sec.log 2>&1
  echo "$sec rc=$? $(( $(date +%s) - s ))s passes=$(grep -o '[0-9]* passes' gpurun_out/r2/s4m/$sec.log | head -1)" >> gpurun_out/r2/s4m/status.txt
done
cat gpurun_out/r2/s4m/status.txt
