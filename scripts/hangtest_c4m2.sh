# Repeats a short full-size C4 bench at HR order m (default 2) under a 90 s limit: a GPU-side hang shows as rc=124.
# (Round 2: a support-mask extension of the packed-pair paths to m = 2, 3 hung 2 runs of 4 here and was reverted.)
mkdir -p gpurun_out/r2/hangtest
for rep in 1 2 3; do
  s=$(date +%s)
  PYTHONFAULTHANDLER=1 timeout -s ABRT 90 python bench.py --config C4 --m ${1:-2} --steps 3 --warmup 3 --no-e2e --cpu-seconds 3 > gpurun_out/r2/hangtest/cur_$rep.json 2> gpurun_out/r2/hangtest/cur_$rep.err
  echo "cur rep$rep rc=$? $(( $(date +%s) - s ))s" | tee -a gpurun_out/r2/hangtest/status.txt
done
