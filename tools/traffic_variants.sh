#!/bin/bash
# Per-kernel DRAM traffic and achieved GB/s of every variant's kernels at the bench size
# (config 2: n_local = 1e8, m = 20; single-pass ncu metrics), run under gpurun from the repo root:
#   bash tools/traffic_variants.sh  ->  gpurun_out/traffic_<variant>.csv
for v in icwy icwy_small cgs2 mgs; do
  base=$v; extra=""
  [ $v = icwy_small ] && { base=icwy; extra="--icwy-merged 2"; }   # ICWY_DELETE = 2 (SMALL)
  python bench.py --only-headline --no-e2e --no-cpu --steps 2 --warmup 3 --variant $base $extra > gpurun_out/plain_$v.json 2>&1 || { echo "plain $v failed"; continue; }
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/traffic_$v.csv python bench.py --only-headline --no-e2e --no-cpu --steps 2 --warmup 3 --variant $base $extra > gpurun_out/traffic_$v.log 2>&1
  echo "$v $?"
done
