#!/bin/bash
# Profiling pass for one round (run under gpurun from the repo root):
#   bash tools/profile.sh <tag>
# 1. plain bench run (must exit 0 before any ncu run)
# 2. ncu launch list (gpu__time_duration) of the headline bench command
# 3. per-launch DRAM traffic (dram__bytes_read/write, single pass) at the full size
# 4. ncu --set full of K1 (DCGS-2 and ICWY) at n_local = 2e7 (same per-tile behaviour)
set -u
TAG=${1:-r01}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
H="python bench.py --only-headline --no-e2e --no-cpu --steps 3 --warmup 3"
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > $OUT/gpu.txt 2>&1
$H > $OUT/plain.json 2> $OUT/plain.err
echo "plain $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $H > $OUT/launches.log 2>&1
echo "launches $?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/traffic.csv $H > $OUT/traffic.log 2>&1
echo "traffic $?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/traffic_icwy.csv $H --variant icwy > $OUT/traffic_icwy.log 2>&1
echo "traffic_icwy $?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/traffic_cgs2.csv $H --variant cgs2 > $OUT/traffic_cgs2.log 2>&1
echo "traffic_cgs2 $?"
S="python bench.py --only-headline --no-e2e --no-cpu --n-local 2e7 --steps 3 --warmup 3"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:stream_kernel<.int.0," -s 22 -c 1 -o $OUT/k1_dcgs2 $S > $OUT/k1_dcgs2.log 2>&1
echo "k1_dcgs2 $?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:stream_kernel<.int.0," -s 22 -c 1 -o $OUT/k1_icwy $S --variant icwy > $OUT/k1_icwy.log 2>&1
echo "k1_icwy $?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:stream_kernel<.int.[34]," -s 44 -c 2 -o $OUT/k2_cgs2 $S --variant cgs2 > $OUT/k2_cgs2.log 2>&1
echo "k2_cgs2 $?"
