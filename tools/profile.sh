#!/bin/bash
# Profiling pass for one round (run under gpurun from the repo root, 1 GPU):
#   bash tools/profile.sh <tag>
# 1. plain bench runs (each command exits 0 before any ncu run of it)
# 2. ncu launch list (gpu__time_duration) of the headline bench command
# 3. per-launch DRAM traffic (dram__bytes_read/write, single pass) at the full size
# 4. ncu --set full (source-level) of K1: DCGS-2 m = 20 at the bench's n_local = 1e8, and
#    the paper-faithful ICWY m = 50 (DMMA Gram) at n_local = 2e7
set -u
TAG=${1:-r02}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
H="python bench.py --only-headline --no-e2e --no-cpu --steps 3 --warmup 3"
S50="python bench.py --only-headline --no-e2e --no-cpu --n-local 2e7 --m 50 --variant icwy --steps 3 --warmup 3"
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > $OUT/gpu.txt 2>&1
$H > $OUT/plain.json 2> $OUT/plain.err && echo "plain ok" || { echo "plain FAILED"; exit 1; }
$S50 > $OUT/plain_icwy50.json 2> $OUT/plain_icwy50.err && echo "plain icwy50 ok" || { echo "plain icwy50 FAILED"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $H > $OUT/launches.log 2>&1
echo "launches $?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/traffic.csv $H > $OUT/traffic.log 2>&1
echo "traffic $?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:stream_kernel<.int.0," -s 22 -c 1 -o $OUT/k1_dcgs2 $H > $OUT/k1_dcgs2.log 2>&1
echo "k1_dcgs2 $?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:stream_kernel<.int.0," -s 52 -c 1 -o $OUT/k1_icwy50 $S50 > $OUT/k1_icwy50.log 2>&1
echo "k1_icwy50 $?"
