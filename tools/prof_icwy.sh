mkdir -p gpurun_out/prof_icwy
S="python bench.py --only-headline --no-e2e --no-cpu --n-local 2e7 --steps 2 --warmup 3 --variant icwy --m 50"
$S > gpurun_out/prof_icwy/plain.json 2>&1
echo plain $?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:stream_kernel<.int.0," -s 52 -c 1 -o gpurun_out/prof_icwy/k1_icwy_m50 $S > gpurun_out/prof_icwy/ncu.log 2>&1
echo ncu $?
