# mid-n regression hunt: per-kernel split at n_local = 1e7 and 1.5e6 (round-1 build vs current,
# current with the early TMA issue off)
for n in 1e7 1.5e6; do for v in mgs dcgs2; do
  for cfg in "AA_LIB=build/libaa_r1.so" "AA_NOP=1" "AA_NO_EARLY_TMA=1"; do
    env $cfg timeout 300 python bench.py --only-headline --no-e2e --no-cpu --steps 10 --n-local $n --variant $v > gpurun_out/midn.json 2>/dev/null
    python -c "import json; L=json.loads(open('gpurun_out/midn.json').read().strip().splitlines()[-1]); d=L['detail']; print('n=$n $v [$cfg] step %.1f us k1 %.1f k2 %.1f k4 %.1f' % (L['ms_per_step']*1e3, d['k1_ms']*1e3, d['k2_ms_per_step']*1e3, d['k4_ms']*1e3))" >> gpurun_out/r02_midn.txt 2>&1
  done
done; done
