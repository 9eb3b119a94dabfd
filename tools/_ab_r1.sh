# interleaved A/B, round-1 build vs current: headline (n = 1e8, DCGS-2, m = 20) and n = 1.5e6 MGS
for rep in 1 2 3; do
  for cfg in "AA_NOP=1" "AA_LIB=build/libaa_r1.so"; do
    env $cfg timeout 300 python bench.py --only-headline --no-e2e --no-cpu --steps 10 > gpurun_out/abr1.json 2>/dev/null
    python -c "import json; L=json.loads(open('gpurun_out/abr1.json').read().strip().splitlines()[-1]); d=L['detail']; print('1e8 dcgs2 rep $rep [$cfg] step %.1f us k1 %.1f k2 %.1f k4 %.1f clk %s' % (L['ms_per_step']*1e3, d['k1_ms']*1e3, d['k2_ms_per_step']*1e3, d['k4_ms']*1e3, L['clocks']['sm_mhz']))" >> gpurun_out/r02_ab_r1.txt 2>&1
    env $cfg timeout 300 python bench.py --only-headline --no-e2e --no-cpu --steps 10 --n-local 1.5e6 --variant mgs > gpurun_out/abr1.json 2>/dev/null
    python -c "import json; L=json.loads(open('gpurun_out/abr1.json').read().strip().splitlines()[-1]); d=L['detail']; print('1.5e6 mgs rep $rep [$cfg] step %.1f us k1 %.1f k2 %.1f k4 %.1f clk %s' % (L['ms_per_step']*1e3, d['k1_ms']*1e3, d['k2_ms_per_step']*1e3, d['k4_ms']*1e3, L['clocks']['sm_mhz']))" >> gpurun_out/r02_ab_r1.txt 2>&1
  done
done
