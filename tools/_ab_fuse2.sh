# fused vs split K1 at the headline configuration, interleaved, several reps (box-to-box the
# fused K1 has measured 6.0-6.5 ms)
for rep in 1 2 3; do
  for cfg in "AA_NOP=1" "AA_K1_NOFUSE=1"; do
    env $cfg timeout 300 python bench.py --only-headline --no-e2e --no-cpu --steps 20 --warmup 5 > gpurun_out/abf2.json 2>/dev/null
    python -c "import json; L=json.loads(open('gpurun_out/abf2.json').read().strip().splitlines()[-1]); d=L['detail']; print('rep $rep [$cfg] step %.1f us k1 %.1f k2 %.1f k4 %.1f clk %s %s' % (L['ms_per_step']*1e3, d['k1_ms']*1e3, d['k2_ms_per_step']*1e3, d['k4_ms']*1e3, L['clocks']['sm_mhz'], L['clocks']['reasons']))" >> gpurun_out/r02_ab_fuse2.txt 2>&1
  done
done
nvidia-smi -q -d POWER,CLOCK > gpurun_out/r02_smi_q.txt 2>&1
