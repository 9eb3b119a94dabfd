# K1 form: auto (timed at aa_init) vs forced fused / split, headline configuration
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_breakdown.py -q -x > gpurun_out/r02_gputest11.log 2>&1; echo rc=$? >> gpurun_out/r02_gputest11.log
for rep in 1 2; do
  for cfg in "AA_NOP=1" "AA_K1_FORM=fused" "AA_K1_FORM=split"; do
    env $cfg timeout 300 python bench.py --only-headline --no-e2e --no-cpu --steps 20 --warmup 5 > gpurun_out/abform.json 2>/dev/null
    python -c "import json; L=json.loads(open('gpurun_out/abform.json').read().strip().splitlines()[-1]); d=L['detail']; print('rep $rep [$cfg] step %.1f us k1 %.1f k2 %.1f k4 %.1f clk %s %s' % (L['ms_per_step']*1e3, d['k1_ms']*1e3, d['k2_ms_per_step']*1e3, d['k4_ms']*1e3, L['clocks']['sm_mhz'], L['clocks']['reasons']))" >> gpurun_out/r02_ab_form.txt 2>&1
  done
done
