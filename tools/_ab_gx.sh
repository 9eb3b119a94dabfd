# K1 with the ICWY Gram: Delta f and f_i as Gram columns (default) vs the block multi-dot
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_config5.py tests/test_gpu_icwy_small.py tests/test_gpu_heat.py -q -x > gpurun_out/r02_gputest_gx.log 2>&1; echo rc=$? >> gpurun_out/r02_gputest_gx.log
for rep in 1 2; do
  for m in 5 10 20 50; do
    for md in 0 1; do
      AA_GRAM_MULTIDOT=$md timeout 300 python bench.py --steps 8 --warmup 3 --m $m --variant icwy --only-headline --no-e2e --no-cpu > gpurun_out/abgx.json 2>/dev/null
      python -c "import json; L=json.loads(open('gpurun_out/abgx.json').read().strip().splitlines()[-1]); r=L['roofline']; d=L['detail']; print('rep $rep icwy m=$m multidot=$md step %.3f ms k1 %.3f frac %.3f step_frac %.3f clk %s' % (L['ms_per_step'], r['k1_ms'], r['frac'], r['step_frac'], L['clocks']['sm_mhz']))" >> gpurun_out/r02_ab_gx.txt 2>&1
    done
  done
done
