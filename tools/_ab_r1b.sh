for rep in 1 2; do
  for cfg in "AA_NOP=1" "AA_LIB=build/libaa_r1.so"; do
    for nv in "1.5e6 mgs" "1.5e6 dcgs2" "1e5 dcgs2" "1e7 mgs"; do set -- $nv
    env $cfg timeout 300 python bench.py --only-headline --no-e2e --no-cpu --steps 10 --n-local $1 --variant $2 > gpurun_out/abr1.json 2>/dev/null
    python -c "import json; L=json.loads(open('gpurun_out/abr1.json').read().strip().splitlines()[-1]); d=L['detail']; print('$1 $2 rep $rep [$cfg] step %.1f us k1 %.1f k2 %.1f k4 %.1f clk %s' % (L['ms_per_step']*1e3, d['k1_ms']*1e3, d['k2_ms_per_step']*1e3, d['k4_ms']*1e3, L['clocks']['sm_mhz']))" >> gpurun_out/r02_ab_r1b.txt 2>&1
    done
  done
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02_gputest10.log 2>&1; echo rc=$? >> gpurun_out/r02_gputest10.log
