for rep in 1 2; do
  for cfg in "AA_NOP=1" "AA_K1_NOFUSE=1"; do
    for nv in "1e7 20" "1e8 20" "1e7 10" "1.5e6 20"; do set -- $nv
    env $cfg timeout 300 python bench.py --only-headline --no-e2e --no-cpu --steps 10 --n-local $1 --m $2 > gpurun_out/abf.json 2>/dev/null
    python -c "import json; L=json.loads(open('gpurun_out/abf.json').read().strip().splitlines()[-1]); d=L['detail']; print('n=$1 m=$2 rep $rep [$cfg] step %.1f us k1 %.1f k2 %.1f k4 %.1f clk %s' % (L['ms_per_step']*1e3, d['k1_ms']*1e3, d['k2_ms_per_step']*1e3, d['k4_ms']*1e3, L['clocks']['sm_mhz']))" >> gpurun_out/r02_ab_fuse.txt 2>&1
    done
  done
done
