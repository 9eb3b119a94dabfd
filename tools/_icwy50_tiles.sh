# the paper-faithful ICWY K1 (DMMA Gram) at m = 50: tile / stage sweep through AA_TILE
for t in "" "0:124:4" "0:124:3" "0:60:6" "0:252:2"; do
  AA_TILE="$t" timeout 300 python bench.py --only-headline --no-e2e --no-cpu --steps 5 --m 50 --variant icwy > gpurun_out/icwy50.json 2>/dev/null
  python -c "import json; L=json.loads(open('gpurun_out/icwy50.json').read().strip().splitlines()[-1]); r=L['roofline']; d=L['detail']; print('icwy m=50 tile=[$t] step %.2f ms k1 %.2f ms frac %.3f step_frac %.3f' % (L['ms_per_step'], r['k1_ms'], r['frac'], r['step_frac']))" >> gpurun_out/r02_icwy50_tiles.txt 2>&1
done
