# K1 tile / stage sweep (AA_TILE override "op:rows:stages", op 0 = K1), DCGS-2 config 2
for m in 10 20; do
  for t in "" "0:512:2" "0:512:3" "0:256:3" "0:256:4" "0:1024:2"; do
    AA_TILE="$t" timeout 300 python bench.py --steps 10 --m $m --only-headline --no-e2e --no-cpu > gpurun_out/tile_m${m}_${t//:/_}.json 2>/dev/null
    python -c "import json,sys; L=json.loads(open('gpurun_out/tile_m${m}_${t//:/_}.json').read().strip().splitlines()[-1]); r=L['roofline']; print('m=$m tile=[$t] step %.3f ms k1 %.3f ms frac %.3f' % (L['ms_per_step'], r['k1_ms'], r['frac']))" >> gpurun_out/r02_k1_tiles.txt 2>&1
  done
done
