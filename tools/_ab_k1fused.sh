# A/B of the fused K1 row-pass variants (build/libaa_g*_p*.so: guarded dots / running pointers)
for r in 1 2; do
for v in g0_p1 g1_p1 g1_p0; do
  for m in 20 10; do
    AA_LIB=build/libaa_$v.so timeout 300 python bench.py --steps 10 --m $m --only-headline --no-e2e --no-cpu > gpurun_out/abf_${v}_m${m}_$r.json 2>/dev/null
    python -c "import json; L=json.loads(open('gpurun_out/abf_${v}_m${m}_$r.json').read().strip().splitlines()[-1]); r=L['roofline']; print('$v m=$m run $r step %.3f k1 %.3f frac %.3f' % (L['ms_per_step'], r['k1_ms'], r['frac']))" >> gpurun_out/r02_ab_fused.txt 2>&1
  done
done
done
python tools/timeline_probe.py 1000 20 dcgs2 > gpurun_out/r02_timeline4.txt 2>&1
python tools/step_latency.py 1000,100000 20 > gpurun_out/r02_step_latency4.txt 2>&1
