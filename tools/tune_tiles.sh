#!/bin/bash
# Per-op tile sweep (run under gpurun): prints k1/k2/k4 ms per configuration.
#   bash tools/tune_tiles.sh <variant> "<AA_TILE cfg> ..." [m]
V=${1:-dcgs2}; CFGS=${2:-""}; M=${3:-20}
for cfg in "" $CFGS; do
  out=$(AA_TILE="$cfg" python bench.py --only-headline --no-e2e --no-cpu --steps 10 --warmup 3 --variant $V --m $M 2>/dev/null)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); t=d['detail']
print('%-22s step %7.3f  k1 %6.3f  k2 %6.3f  k4 %6.3f  frac %.3f' % (sys.argv[2] or 'default', t['ms_per_step'], t['k1_ms'], t['k2_ms_per_step'], t['k4_ms'], d['roofline']['step_frac']))" "$out" "$cfg"
done
