"""Print the key numbers of bench.py JSON lines: python tools/bench_summary.py file.json ..."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path).read().strip().splitlines():
        try:
            l = json.loads(line)
        except ValueError:
            continue
        d = l.get("detail", {})
        roof = l.get("roofline") or {}
        print(f"{path}: {l.get('config', {}).get('variant', '?')} n_gpus={l.get('n_gpus')} "
              f"{l.get('value', 0):.1f} {l.get('unit', '')} step_frac={roof.get('step_frac', 0):.3f} "
              f"k1_frac={roof.get('frac', 0):.3f} k1={d.get('k1_ms', 0):.3f} k2/step={d.get('k2_ms_per_step', 0):.3f} "
              f"k4={d.get('k4_ms', 0):.3f} ar/step={d.get('allreduce_ms_per_step', 0):.3f} ms")
        sw = l.get("sweep") or {}
        if sw:
            names = sorted({k.rsplit("_m", 1)[0] for k in sw})
            for v in names:
                print(f"    sweep {v:11s}", " ".join(
                    f"m{m}: {sw[f'{v}_m{m}']['step_hbm_frac'] * 100:5.1f}%" for m in (5, 10, 20, 50) if f"{v}_m{m}" in sw))
        for k, v in (l.get("variants") or {}).items():
            print(f"    {k:11s} {v['us_per_iter']:10.1f} us  frac {v['step_hbm_frac']:.3f}  k1 {v.get('k1_ms', 0):.3f} "
                  f"k2/step {v.get('k2_ms_per_step', 0):.3f} k4 {v.get('k4_ms', 0):.3f} ms")
