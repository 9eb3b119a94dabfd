#!/bin/bash
# ncu launch list (pure kernel durations) of the small-n latency probe; prints medians.
N=${1:-1000}; M=${2:-20}; V=${3:-dcgs2,icwy,cgs2,mgs}
python tools/latency_probe.py $N $M $V > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sn_launches.csv python tools/latency_probe.py $N $M $V > /dev/null 2>&1
python - <<'PY'
import csv, re
from collections import defaultdict
rows = list(csv.reader(open('gpurun_out/sn_launches.csv')))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
agg = defaultdict(list)
for d in data:
    m_ = re.search(r"aa_stream_kernel<(\d+), (\d+), (\d+)>", d['Kernel Name'])
    k = f"OP{m_.group(1)}" if m_ else d['Kernel Name'][:30]
    agg[k].append(float(d['Metric Value']))
print(" ".join("%s:%.2fus(x%d)" % (k, sorted(v)[len(v)//2] / 1e3, len(v)) for k, v in sorted(agg.items())))
PY
