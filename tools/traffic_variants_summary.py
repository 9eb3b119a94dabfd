#!/usr/bin/env python
"""Summarise tools/traffic_variants.sh captures: per kernel of each variant, DRAM bytes per
launch vs the DESIGN.md §7 byte model and the achieved GB/s (recycle launches of the last
two timed steps; config 2, n_local = 1e8, m = 20).  Writes profiles/r02final/traffic_variants.md.
    python tools/traffic_variants_summary.py"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import OP_NAMES, op_of, read_ncu_csv  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
V = 8 * 1e8 / 1e9   # GB per vector
m, k = 20, 19
MODEL = {0: (2 * m + 7) * V, 1: (k + 3) * V, 2: (k + 4) * V, 5: 4 * V, 6: (m + 3) * V}
PEAK = 6553.0
lines = ["# DRAM traffic and achieved bandwidth per kernel, every variant (final build)", "",
         "`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum` (single pass,",
         "cold-cache serialised launches), config 2: n_local = 1e8, m = 20, the launches of the last two",
         "timed recycle steps; model = DESIGN.md §7 bytes; GB/s over the ncu duration, and as a fraction",
         "of the measured copy peak 6553 GB/s (MEASURED_PEAKS.json).", "",
         "| variant | kernel | launches | DRAM GB / launch | model GB | ratio | ms | GB/s | of peak |",
         "|---|---|---|---|---|---|---|---|---|"]
for v in ("icwy", "icwy_small", "cgs2", "mgs"):
    path = os.path.join(ROOT, "gpurun_out", f"traffic_{v}.csv")
    if not os.path.exists(path):
        continue
    rows = read_ncu_csv(path)
    per = defaultdict(dict)
    names = {}
    for d in rows:
        per[d["ID"]][d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d.get("Metric Unit", ""))
        names[d["ID"]] = d["Kernel Name"]
    ids = [i for i in sorted(per, key=int) if op_of(names[i]) is not None]
    k4 = [j for j, i in enumerate(ids) if op_of(names[i]) == 6]
    sel = ids[k4[-3] + 1:k4[-1] + 1]   # the last two steps
    agg = defaultdict(list)
    for i in sel:
        d = per[i]
        def gb(key):
            val, unit = d[key]
            return val * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(unit, 1e-9)
        def ms(key):
            val, unit = d[key]
            return val * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6}.get(unit, 1e-6)
        agg[op_of(names[i])].append((gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum"),
                                     ms("gpu__time_duration.sum")))
    for op in sorted(agg):
        lst = agg[op]
        n = len(lst)
        b = sum(x for x, _ in lst) / n
        t = sum(y for _, y in lst) / n
        model = MODEL.get(op)
        if op == 3:
            model = (k + 2) * V
        if op == 4:
            model = (k + 3) * V
        gbs = b / (t * 1e-3)
        lines.append(f"| {v} | {OP_NAMES.get(op, op)} | {n} | {b:.2f} | {model:.2f} | {b / model:.3f} | {t:.3f} | "
                     f"{gbs:.0f} | {gbs / PEAK:.3f} |")
out = os.path.join(ROOT, "profiles", "r02final", "traffic_variants.md")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
