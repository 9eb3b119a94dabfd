#!/usr/bin/env python
"""Warp-stall samples and executed instructions per SASS opcode of one ncu --set full capture
(the source page, SASS view).  python tools/ncu_sass_summary.py <rep> <out.md> [title]"""
import csv
import subprocess
import sys
from collections import defaultdict


def main():
    rep, out = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = next(r for r in rows if "Source" in r and "Address" in r)
    data = rows[rows.index(hdr) + 1:]
    ia, iw, ie = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    agg = defaultdict(lambda: [0, 0])
    tot_w = tot_e = 0
    for r in data:
        if len(r) < len(hdr):
            continue
        toks = r[ia].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        w, e = int(r[iw] or 0), int(r[ie] or 0)
        agg[op][0] += w
        agg[op][1] += e
        tot_w += w
        tot_e += e
    lines = [f"# {title}", "", "Per SASS opcode: share of warp-stall samples and of executed (warp-level) instructions.",
             "", "| opcode | stall samples | executed instructions |", "|---|---|---|"]
    for op, (w, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
        lines.append(f"| {op} | {w / tot_w * 100:.1f} % | {e / 1e6:.1f} M ({e / tot_e * 100:.1f} %) |")
    lines.append(f"\nTotal executed: {tot_e / 1e6:.0f} M warp instructions.")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
