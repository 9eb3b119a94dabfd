#!/usr/bin/env python
"""Summarise a tools/profile.sh capture into profiles/<tag>/ (committed evidence).

    python tools/ncu_summary.py r01

Writes profiles/<tag>/launches.md (per-kernel launch list + share of the step),
traffic.md (DRAM bytes per launch vs the algorithmic byte model), k1_*.md (key
`ncu --set full` metrics and stall reasons of K1) and merges the per-launch traffic of
K1 into profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OP_NAMES = {0: "K1 pass1 (prologue+QRDelete+multi-dot)", 1: "K2 ICWY", 2: "K2 DCGS-2", 3: "K2a CGS-2",
            4: "K2b CGS-2", 5: "K2_j MGS", 6: "K4 update+commit", 7: "Gram (LOO)"}


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def op_of(name):
    import re
    m = re.search(r"aa_stream_kernel<\(?(?:int\)?)?(\d+)", name)
    return int(m.group(1)) if m else None


def kernel_label(name):
    op = op_of(name)
    if op is not None:
        return OP_NAMES.get(op, f"op{op}")
    return name.split("(")[0][:60]


def launches(tag, src):
    data = read_ncu_csv(os.path.join(src, "launches.csv"))
    per = []
    for d in data:
        if d.get("Metric Name") == "gpu__time_duration.sum":
            unit = d.get("Metric Unit", "ns")
            v = float(d["Metric Value"].replace(",", ""))
            ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
            per.append((d["Kernel Name"], ns))
    # the timed region = the last 3 steps: last 3 K4 launches bound it
    lib = [(n, t) for n, t in per if op_of(n) is not None]
    k4_idx = [i for i, (n, _) in enumerate(lib) if op_of(n) == 6]
    start = k4_idx[-4] + 1 if len(k4_idx) >= 4 else 0
    timed = lib[start:]
    agg = defaultdict(list)
    for n, t in timed:
        agg[kernel_label(n)].append(t)
    total = sum(t for _, t in timed)
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             "Command: `python bench.py --only-headline --no-e2e --no-cpu --steps 3 --warmup 3` "
             "(config 2: n_local = 1e8, m = 20, DCGS-2 recycle).  Cold-cache, serialised launches:",
             "compare SHARES with the bench's CUDA-event split, not absolutes.", "",
             "| kernel | launches in the 3 timed steps | mean µs | share of libaa time |", "|---|---|---|---|"]
    for k, v in agg.items():
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / total * 100:.1f}% |")
    lines.append("")
    lines.append(f"All launches in the capture: {len(per)} (libaa: {len(lib)}).")
    return "\n".join(lines), {k: {"n": len(v), "mean_us": sum(v) / len(v) / 1e3, "share": sum(v) / total}
                              for k, v in agg.items()}


def traffic(src, fname, m, variant):
    data = read_ncu_csv(os.path.join(src, fname))
    per = defaultdict(dict)
    for d in data:
        key = (d["ID"], d["Kernel Name"])
        unit = d.get("Metric Unit", "")
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "ns": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1}.get(unit, 1)
        per[key][d["Metric Name"]] = v * scale
    V = 8e8
    k = m - 1
    algo = {0: (2 * m + 7) * V, 6: (m + 3) * V,
            2: (k + 4) * V, 1: (k + 3) * V, 3: (k + 2) * V, 4: (k + 3) * V, 5: 4 * V}
    rows = []
    k4 = [i for i, (key, _) in enumerate(per.items()) if op_of(key[1]) == 6]
    items = list(per.items())
    last = items[k4[-4] + 1:] if len(k4) >= 4 else items
    agg = defaultdict(list)
    for (id_, name), mets in last:
        op = op_of(name)
        if op is None:
            continue
        tr = mets.get("dram__bytes_read.sum", 0) + mets.get("dram__bytes_write.sum", 0)
        agg[op].append((tr, mets.get("gpu__time_duration.sum", 0)))
    out = {}
    for op, lst in sorted(agg.items()):
        tr = sum(t for t, _ in lst) / len(lst)
        dur = sum(d for _, d in lst) / len(lst)
        a = algo.get(op)
        out[op] = {"dram_bytes_per_launch": tr, "algorithmic_bytes": a, "ratio": tr / a if a else None,
                   "ncu_duration_s": dur, "ncu_gbs": tr / dur / 1e9 if dur else None}
        rows.append(f"| {OP_NAMES.get(op)} ({variant}) | {tr / 1e9:.2f} | {a / 1e9 if a else float('nan'):.2f} | "
                    f"{tr / a if a else float('nan'):.3f} | {dur * 1e3:.2f} | {tr / dur / 1e9:.0f} |")
    return rows, out


def full(src, name, tag):
    rep = os.path.join(src, name + ".ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        return f"(no data in {rep})"
    return "\n\n".join(_full_one(dict(zip(rows[0], r)), name, tag) for r in rows[2:])


def _full_one(d, name, tag):
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__shared_mem_per_block_dynamic"]
    size = {"k1_icwy50": "n_local = 2e7, m = 50", "k1_dcgs2": "n_local = 1e8, m = 20" if tag != "r01" else "n_local = 2e7, m = 20"}.get(name, "n_local = 2e7, m = 20")
    lines = [f"# {tag}: `ncu --set full` of {name} ({size}, recycle): "
             f"{d.get('Kernel Name', '')[:60]}", "", "| metric | value |", "|---|---|"]
    for kk in keys:
        if kk in d:
            lines.append(f"| {kk} | {d[kk]} |")
    st = {k2: v for k2, v in d.items() if "pcsamp_warps_issue_stalled" in k2 and not k2.endswith("not_issued")}
    tot = sum(float(v) for v in st.values() if v)
    lines += ["", "Warp-stall samples:", "", "| reason | share |", "|---|---|"]
    for k2, v in sorted(st.items(), key=lambda kv: -float(kv[1] or 0)):
        if float(v or 0) > 0:
            lines.append(f"| {k2.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {float(v) / tot * 100:.1f}% |")
    return "\n".join(lines)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = os.path.join(ROOT, "gpurun_out", f"prof_{tag}")
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    md, shares = launches(tag, src)
    open(os.path.join(dst, "launches.md"), "w").write(md + "\n")
    rows = ["# DRAM traffic per launch at the bench size (n_local = 1e8, m = 20)", "",
            "`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum` "
            "(single pass), averaged over the 3 timed steps.  algorithmic = DESIGN.md §7 byte model.", "",
            "| kernel | DRAM GB/launch | algorithmic GB | ratio | ncu ms | ncu GB/s |", "|---|---|---|---|---|---|"]
    r1, t_d = traffic(src, "traffic.csv", 20, "dcgs2")
    r2, t_i = traffic(src, "traffic_icwy.csv", 20, "icwy") if os.path.exists(os.path.join(src, "traffic_icwy.csv")) else ([], {})
    r3 = traffic(src, "traffic_cgs2.csv", 20, "cgs2")[0] if os.path.exists(os.path.join(src, "traffic_cgs2.csv")) else []
    open(os.path.join(dst, "traffic.md"), "w").write("\n".join(rows + r1 + r2 + r3) + "\n")
    for name in ("k1_dcgs2", "k1_icwy", "k2_cgs2", "k1_icwy50"):
        if os.path.exists(os.path.join(src, name + ".ncu-rep")):
            open(os.path.join(dst, name + ".md"), "w").write(full(src, name, tag) + "\n")
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    summ.setdefault("k1", {})
    if 0 in t_d:
        summ["k1"]["dcgs2_m20"] = dict(t_d[0], round=tag)
    if 0 in t_i:
        summ["k1"]["icwy_m20"] = dict(t_i[0], round=tag)
    summ["launch_shares_" + tag] = shares
    json.dump(summ, open(summ_path, "w"), indent=1)
    print(open(os.path.join(dst, "launches.md")).read())
    print(open(os.path.join(dst, "traffic.md")).read())


if __name__ == "__main__":
    main()
