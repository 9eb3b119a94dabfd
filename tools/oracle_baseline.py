"""The CPU oracle (O2, numpy fp64, as it stands) timed on the GPU box's host cores
(SURVEY.md §8(d) "How the oracle is timed beside the GPU"): config 2's DCGS-2 recycle
iteration at n = 1e7 (all BLAS threads and 1 thread) and at n = 1e8 when host RAM allows,
with lscpu and RAM recorded.  Writes gpurun_out/oracle_baseline.json.

    python tools/oracle_baseline.py [--m 20] [--variant dcgs2] [--big]
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from aa_inputs import problems  # noqa: E402
from oracle import aa_variant  # noqa: E402


def time_o2(n, m, variant, recycle_steps, threads):
    from threadpoolctl import threadpool_limits
    d, b = problems.diagonal(n)
    stamps = []

    def G(x):
        stamps.append(time.perf_counter())
        return d * x + b

    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        aa_variant(G, np.zeros(n), m, variant, m + recycle_steps, record_x=False, record_loo=False)
        total = time.perf_counter() - t0
    # G is called at x_0 and then once per iteration: the gap between consecutive calls is one
    # AA iteration (G excluded up to the cost of one fused multiply-add pass)
    gaps = np.diff(stamps)
    startup = float(np.sum(gaps[:m]))
    rec = gaps[m:]
    return {"n": n, "m": m, "variant": variant, "threads": threads, "startup_s_total": startup,
            "recycle_s_per_iter": float(np.mean(rec)) if len(rec) else None,
            "recycle_samples": [round(float(v), 4) for v in rec], "wall_s": total}


def host_info():
    info = {"cpu_count": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None}
    try:
        info["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=30).stdout
    except Exception as e:
        info["lscpu"] = f"unavailable: {e}"
    try:
        mem = {l.split(":")[0]: l.split(":")[1].strip() for l in open("/proc/meminfo") if ":" in l}
        info["MemTotal"], info["MemAvailable"] = mem.get("MemTotal"), mem.get("MemAvailable")
    except Exception:
        pass
    return info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=20)
    ap.add_argument("--variant", default="dcgs2")
    ap.add_argument("--big", action="store_true", help="also n = 1e8 if MemAvailable allows")
    args = ap.parse_args()
    host = host_info()
    ncores = host["affinity"] or host["cpu_count"]
    runs = [time_o2(10_000_000, args.m, args.variant, 3, ncores),
            time_o2(10_000_000, args.m, args.variant, 2, 1)]
    avail_kb = int(str(host.get("MemAvailable", "0 kB")).split()[0])
    need_gb = (2 * args.m + 12) * 0.8 * 1.5      # window + vectors + numpy temporaries, with margin
    if args.big and avail_kb / 1e6 > need_gb:
        runs.append(time_o2(100_000_000, args.m, args.variant, 2, ncores))
    elif args.big:
        runs.append({"n": 100_000_000, "skipped": f"MemAvailable {avail_kb / 1e6:.1f} GB < {need_gb:.0f} GB"})
    out = {"host": host, "runs": runs}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "oracle_baseline.json"), "w"), indent=1)
    for r in runs:
        print(json.dumps({k: v for k, v in r.items() if k != "recycle_samples"}), flush=True)


if __name__ == "__main__":
    main()
