"""Steady-state AA step latency at small n (1 GPU): CUDA events around K back-to-back
recycle steps (G = d*x + b included, and timed alone so it can be subtracted)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09667_b200 import aa
ns = [int(float(a)) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1000", "1e5"])]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 20
K = 200
stream = torch.cuda.current_stream()
torch.manual_seed(9667)   # the same d, b every run


def step(s, x, g, xn):
    """aa_step with the caller's restart policy: a breakdown surfaced at entry
    (the nudged problem's differences can become collinear) resets the window once"""
    try:
        s.step(x, g, xn)
    except aa.AAError as e:
        if e.code != 6:
            raise
        s.reset()
        s.step(x, g, xn)
for n in ns:
    d = torch.rand(n, dtype=torch.float64, device="cuda") * 1.8 - 0.9
    b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
    # b is nudged every step (b += 1e-3 b), so the iteration never reaches its fixed point
    # exactly (Delta f = 0 would be a breakdown, reading A12) and every timed step is a full one
    x = torch.zeros(n, dtype=torch.float64, device="cuda"); xn = torch.empty_like(x)
    g = torch.empty_like(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(20): b.mul_(1.0 + 1e-3); torch.addcmul(b, d, x, out=g)
    e0.record()
    for _ in range(K): b.mul_(1.0 + 1e-3); torch.addcmul(b, d, x, out=g)
    e1.record(); torch.cuda.synchronize()
    tg = e0.elapsed_time(e1) / K * 1e3
    out = [f"n={n:>8d} m={m} G {tg:5.1f} us |"]
    for v in ("dcgs2", "icwy", "icwy_small", "cgs2", "mgs"):
        s = aa.AndersonSolver(n, m, "icwy" if v == "icwy_small" else v, stream=stream,
                              icwy_delete="small" if v == "icwy_small" else None)
        x.zero_()
        s.init(x, torch.addcmul(b, d, x), xn); x, xn = xn, x
        for _ in range(m + 10):
            b.mul_(1.0 + 1e-3); torch.addcmul(b, d, x, out=g); step(s, x, g, xn); x, xn = xn, x
        torch.cuda.synchronize()
        e0.record()
        for _ in range(K):
            b.mul_(1.0 + 1e-3); torch.addcmul(b, d, x, out=g); step(s, x, g, xn); x, xn = xn, x
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / K * 1e3
        out.append(f"{v} {t - tg:6.1f}")
        s.close()
    print(" ".join(out) + "  (us per AA step, G subtracted)", flush=True)
