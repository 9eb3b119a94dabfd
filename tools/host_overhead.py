"""Host-side enqueue cost of aa_step (GPU queue never drains: large backlog)."""
import sys, os, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09667_b200 import aa
n, m = 1000, 20
stream = torch.cuda.current_stream()
d = torch.rand(n, dtype=torch.float64, device="cuda") * 1.8 - 0.9
b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
for v in ("dcgs2", "mgs"):
    s = aa.AndersonSolver(n, m, v, stream=stream, breakdown_eps=0.0)   # rounding-level windows: time full steps
    x = torch.zeros(n, dtype=torch.float64, device="cuda"); xn = torch.empty_like(x)
    g = torch.addcmul(b, d, x)
    s.init(x, g, xn)
    for _ in range(m + 5):
        s.step(x, g, xn)
    torch.cuda.synchronize()
    N = 300
    t0 = time.perf_counter()
    for _ in range(N):
        s.step(x, g, xn)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    xp, gp, xnp = x.data_ptr(), g.data_ptr(), xn.data_ptr()
    t3 = time.perf_counter()
    for _ in range(N):
        aa._lib.aa_step(s.h, xp, gp, xnp)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"{v}: python step enqueue {(t1-t0)/N*1e6:.1f} us/call, drain {(t2-t0)/N*1e6:.1f} us/iter; "
          f"raw ctypes enqueue {(t4-t3)/N*1e6:.1f} us/call, total {(t5-t3)/N*1e6:.1f} us/iter")
    s.close()
