"""Host-side enqueue cost of aa_step at small n (1 GPU): wall time of the aa_step call alone
(Python binding and raw ctypes), G evaluated between calls but outside the measured span."""
import sys, os, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09667_b200 import aa
n, m = 1000, 20
stream = torch.cuda.current_stream()
d = torch.rand(n, dtype=torch.float64, device="cuda") * 1.8 - 0.9
b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
for v in ("dcgs2", "mgs"):
    s = aa.AndersonSolver(n, m, v, stream=stream)
    x = torch.zeros(n, dtype=torch.float64, device="cuda"); xn = torch.empty_like(x)
    g = torch.empty_like(x)
    s.init(x, torch.addcmul(b, d, x), xn); x, xn = xn, x
    for _ in range(m + 5):
        b.mul_(1.0 + 1e-3); torch.addcmul(b, d, x, out=g); s.step(x, g, xn); x, xn = xn, x
    torch.cuda.synchronize()
    N = 300
    tpy = traw = 0.0
    for i in range(2 * N):
        b.mul_(1.0 + 1e-3); torch.addcmul(b, d, x, out=g)    # the caller's G (not timed)
        if i < N:
            t0 = time.perf_counter(); s.step(x, g, xn); tpy += time.perf_counter() - t0
        else:
            t0 = time.perf_counter(); aa._lib.aa_step(s.h, x.data_ptr(), g.data_ptr(), xn.data_ptr())
            traw += time.perf_counter() - t0
        x, xn = xn, x
    torch.cuda.synchronize()
    print(f"{v}: aa_step host enqueue {tpy / N * 1e6:.1f} us/call (Python binding), "
          f"{traw / N * 1e6:.1f} us/call (raw ctypes)")
    s.close()
