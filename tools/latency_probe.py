"""Per-kernel latency at small n (profile events inside libaa), 1 GPU."""
import sys, os, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09667_b200 import aa
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 20
stream = torch.cuda.current_stream()
d = torch.rand(n, dtype=torch.float64, device="cuda") * 1.8 - 0.9
b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
G = lambda x: torch.addcmul(b, d, x)
VS = sys.argv[3].split(",") if len(sys.argv) > 3 else ["dcgs2", "icwy", "cgs2", "mgs"]
for v in VS:
    s = aa.AndersonSolver(n, m, "icwy" if v == "icwy_small" else v, stream=stream, profile=1,
                          icwy_delete="small" if v == "icwy_small" else None)
    x = torch.zeros(n, dtype=torch.float64, device="cuda"); xn = torch.empty_like(x)
    s.init(x, G(x), xn); x, xn = xn, x
    for _ in range(m + 5):
        s.step(x, G(x), xn); x, xn = xn, x
    aa.aa_timings(s.h, reset=True)
    K = 20
    for _ in range(K):
        s.step(x, G(x), xn); x, xn = xn, x
    ms, cnt = aa.aa_timings(s.h, reset=True)
    print(f"{v:6s} n={n} m={m}: step {ms[4]/K*1e3:7.1f} us | K1 {ms[0]/max(cnt[0],1)*1e3:6.1f} us x{cnt[0]//K} | "
          f"K2 {ms[1]/max(cnt[1],1)*1e3:6.1f} us x{cnt[1]//K} | K4 {ms[2]/max(cnt[2],1)*1e3:6.1f} us x{cnt[2]//K}")
    s.close()
