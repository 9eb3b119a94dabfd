"""Small libaa workload for compute-sanitizer runs: every op/variant, start-up + recycle,
ragged n, ICWY Gram, delete-only, test_qradd, LOO."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09667_b200 import aa
stream = torch.cuda.current_stream()
torch.manual_seed(9667)
for n, m in ((1000, 4), (4097, 9), (70001, 3), (20003, 34)):
    d = torch.rand(n, dtype=torch.float64, device="cuda") * 1.8 - 0.9
    b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
    for v in ("mgs", "icwy", "icwy_small", "cgs2", "dcgs2"):
        s = aa.AndersonSolver(n, m, "icwy" if v == "icwy_small" else v, stream=stream,
                              beta=0.7 if n == 4097 else None, icwy_delete="small" if v == "icwy_small" else None)
        x = torch.zeros(n, dtype=torch.float64, device="cuda"); xn = torch.empty_like(x)
        s.init(x, d * x + b, xn); x, xn = xn, x
        for _ in range(m + 3):
            s.step(x, d * x + b, xn); x, xn = xn, x
        st = s.stats(loo=True)
        s.delete_oldest()
        s.step(x, d * x + b, xn)
        aa.aa_test_qradd(s.h, x)
        st = s.stats(loo=True)
        print(n, m, v, st.m_i, f"{st.loo:.2e}", flush=True)
        s.close()
# deterministic mode (whole 65536-row chunks)
n, m = 2 * 65536, 5
d = torch.rand(n, dtype=torch.float64, device="cuda") * 1.8 - 0.9
b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
for v in ("icwy", "dcgs2"):
    s = aa.AndersonSolver(n, m, v, stream=stream, deterministic=1)
    x = torch.zeros(n, dtype=torch.float64, device="cuda"); xn = torch.empty_like(x)
    s.init(x, d * x + b, xn); x, xn = xn, x
    for _ in range(m + 3):
        s.step(x, d * x + b, xn); x, xn = xn, x
    print(n, m, v, "det", s.stats().m_i, flush=True)
    s.close()
torch.cuda.synchronize()
print("ok")
