"""Dump the steady-state R factor (K x K in a 64 x 64 column-major fp64 file) of a small-n
AA run, for tools/k3_bench with real data.  argv: n m iters out.bin"""
import sys, os, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_09667_b200 import aa
n, m, iters, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
stream = torch.cuda.current_stream()
d = torch.rand(n, dtype=torch.float64, device="cuda") * 1.8 - 0.9
b = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
s = aa.AndersonSolver(n, m, "dcgs2", stream=stream)
x = torch.zeros(n, dtype=torch.float64, device="cuda"); xn = torch.empty_like(x)
s.init(x, d * x + b, xn); x, xn = xn, x
for _ in range(iters):
    s.step(x, d * x + b, xn); x, xn = xn, x
st = s.stats()
R, T, g, sc = aa.aa_get_small(s.h, m, st.m_i)
full = np.zeros((64, 64)); K = st.m_i
full[:K, :K] = R[:K, :K]
full.ravel(order="F").tofile(out)
print("K", K, "f_norm", st.f_norm, "diag", np.diag(full)[:K][:6], "min|diag|", np.min(np.abs(np.diag(full)[:K])))
