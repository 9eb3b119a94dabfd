"""BASELINE config 5 (orthogonality stress, n = 1e7, m = 50) as a report for profiles/:
5a  kappa = 1e12 columns appended with aa_test_qradd: LOO ||I - Q^T Q||_F, ||A - QR||/||A||,
    ms per QRAdd;
5b  AA on G = d*x + b, d ~ U[0.5, 0.99) (ill-conditioned windows, SURVEY Pr7), tol 1e-10 on
    ||Delta x|| / ||x||: iterations, max LOO (sampled every 5 iterations), us per iteration.
Parity with the oracle is asserted by tests/test_gpu_config5.py; this only records values."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from aa_inputs import problems  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402

N, M = 10_000_000, 50
out = {"config": "BASELINE config 5: n = 1e7, m = 50, fp64, 1 B200", "5a": {}, "5b": {}}
A = problems.ortho_test_matrix(N, M, 1e12, seed=5)
At = torch.from_numpy(np.ascontiguousarray(A.T)).to("cuda")
stream = torch.cuda.current_stream()
for v in ("mgs", "icwy", "cgs2", "dcgs2", "dcgs2_rscale"):
    base = "dcgs2" if v.startswith("dcgs2") else v
    s = aa.AndersonSolver(N, M, base, stream=stream, breakdown_eps=0.0,
                          dcgs2_rscale=1 if v == "dcgs2_rscale" else None)
    z = torch.zeros(N, dtype=torch.float64, device="cuda")
    x1 = torch.empty_like(z)
    s.init(z, z, x1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for j in range(M):
        aa.aa_test_qradd(s.h, At[j])
    e1.record(stream)
    torch.cuda.synchronize()
    loo = s.stats(loo=True).loo
    R, _, _, _ = aa.aa_get_small(s.h, M, M)
    q = torch.empty(N * M, dtype=torch.float64, device="cuda")
    aa.aa_get_q(s.h, q)
    resid = float(torch.linalg.norm(At - torch.tensor(R.T, device="cuda") @ q.view(M, N)) / torch.linalg.norm(At))
    out["5a"][v] = {"loo": loo, "rel_residual": resid, "ms_per_qradd": e0.elapsed_time(e1) / M}
    s.close()
    del q
    print(v, out["5a"][v], flush=True)
del At
torch.cuda.empty_cache()
d = torch.empty(N, dtype=torch.float64, device="cuda")
b = torch.empty_like(d)
aa.aa_fill_uniform(d, N, 0.5, 0.99, stream_id=1, stream=stream)
aa.aa_fill_uniform(b, N, -1.0, 1.0, stream_id=2, stream=stream)
for v in ("mgs", "icwy", "icwy_small", "cgs2", "dcgs2", "dcgs2_rscale"):
    base = {"icwy_small": "icwy", "dcgs2_rscale": "dcgs2"}.get(v, v)
    s = aa.AndersonSolver(N, M, base, stream=stream, icwy_delete="small" if v == "icwy_small" else None,
                          dcgs2_rscale=1 if v == "dcgs2_rscale" else None)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    xn, g = torch.empty_like(x), torch.empty_like(x)
    s.init(x, torch.addcmul(b, d, x, out=g), xn)
    x, xn = xn, x
    maxloo, it, t_ms, conv = 0.0, 0, 0.0, False
    for it in range(1, 301):
        torch.addcmul(b, d, x, out=g)
        e0.record(stream)
        s.step(x, g, xn)
        e1.record(stream)
        st = s.stats(loo=(it % 5 == 0))
        t_ms += e0.elapsed_time(e1)
        if st.loo >= 0:
            maxloo = max(maxloo, st.loo)
        x, xn = xn, x
        if st.dx_norm <= 1e-10 * float(torch.linalg.norm(x)):
            conv = True
            break
    out["5b"][v] = {"iterations": it, "converged": conv, "max_loo_sampled": maxloo,
                    "us_per_iter": t_ms * 1e3 / it, "final_f_norm": st.f_norm}
    s.close()
    print(v, out["5b"][v], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/config5_report.json", "w"), indent=1)
