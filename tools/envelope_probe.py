"""Measure the oracle's summation-order envelope of iteration counts (SURVEY.md §8(c)
criteria 4 and 7) against the GPU's count on the sensitive workloads the tests check (heat
term 1 / term 2, Bratu, config 5b).  Writes gpurun_out/envelope_probe.json.

    python tools/envelope_probe.py [--quick]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from aa_inputs import problems as P  # noqa: E402
from aa_inputs.heat_torch import HeatG  # noqa: E402
from oracle import aa_variant  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402

SHARDS = (1, 2, 3, 4, 5, 7, 8, 16, 37, 64, 148, 592)


def gpu_solve(Gt, n, m, variant, tol, maxit, **opts):
    s = aa.AndersonSolver(n, m, variant, stream=torch.cuda.current_stream(), **opts)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    xn = torch.empty_like(x)
    s.init(x, Gt(x), xn)
    x, xn = xn, x
    bd_prev, it = False, None
    for i in range(1, maxit + 1):
        s.step(x, Gt(x), xn)
        x, xn = xn, x
        st = s.stats()
        if st.breakdown:
            if bd_prev:
                break
            s.reset()
        bd_prev = st.breakdown
        if st.dx_norm < tol:
            it = i
            break
    s.close()
    return it, x.cpu().numpy()


def main():
    out = []
    cases = [("heat1", 256, 1, 5, 1e-8, 300, v, {}) for v in ("mgs", "icwy", "cgs2", "dcgs2")]
    cases += [("heat2", 128, 2, 10, 1e-8, 300, v, {}) for v in ("mgs", "icwy", "cgs2")]
    cases += [("bratu", 128, 3, 30, 1e-10, 100, v, {}) for v in ("mgs", "icwy", "cgs2")]
    cases += [("bratu", 128, 3, 30, 1e-10, 100, "dcgs2", {"dcgs2_rscale": 1})]
    for name, N, term, m, tol, maxit, v, opts in cases:
        b = P.heat_rhs(N, term)
        G = lambda u: P.heat_G(u, N, term, b)
        env, sols = {}, []
        okw = {"dcgs2_rscale": True} if opts.get("dcgs2_rscale") else {}
        for p in SHARDS:
            r = aa_variant(G, np.zeros(N * N), m, v, maxit, tol=tol, shards=p, record_x=False,
                           record_loo=False, breakdown="restart", **okw)
            env[p] = r.iters if r.converged else None
            if r.converged:
                sols.append(r.x)
        Gt = HeatG(N, term, torch.tensor(b, device="cuda"))
        it, u = gpu_solve(Gt, N * N, m, v, tol, maxit, **opts)
        dist = min(float(np.linalg.norm(u - s_)) for s_ in sols) if sols else None
        rec = {"case": name, "N": N, "m": m, "variant": v, "opts": opts, "gpu_iters": it,
               "oracle_iters_by_shards": env, "min_dist_to_oracle_solution": dist, "tol": tol}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    # config 5b (block-constant, 1e4-row oracle; tests/test_gpu_config5.py)
    N5, M5, P5 = 10_000_000, 50, 10_000
    W = N5 // P5
    w, d, bb = P.block_constant(N5, P5, 0.5, 0.99)
    dt = torch.tensor(d, device="cuda").repeat_interleave(W)
    bt = torch.tensor(bb, device="cuda").repeat_interleave(W)
    for v in ("mgs", "icwy", "cgs2", "dcgs2"):
        env = {}
        for p in SHARDS:
            r = aa_variant(lambda x: d * x + bb, np.zeros(P5), M5, v, 500, tol=1e-10, shards=p,
                           record_x=False, record_loo=False)
            env[p] = r.iters if r.converged else None
        it, _ = gpu_solve(lambda x: torch.addcmul(bt, dt, x), N5, M5, v, 1e-10 * np.sqrt(W), 500,
                          breakdown_eps=0.0)
        rec = {"case": "config5b", "variant": v, "gpu_iters": it, "oracle_iters_by_shards": env}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "envelope_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
