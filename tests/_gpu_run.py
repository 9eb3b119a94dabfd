"""Drive libaa from Python for the GPU tests (the caller's loop of Alg. 1).

G is the caller's map, evaluated with torch on the device; AA runs entirely in
libaa through the C ABI."""
import numpy as np
import torch

from paper_2110_09667_b200 import aa


class Run:
    def __init__(self):
        self.xs, self.f_norms, self.dx_norms, self.loo, self.ledgers = [], [], [], [], []
        self.sync_points, self.iters, self.converged, self.x = [], 0, False, None
        self.breakdown, self.hard_error = [], False


def run_gpu(G, x0, m, variant, iters, tol=0.0, record_x=True, loo=False, stats_every=True, **opts):
    """G: torch function on a cuda float64 vector.  Returns a Run mirroring oracle.AAResult.

    With stats_every (the default) the loop applies SPEC's breakdown policy as
    oracle.aa_variant(breakdown="restart") does: aa_reset after a breakdown, stop on
    a second consecutive one (Run.hard_error)."""
    stream = torch.cuda.current_stream()
    n = x0.shape[0]
    s = aa.AndersonSolver(n, m, variant, stream=stream, **opts)
    x = torch.as_tensor(np.asarray(x0), dtype=torch.float64, device="cuda").clone()
    xn = torch.empty_like(x)
    g = G(x)
    s.init(x, g, xn)
    x, xn = xn, x
    r = Run()
    for i in range(1, iters + 1):
        g = G(x)
        s.step(x, g, xn)
        if stats_every or i == iters:
            st = s.stats(loo=loo)
            r.f_norms.append(st.f_norm)
            r.dx_norms.append(st.dx_norm)
            r.loo.append(st.loo)
            r.ledgers.append(dict(st.logical))
            r.sync_points.append(st.sync_points_last)
            r.breakdown.append(st.breakdown)
        if record_x:
            r.xs.append(xn.cpu().numpy())
        x, xn = xn, x
        r.iters = i
        if stats_every and r.breakdown[-1]:
            if len(r.breakdown) >= 2 and r.breakdown[-2]:
                r.hard_error = True
                break
            s.reset()
        if tol > 0 and stats_every and r.dx_norms[-1] < tol:
            r.converged = True
            break
    r.x = x.cpu().numpy()
    r.solver = s
    return r
