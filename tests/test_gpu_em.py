"""EM-mixture workload (§5.3) through libaa on the GPU: n_local = 1.5e6
(the paper's per-GPU size), m = 3, stopping on the per-replica norm ||Delta mu||_2 < 1e-8.
Iteration count identical to the oracle's for every variant; means to 1e-9."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from aa_inputs import problems as P  # noqa: E402
from oracle import aa_variant, VARIANTS  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402


def em_G_torch(xs, alpha, sigma):
    def G(u, out):
        mu = u[:3]
        dens = alpha[:, None] / (math.sqrt(2 * math.pi) * sigma[:, None]) * torch.exp(
            -(xs[None, :] - mu[:, None]) ** 2 / (2 * sigma[:, None] ** 2))
        w = dens / dens.sum(dim=0, keepdim=True)
        new = (w * xs[None, :]).sum(dim=1) / w.sum(dim=1)
        out.view(-1, 3).copy_(new.expand(out.shape[0] // 3, 3))
        return out
    return G


@pytest.mark.parametrize("variant", VARIANTS)
def test_em_gpu_matches_oracle(variant):
    n = 1_500_000
    xs_np = P.em_samples()
    ref = aa_variant(lambda u: P.em_G_replicated(u, xs_np), np.array([0.2, 0.4, 0.6]), 3, variant, 100,
                     tol=1e-8, record_x=False, record_loo=False)
    xs = torch.tensor(xs_np, device="cuda")
    G = em_G_torch(xs, torch.tensor(P.EM_ALPHA, device="cuda", dtype=torch.float64),
                   torch.tensor(P.EM_SIGMA, device="cuda", dtype=torch.float64))
    s = aa.AndersonSolver(n, 3, variant, stream=torch.cuda.current_stream())
    x = torch.tensor([0.2, 0.4, 0.6], dtype=torch.float64, device="cuda").repeat(n // 3)
    g = torch.empty_like(x)
    xn = torch.empty_like(x)
    s.init(x, G(x, g), xn)
    x, xn = xn, x
    it = 0
    for it in range(1, 101):
        s.step(x, G(x, g), xn)
        x, xn = xn, x
        if s.stats().dx_norm * math.sqrt(3 / n) < 1e-8:    # per-replica ||Delta mu||_2
            break
    mu = x[:3].cpu().numpy()
    rep = x.view(-1, 3)
    assert torch.equal(rep[0].expand_as(rep), rep), "every triple must stay bitwise identical"
    s.close()
    assert it == ref.iters
    assert np.max(np.abs(mu - ref.x)) < 1e-9
