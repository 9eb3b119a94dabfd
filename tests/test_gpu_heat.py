"""Heat + nonlinear term (§5.1; BASELINE config 4 at test size) through libaa on
the GPU.  The Picard map is sensitive (plain FP is expansive for term 2), so per-iterate
1e-10 parity is not required (SURVEY.md §8(c) criterion 7): the iteration count must lie in
the oracle's summation-order envelope and the converged solution match the oracle's to
100*tol."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from aa_inputs import problems as P  # noqa: E402
from aa_inputs.heat_torch import HeatG, dst1_lastdim  # noqa: E402
from oracle import aa_variant  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402

# SURVEY.md §8(c) criteria 4 and 7: the oracle's iteration-count envelope over summation
# orders (simulated contiguous shards summed in rank order).  Twelve orders, including the
# GPU-like 148- and 592-way splits; profiles/r02/envelope_probe.json records the widths
# (heat term 2: MGS 39-43, ICWY 38-42, CGS-2 39-40; Bratu 12-13) and that the GPU's count
# falls inside with no slack.
ENVELOPE_SHARDS = (1, 2, 3, 4, 5, 7, 8, 16, 37, 64, 148, 592)


def test_torch_dst_matches_scipy():
    from scipy.fft import dst
    x = np.random.default_rng(1).standard_normal((5, 37))
    y = dst1_lastdim(torch.tensor(x, device="cuda")).cpu().numpy()
    assert np.allclose(y, dst(x, type=1, norm="ortho", axis=-1), rtol=1e-13, atol=1e-13)
    N = 32
    b = P.heat_rhs(N, 2)
    u = np.random.default_rng(2).standard_normal(N * N) * 0.1
    G = HeatG(N, 2, torch.tensor(b, device="cuda"))
    assert np.allclose(G(torch.tensor(u, device="cuda")).cpu().numpy(), P.heat_G(u, N, 2, b), rtol=1e-12, atol=1e-14)


def _gpu_solve(N, term, m, variant, tol, maxit, **opts):
    b = torch.tensor(P.heat_rhs(N, term), device="cuda")
    G = HeatG(N, term, b)
    s = aa.AndersonSolver(N * N, m, variant, stream=torch.cuda.current_stream(), **opts)
    x = torch.zeros(N * N, dtype=torch.float64, device="cuda")
    xn = torch.empty_like(x)
    s.init(x, G(x), xn)
    x, xn = xn, x
    bd_prev = False
    for it in range(1, maxit + 1):
        s.step(x, G(x), xn)
        x, xn = xn, x
        st = s.stats()
        if st.breakdown:            # SPEC's restart policy, as oracle breakdown="restart"
            if bd_prev:
                break
            s.reset()
        bd_prev = st.breakdown
        if st.dx_norm < tol:
            s.close()
            return it, x.cpu().numpy()
    s.close()
    return None, x.cpu().numpy()


@pytest.mark.parametrize("term,m,N,variant", [(1, 5, 256, v) for v in ("mgs", "icwy", "cgs2", "dcgs2")]
                         + [(2, 10, 128, v) for v in ("mgs", "icwy", "cgs2")])
def test_heat_envelope(term, m, N, variant):
    tol = 1e-8
    b = P.heat_rhs(N, term)
    G = lambda u: P.heat_G(u, N, term, b)
    env, sols = [], []
    for p in ENVELOPE_SHARDS:
        r = aa_variant(G, np.zeros(N * N), m, variant, 300, tol=tol, shards=p, record_x=False, record_loo=False,
                        breakdown="restart")
        if r.converged:
            env.append(r.iters)
            sols.append(r.x)
    assert env, "oracle envelope empty"
    it, u = _gpu_solve(N, term, m, variant, tol, 300)
    assert it is not None and min(env) <= it <= max(env), (it, env)
    assert min(np.linalg.norm(u - s_) for s_ in sols) <= 100 * tol


def test_heat_term2_dcgs2_reported_not_failed():
    """Verbatim DCGS-2 does not converge on term 2 in the oracle either (SURVEY
    [Pr8]); the GPU run must simply complete without error."""
    it, u = _gpu_solve(128, 2, 10, "dcgs2", 1e-8, 60)
    assert u.shape == (128 * 128,)


@pytest.mark.parametrize("variant,opts,okw", [("mgs", {}, {}), ("icwy", {}, {}), ("cgs2", {}, {}),
                                              ("dcgs2", {"dcgs2_rscale": 1}, {"dcgs2_rscale": True})])
def test_bratu_envelope(variant, opts, okw):
    """Bratu (§5.2): lambda = 6.7, m = 30, tol 1e-10, 128^2."""
    N, tol = 128, 1e-10
    b = P.heat_rhs(N, 3)
    G = lambda u: P.heat_G(u, N, 3, b)
    env, sols = [], []
    for p in ENVELOPE_SHARDS:
        r = aa_variant(G, np.zeros(N * N), 30, variant, 100, tol=tol, shards=p, record_x=False,
                       record_loo=False, breakdown="restart", **okw)
        if r.converged:
            env.append(r.iters)
            sols.append(r.x)
    assert env and max(env) < 30
    it, u = _gpu_solve(N, 3, 30, variant, tol, 100, **opts)
    assert it is not None and min(env) <= it <= max(env), (it, env)
    assert min(np.linalg.norm(u - s_) for s_ in sols) <= 100 * tol
