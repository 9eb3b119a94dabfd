"""GPU parity for ICWY with the reduction-free T update after QRDelete
(AA_OPT_ICWY_DELETE = SMALL; a variant, not in the paper: SURVEY.md §8(f) row 1,
DESIGN.md A6b).  Reference: oracle.aa_variant(..., icwy_delete="small"), pinned in
tests/test_oracle_pins.py against the explicit Gram of the rotated Q."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from aa_inputs import problems  # noqa: E402
from oracle import EPS, aa_variant  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2110_09667_b200 import aa  # noqa: E402
from tests._gpu_run import run_gpu  # noqa: E402

SMALL = dict(icwy_delete="small")


def _rel_x(gpu, orc, K):
    return max((np.linalg.norm(a - b) / np.linalg.norm(b) for a, b in zip(gpu.xs[:K], orc.xs[:K])), default=0.0)


def _K(o2, tol=1e-11):
    return next((i for i, f in enumerate(o2.f_norms) if f < tol * np.linalg.norm(o2.x1)), len(o2.f_norms))


def test_config1_small():
    M, b = problems.linear_dense(1000, 0.95)
    Mt, bt = torch.tensor(M, device="cuda"), torch.tensor(b, device="cuda")
    o2 = aa_variant(lambda x: M @ x + b, np.zeros(1000), 5, "icwy", 30, icwy_delete="small")
    gpu = run_gpu(lambda x: Mt @ x + bt, np.zeros(1000), 5, "icwy", 30, loo=True, **SMALL)
    assert _rel_x(gpu, o2, 20) <= 1e-10
    for lg, lo in zip(gpu.loo, o2.loo):
        assert lg <= max(10 * lo, 10 * 5 * EPS)
    # recycle: 2 reductions, no qrdelete reduction (logical ledger equals the oracle's)
    assert gpu.sync_points[-1] == 2
    assert gpu.ledgers[-1] == o2.ledgers[-1]
    assert gpu.ledgers[-1]["qrdelete"] == 0


@pytest.mark.parametrize("n,m", [(1, 3), (257, 2), (4097, 7), (70001, 20), (1000, 3)])
def test_ragged_small(n, m):
    d, b = problems.diagonal(n)
    dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
    iters = min(2 * m + 6, 30)
    o2 = aa_variant(lambda x: d * x + b, np.zeros(n), m, "icwy", iters, icwy_delete="small")
    gpu = run_gpu(lambda x: dt * x + bt, np.zeros(n), m, "icwy", iters, **SMALL)
    K = _K(o2)
    if K > 0:
        assert _rel_x(gpu, o2, K) <= 1e-10
    for i in range(K):
        assert gpu.ledgers[i] == o2.ledgers[i]


@pytest.mark.parametrize("n,m,iters", [(20003, 50, 56), (3000, 64, 68)])
def test_large_windows_small(n, m, iters):
    d, b = problems.diagonal(n, -0.95, 0.95)
    dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
    o2 = aa_variant(lambda x: d * x + b, np.zeros(n), m, "icwy", iters, icwy_delete="small")
    gpu = run_gpu(lambda x: dt * x + bt, np.zeros(n), m, "icwy", iters, loo=True, **SMALL)
    K = _K(o2, 1e-9)
    assert _rel_x(gpu, o2, K) <= 1e-10
    for lg, lo in zip(gpu.loo[:K], o2.loo[:K]):
        assert lg <= max(10 * lo, 10 * m * EPS)


def test_ill_conditioned_window_converges():
    """SURVEY Pr6 window (d in U[0.9, 0.99], LOO ~ 0.5): the small update converges like
    the oracle and the paper's rebuild; LOO stays in the oracle's class."""
    n, m, iters = 4000, 20, 80
    d, b = problems.diagonal(n, 0.9, 0.99, seed=11)
    dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
    o2 = aa_variant(lambda x: d * x + b, np.zeros(n), m, "icwy", iters, icwy_delete="small", record_x=False)
    gpu = run_gpu(lambda x: dt * x + bt, np.zeros(n), m, "icwy", iters, loo=True, record_x=False, **SMALL)
    f0 = o2.f_norms[0]
    assert o2.f_norms[-1] <= 1e-9 * f0
    assert gpu.f_norms[-1] <= 1e-9 * f0, gpu.f_norms[-1] / f0
    assert max(gpu.loo) <= 10 * max(o2.loo)


def test_small_after_init_is_refused_and_delete_oldest_works():
    n, m = 3001, 5
    d, b = problems.diagonal(n)
    dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
    s = aa.AndersonSolver(n, m, "icwy", stream=torch.cuda.current_stream())
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    xn = torch.empty_like(x)
    s.init(x, dt * x + bt, xn)
    with pytest.raises(aa.AAError):
        aa.aa_set_option(s.h, aa.OPT_ICWY_DELETE, 2.0)
    s.close()
    # SMALL chosen before init; a stand-alone delete (which uses the paper's rebuild) in the
    # middle of the run leaves a consistent factorisation the following steps build on
    gpu = aa.AndersonSolver(n, m, "icwy", stream=torch.cuda.current_stream(), **SMALL)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    gpu.init(x, dt * x + bt, xn)
    x, xn = xn, x
    for i in range(m + 3):
        gpu.step(x, dt * x + bt, xn)
        x, xn = xn, x
    gpu.delete_oldest()
    for i in range(4):
        gpu.step(x, dt * x + bt, xn)
        x, xn = xn, x
    st = gpu.stats(loo=True)
    gpu.close()
    assert np.isfinite(st.f_norm) and st.loo <= 1e-12
