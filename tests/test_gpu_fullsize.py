"""Parity at the bench's full size (config 2: n_local = 1e8 fp64, m = 20 and 50), in the
launch configuration bench.py times.

The problem is block-constant: d and b are constant on 1000 equal row blocks of 1e5
rows, so every AA iterate is block-constant and — the inner product being 1e5 times the
1000-row one, which leaves gamma unchanged — equal blockwise to the iterate of the
1000-row problem, which the oracle runs (pinned on CPU by
tests/test_oracle_pins.py::test_block_constant_reduction_property).  Checked per
iteration on one sampled row per block; rows within a block must be bitwise equal.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from aa_inputs import problems  # noqa: E402
from oracle import EPS, aa_variant, VARIANTS  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402

N, P = 100_000_000, 1000
W = N // P


@pytest.fixture(scope="module")
def big_problem():
    w, d, b = problems.block_constant(N, P)
    assert (w == W).all()
    dt = torch.tensor(d, device="cuda").repeat_interleave(W)
    bt = torch.tensor(b, device="cuda").repeat_interleave(W)
    return d, b, dt, bt


@pytest.mark.parametrize("variant,m,iters", [(v, 20, 26) for v in VARIANTS] + [("dcgs2", 50, 56), ("icwy", 50, 56)])
def test_full_size_block_constant(big_problem, variant, m, iters):
    d, b, dt, bt = big_problem
    ref = aa_variant(lambda x: d * x + b, np.zeros(P), m, variant, iters)
    stream = torch.cuda.current_stream()
    s = aa.AndersonSolver(N, m, variant, stream=stream)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    xn = torch.empty_like(x)
    s.init(x, torch.addcmul(bt, dt, x), xn)
    x, xn = xn, x
    starts = torch.arange(0, N, W, device="cuda")
    worst = 0.0
    K = next((i for i, f in enumerate(ref.f_norms) if f < 1e-11 * np.linalg.norm(ref.x1)), iters)
    for i in range(iters):
        s.step(x, torch.addcmul(bt, dt, x), xn)
        x, xn = xn, x
        if i < K:
            samp = x[starts].cpu().numpy()
            last = x[starts + W - 1].cpu().numpy()
            assert np.array_equal(samp, last), "rows of a block must be bitwise equal"
            r = ref.xs[i]
            worst = max(worst, float(np.linalg.norm(samp - r) / np.linalg.norm(r)))
    st = s.stats(loo=True)
    s.close()
    assert worst <= 1e-10, worst
    assert st.m_i == m
    # LOO of a length-1e8 factorisation carries the summation error of its own inner
    # products (each of the 148x32 lanes accumulates ~2e4 products): floor
    # 10 m eps sqrt(n / 4736); the 1000-row oracle cannot see that term.
    assert st.loo <= max(10 * ref.loo[-1], 10 * m * EPS * np.sqrt(N / 4736)), (st.loo, ref.loo[-1])
