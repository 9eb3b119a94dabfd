"""aa_step_host at large n (>= 4M rows) splits the PCIe copies into row chunks overlapped
with row-chunked K1 / K4 launches whose reductions accumulate over the chunks.  It must
follow the device path (aa_step) to rounding, for every variant, through start-up and
recycle iterations, and match the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from aa_inputs import problems  # noqa: E402
from oracle import aa_variant  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402

N = 5_000_003   # > 4M rows (chunked), odd (ragged last tile and odd exact-vector tail)


@pytest.fixture(scope="module")
def prob():
    d, b = problems.diagonal(N)
    return d, b, torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")


@pytest.mark.parametrize("variant", ["dcgs2", "icwy", "cgs2", "mgs", "icwy_small"])
def test_step_host_chunked_matches_device(prob, variant):
    d, b, dt, bt = prob
    m, iters = 5, 12
    base = "icwy" if variant == "icwy_small" else variant
    opt = dict(icwy_delete="small") if variant == "icwy_small" else {}
    stream = torch.cuda.current_stream()
    dev = aa.AndersonSolver(N, m, base, stream=stream, **opt)
    hst = aa.AndersonSolver(N, m, base, stream=stream, **opt)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    xn = torch.empty_like(x)
    dev.init(x, dt * x + bt, xn)
    x, xn = xn, x
    xh = torch.zeros(N, dtype=torch.float64).pin_memory()
    gh = torch.empty(N, dtype=torch.float64).pin_memory()
    oh = torch.empty(N, dtype=torch.float64).pin_memory()
    x0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    x1 = torch.empty_like(x0)
    hst.init(x0, dt * x0 + bt, x1)
    xh.copy_(x1.cpu())
    bh, dh = bt.cpu(), dt.cpu()
    worst = 0.0
    for i in range(iters):
        dev.step(x, dt * x + bt, xn)
        x, xn = xn, x
        torch.addcmul(bh, dh, xh, out=gh)
        hst.step_host(xh, gh, oh)
        xh, oh = oh, xh
        a = x.cpu().numpy()
        worst = max(worst, float(np.linalg.norm(xh.numpy() - a) / np.linalg.norm(a)))
    sd, sh = dev.stats(), hst.stats()
    dev.close()
    hst.close()
    assert worst <= 1e-12, worst
    assert abs(sd.f_norm - sh.f_norm) <= 1e-12 * sd.f_norm
    assert abs(sd.dx_norm - sh.dx_norm) <= 1e-10 * sd.dx_norm + 1e-300
    assert sd.logical == sh.logical
    if variant == "dcgs2":   # and the oracle, once
        o2 = aa_variant(lambda v: d * v + b, np.zeros(N), m, "dcgs2", iters, record_loo=False)
        assert np.linalg.norm(xh.numpy() - o2.xs[-1]) <= 1e-10 * np.linalg.norm(o2.xs[-1])


@pytest.mark.parametrize("n", [4097, 5_000_003])
def test_step_host_reuses_device_x(n):
    """aa_step_host(x_i = NULL) takes the x_{i+1} its previous call returned (kept on the
    device): bitwise the same iterates as uploading x_i every time, small and row-chunked
    sizes; NULL without a previous host step (or after an aa_step) is AA_ERR_STATE."""
    d, b = problems.diagonal(n)
    dh, bh = torch.tensor(d), torch.tensor(b)
    stream = torch.cuda.current_stream()
    outs = []
    for reuse in (False, True):
        s = aa.AndersonSolver(n, 4, "dcgs2", stream=stream)
        x0 = torch.zeros(n, dtype=torch.float64, device="cuda")
        x1 = torch.empty_like(x0)
        s.init(x0, torch.tensor(b, device="cuda"), x1)
        xh = x1.cpu().pin_memory()
        gh = torch.empty(n, dtype=torch.float64).pin_memory()
        oh = torch.empty(n, dtype=torch.float64).pin_memory()
        if reuse:
            torch.addcmul(bh, dh, xh, out=gh)
            with pytest.raises(aa.AAError) as ei:   # nothing to reuse yet
                s.step_host(None, gh, oh)
            assert ei.value.code == 2
        xs = []
        for i in range(9):
            torch.addcmul(bh, dh, xh, out=gh)
            s.step_host(None if (reuse and i > 0) else xh, gh, oh)
            xh, oh = oh, xh
            xs.append(xh.numpy().copy())
        s.close()
        outs.append(xs)
    for a, c in zip(*outs):
        assert np.array_equal(a, c)


@pytest.mark.parametrize("n", [4097, 5_000_003])
def test_step_host_breakdown_then_restart_reuses_device_x(n):
    """The restart policy through aa_step_host (aa.h BREAKDOWN): G(x) = x + 1 makes
    every Delta f exactly 0, so the first AA step breaks down and degrades to x_{i+1} = G(x_i);
    the next aa_step_host refuses at entry (AA_ERR_BREAKDOWN) without consuming its inputs;
    after aa_reset the same call with x_i = NULL finds the device copy of x_{i+1} and again
    returns G(x_i) -- all exact in fp64."""
    stream = torch.cuda.current_stream()
    s = aa.AndersonSolver(n, 3, "dcgs2", stream=stream)
    one = torch.ones(n, dtype=torch.float64)
    x0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    x1 = torch.empty_like(x0)
    s.init(x0, one.cuda(), x1)                       # x1 = G(0) = 1
    xh = x1.cpu().pin_memory()
    gh = torch.empty(n, dtype=torch.float64).pin_memory()
    oh = torch.empty(n, dtype=torch.float64).pin_memory()
    torch.add(xh, one, out=gh)
    s.step_host(xh, gh, oh)                          # Delta f = 0: breakdown, x2 = G(x1) = 2
    assert torch.equal(oh, torch.full_like(oh, 2.0))
    xh, oh = oh, xh
    torch.add(xh, one, out=gh)
    with pytest.raises(aa.AAError) as ei:
        s.step_host(None, gh, oh)
    assert ei.value.code == aa.AA_ERR_BREAKDOWN
    s.reset()
    s.step_host(None, gh, oh)                        # reuses x2 on the device: x3 = G(x2) = 3
    assert torch.equal(oh, torch.full_like(oh, 3.0))
    s.close()
