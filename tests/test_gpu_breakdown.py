"""Breakdown (reading A12) through libaa vs the oracle's restart policy (SPEC S:145, S:215,
S:256): the GPU detects R_kk <= eps_a ||Delta f|| in K4, degrades the
step to x_{i+1} = G(x_i), keeps the flag until aa_reset, refuses aa_step while it is set
(1 rank), and the caller restarts once (a second consecutive breakdown is a hard error).
The flag sequence and every iterate are compared with oracle.aa_variant(breakdown="restart")."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from aa_inputs import problems  # noqa: E402
from oracle import EPS, aa_variant  # noqa: E402
from paper_2110_09667_b200 import aa  # noqa: E402

VARIANTS5 = [("mgs", {}), ("icwy", {}), ("icwy", {"icwy_delete": "small"}), ("cgs2", {}), ("dcgs2", {})]


def _oracle_kw(opts):
    return {"icwy_delete": "small"} if opts.get("icwy_delete") == "small" else {}


def run_restart(Gt, x0, m, variant, iters, **opts):
    """The caller's loop of Alg. 1 with SPEC's restart policy on top of libaa."""
    n = x0.shape[0]
    s = aa.AndersonSolver(n, m, variant, stream=torch.cuda.current_stream(), **opts)
    x = torch.as_tensor(x0, dtype=torch.float64, device="cuda").clone()
    xn = torch.empty_like(x)
    s.init(x, Gt(x), xn)
    x, xn = xn, x
    xs, flags, hard, restarted = [], [], False, False
    for _ in range(iters):
        s.step(x, Gt(x), xn)
        st = s.stats()
        flags.append(st.breakdown)
        xs.append(xn.cpu().numpy())
        x, xn = xn, x
        if st.breakdown:
            if restarted:
                hard = True
                break
            restarted = True
            s.reset()
            assert not s.stats().breakdown
        else:
            restarted = False
    s.close()
    return xs, flags, hard


@pytest.mark.parametrize("variant,opts", VARIANTS5)
@pytest.mark.parametrize("m,eps", [(2, 0.2), (3, 0.2), (2, 0.5)])
def test_restart_policy_matches_oracle(variant, opts, m, eps):
    """eps_a = 0.2 / 0.5 (AA_OPT_BREAKDOWN_EPS) on d in U[0.5, 0.99]: breakdowns at steps the
    oracle decides with a margin >= 5 % from the threshold, restarts, and (m = 2, eps 0.2)
    recycle steps after the restart."""
    n, iters = 100_003, 20
    d, b = problems.diagonal(n, 0.5, 0.99)
    ref = aa_variant(lambda x: d * x + b, np.zeros(n), m, variant, iters, breakdown="restart",
                     breakdown_eps=eps, record_loo=False, **_oracle_kw(opts))
    assert np.min(np.abs(np.array(ref.rratio) / eps - 1.0)) > 0.04
    dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
    xs, flags, hard = run_restart(lambda x: dt * x + bt, np.zeros(n), m, variant, iters, breakdown_eps=eps, **opts)
    assert flags == ref.breakdown and hard == ref.hard_error
    assert any(flags)
    for a, r in zip(xs, ref.xs):
        assert np.isfinite(a).all()
        assert np.linalg.norm(a - r) <= 1e-10 * np.linalg.norm(r)


@pytest.mark.parametrize("variant,opts", VARIANTS5)
def test_lucky_breakdown_default_threshold(variant, opts):
    """Two distinct eigenvalues: AA == GMRES converges exactly at step 2, the third Delta f is
    dependent (R_kk / ||Delta f|| at rounding level, under 10 eps sqrt(n)): flagged at i = 3
    by the default threshold, x_4 = G(x_3), and every iterate stays finite and matches."""
    n, m, iters = 10_007, 5, 6
    rng = np.random.default_rng(5)
    d = np.where(rng.random(n) < 0.5, 0.3, -0.5)
    b = rng.uniform(-1.0, 1.0, n)
    ref = aa_variant(lambda x: d * x + b, np.zeros(n), m, variant, iters, breakdown="restart",
                     record_loo=False, **_oracle_kw(opts))
    dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
    xs, flags, hard = run_restart(lambda x: dt * x + bt, np.zeros(n), m, variant, iters, **opts)
    assert flags[:3] == [False, False, True] == ref.breakdown[:3]
    assert not hard
    for a, r in zip(xs, ref.xs):
        assert np.isfinite(a).all()
        assert np.linalg.norm(a - r) <= 1e-10 * np.linalg.norm(r)
    assert np.array_equal(xs[2], (dt * torch.tensor(xs[1], device="cuda") + bt).cpu().numpy())


@pytest.mark.parametrize("variant,opts", VARIANTS5)
def test_qradd_dependent_and_boundary_columns(variant, opts):
    """aa_test_qradd (config 5a's hook): a column in the span of the window flags, the same
    column 1e-3 off the span does not; the default threshold eps_a = 10 eps sqrt(n) is hit
    1 % under / over by v = e_0 + delta e_2 against [e_0, e_1] -- the GPU agrees with the
    oracle's decision in every case."""
    from oracle import QRState, Ledger, Reducer, qradd
    n = 4097
    rng = np.random.default_rng(12)
    A = rng.standard_normal((n, 3))
    v = A @ np.array([0.3, -1.7, 0.9])
    w = rng.standard_normal(n)
    w -= A @ np.linalg.lstsq(A, w, rcond=None)[0]
    v2 = v + 1e-3 * np.linalg.norm(v) * w / np.linalg.norm(w)
    eps_a = 10 * EPS * np.sqrt(n)
    e = np.eye(n)[:, :3]
    cases = [([A[:, 0], A[:, 1], A[:, 2], v], True), ([A[:, 0], A[:, 1], A[:, 2], v2], False),
             ([e[:, 0], e[:, 1], e[:, 0] + 0.99 * eps_a * e[:, 2]], True),
             ([e[:, 0], e[:, 1], e[:, 0] + 1.01 * eps_a * e[:, 2]], False)]
    for cols, want in cases:
        # the oracle's decision on the same columns
        st, led, red = QRState(n, 4), Ledger(), Reducer(1)
        r0 = red.norm(cols[0])
        st.R[0, 0], st.Q[:, 0], st.T[0, 0], st.mi = r0, cols[0] / r0, 1.0, 1
        for c in cols[1:]:
            st.breakdown = False
            qradd(variant, st, c, led, red)
        assert st.breakdown == want
        s = aa.AndersonSolver(n, 4, variant, stream=torch.cuda.current_stream(), **opts)
        z = torch.zeros(n, dtype=torch.float64, device="cuda")
        s.init(z, z, torch.empty_like(z))
        got = []
        for c in cols:
            aa.aa_test_qradd(s.h, torch.tensor(c, device="cuda"))
            got.append(s.stats().breakdown)
        s.close()
        assert got == [False] * (len(cols) - 1) + [want], (variant, want, got)


def test_degraded_steps_until_reset_and_entry_poll():
    """Without a reset the flag stays: aa_step refuses at entry once the flag is visible
    (AA_ERR_BREAKDOWN, nothing enqueued, handle not failed); a step enqueued before it was
    visible degrades to x_{i+1} = G(x_i) bitwise; aa_reset clears it and the run continues."""
    n, m, eps = 100_003, 2, 0.5
    d, b = problems.diagonal(n, 0.5, 0.99)
    dt, bt = torch.tensor(d, device="cuda"), torch.tensor(b, device="cuda")
    s = aa.AndersonSolver(n, m, "dcgs2", stream=torch.cuda.current_stream(), breakdown_eps=eps)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    xn = torch.empty_like(x)
    s.init(x, dt * x + bt, xn)
    x, xn = xn, x
    s.step(x, dt * x + bt, xn)          # i = 1: no breakdown (k = 0)
    x, xn = xn, x
    s.step(x, dt * x + bt, xn)          # i = 2: breaks down (oracle: ratio 0.26 < 0.5)
    x, xn = xn, x
    accepted = True
    g = dt * x + bt
    try:
        s.step(x, g, xn)                # may be enqueued before K4 of step 2 has run
    except aa.AAError as e:
        assert e.code == aa.AA_ERR_BREAKDOWN
        accepted = False
    torch.cuda.synchronize()
    if accepted:
        assert torch.equal(xn, g)       # degraded: x_{i+1} = G(x_i) exactly
    st = s.stats()
    assert st.breakdown and st.breakdown_count == 1
    with pytest.raises(aa.AAError) as ei:
        s.step(x, dt * x + bt, xn)
    assert ei.value.code == aa.AA_ERR_BREAKDOWN
    s.reset()
    st = s.stats()
    assert not st.breakdown and st.m_i == 0 and st.breakdown_count == 1
    s.step(x, dt * x + bt, xn)          # the i = 1 branch again
    assert s.stats().m_i == 1
    s.close()


@pytest.mark.parametrize("variant", ["mgs", "icwy", "cgs2", "dcgs2"])
def test_second_consecutive_breakdown_and_damping(variant):
    """G(x) = x + u with integer u: Delta f = 0 exactly at the first step and again right after
    the restart (hard error, like the oracle); the degraded steps are G(x_i) exactly even with
    damping beta = 0.5 (a restart is Alg. 1 l.1, undamped)."""
    n = 4097
    u = np.arange(n, dtype=np.float64) - 2048.0
    ut = torch.tensor(u, device="cuda")
    ref = aa_variant(lambda x: x + u, np.zeros(n), 3, variant, 10, breakdown="restart", record_loo=False)
    for beta in (None, 0.5):
        xs, flags, hard = run_restart(lambda x: x + ut, np.zeros(n), 3, variant, 10, beta=beta)
        assert hard and flags == [True, True] == ref.breakdown
        assert np.array_equal(xs[0], 2 * u) and np.array_equal(xs[1], 3 * u)
