"""Pins for the oracle's breakdown test (reading A12) and the restart policy (SPEC S:145,
S:215).  The paper is silent on linear dependence in the
window (A12), so the pins are mathematical facts: an exactly dependent column has
R_kk = 0 in exact arithmetic; a column at a known distance from the span has exactly that
R_kk; GMRES on a matrix with two distinct eigenvalues converges exactly at step 2, so AA
(== GMRES) finds its third Delta f dependent; and a restart is Alg. 1 started
afresh from the current iterate."""
import math

import numpy as np
import pytest

from aa_inputs import problems
from oracle import EPS, Ledger, QRState, Reducer, aa_variant, qradd, VARIANTS
from oracle.qr import breakdown_eps_default


def _add_columns(variant, cols, n, m, eps_a=None):
    """Append columns with the variant's QRAdd; returns the breakdown flag of each add."""
    st, led, red = QRState(n, m), Ledger(), Reducer(1)
    st.eps_a = eps_a
    flags = []
    for j, a in enumerate(cols):
        st.breakdown = False
        if j == 0:   # Alg. 2 l.1-2
            r = red.norm(a)
            st.R[0, 0] = r
            st.Q[:, 0] = a / r
            st.T[0, 0] = 1.0
            st.mi = 1
        else:
            qradd(variant, st, a, led, red)
        flags.append(st.breakdown)
    return st, flags


@pytest.mark.parametrize("variant", VARIANTS)
def test_dependent_column_flags_and_perturbed_does_not(variant):
    """A column in the span of the window (R_kk = 0 exactly; in fp64 ~ eps ||v||) must flag;
    the same column moved 1e-3 ||v|| off the span (R_kk / ||v|| ~ 1e-3) must not."""
    n = 400
    rng = np.random.default_rng(12)
    A = rng.standard_normal((n, 3))
    v = A @ np.array([0.3, -1.7, 0.9])
    _, flags = _add_columns(variant, [A[:, 0], A[:, 1], A[:, 2], v], n, 4)
    assert flags == [False, False, False, True]
    w = rng.standard_normal(n)
    w -= A @ np.linalg.lstsq(A, w, rcond=None)[0]            # orthogonal to the span
    v2 = v + 1e-3 * np.linalg.norm(v) * w / np.linalg.norm(w)
    st, flags = _add_columns(variant, [A[:, 0], A[:, 1], A[:, 2], v2], n, 4)
    assert flags == [False, False, False, False]
    assert abs(st.R[3, 3] / np.linalg.norm(v2) - 1e-3) < 1e-6  # R_kk = the distance to the span


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n", [16, 10_000])
def test_threshold_boundary(variant, n):
    """v = e_0 + delta e_2 against the window [e_0, e_1]: every variant's projection is exact,
    so R_kk = delta and ||v|| = 1 in fp64; delta 1 % under eps_a = 10 eps sqrt(n) flags, 1 %
    over does not (the threshold's sqrt(n) and its factor 10 are both pinned)."""
    eps_a = breakdown_eps_default(n)
    assert eps_a == 10.0 * EPS * math.sqrt(n)
    e = np.eye(n)[:, :3]
    for delta, want in ((0.99 * eps_a, True), (1.01 * eps_a, False)):
        v = e[:, 0] + delta * e[:, 2]
        st, flags = _add_columns(variant, [e[:, 0], e[:, 1], v], n, 3)
        assert flags == [False, False, want], (delta, st.R[2, 2])
    # an explicit eps_a (AA_OPT_BREAKDOWN_EPS): ratio 0.2 / sqrt(1.04) = 0.196
    for eps_set, want in ((0.2, True), (0.19, False)):
        v = e[:, 0] + 0.2 * e[:, 2]
        _, flags = _add_columns(variant, [e[:, 0], e[:, 1], v], n, 3, eps_a=eps_set)
        assert flags[-1] == want


def test_nan_and_zero_count_as_breakdown():
    n = 8
    e = np.eye(n)
    _, flags = _add_columns("mgs", [e[:, 0], np.zeros(n)], n, 2, eps_a=0.0)
    assert flags == [False, True]                              # R_kk = 0 <= 0 * ||v||
    _, flags = _add_columns("mgs", [e[:, 0], np.full(n, np.nan)], n, 2)
    assert flags == [False, True]                              # not (NaN > threshold)


@pytest.mark.parametrize("variant", VARIANTS)
def test_lucky_breakdown_two_eigenvalues(variant):
    """G(x) = D x + b with D = diag of two distinct values: GMRES on (I - D) x = b converges
    exactly at step 2 (the minimal polynomial has degree 2), so AA (== GMRES untruncated,
    P:61-62) has x_3 = x* and its third Delta f = f_3 - f_2 = -f_2 lies in the span of the
    first two: the first breakdown is at i = 3, never before; R_kk / ||Delta f|| is at
    rounding level there.  The restart step is x_4 = G(x_3) exactly."""
    n = 10_007
    rng = np.random.default_rng(5)
    d = np.where(rng.random(n) < 0.5, 0.3, -0.5)
    b = rng.uniform(-1.0, 1.0, n)
    xstar = b / (1.0 - d)
    r = aa_variant(lambda x: d * x + b, np.zeros(n), 5, variant, 6, breakdown="restart", record_loo=False)
    assert r.breakdown[:3] == [False, False, True]
    assert r.rratio[2] < 10 * EPS * math.sqrt(n)
    assert np.linalg.norm(r.xs[1] - xstar) <= 1e-13 * np.linalg.norm(xstar)      # x_3 = x*
    x3 = r.xs[1]
    assert np.array_equal(r.xs[2], d * x3 + b)                                   # x_4 = G(x_3)
    assert all(np.isfinite(x).all() for x in r.xs)
    # "record" keeps the dependent column and breaks on it
    rec = aa_variant(lambda x: d * x + b, np.zeros(n), 5, variant, 6, breakdown="record", record_loo=False)
    assert rec.breakdown[:3] == [False, False, True]


@pytest.mark.parametrize("variant", VARIANTS)
def test_restart_is_a_fresh_run_from_the_current_iterate(variant):
    """After a breakdown at step i the restart policy continues exactly like Alg. 1 started
    afresh at x_0' = x_i (x_1' = G(x_i) = the degraded x_{i+1}, f_0' = f_i): compared bitwise
    with a new aa_variant run up to the next breakdown.  eps_a = 0.2 (an artificial threshold)
    makes breakdowns frequent and far from rounding (d in U[0.5, 0.99])."""
    n, m, eps = 20_011, 3, 0.2
    d, b = problems.diagonal(n, 0.5, 0.99)
    G = lambda x: d * x + b
    r = aa_variant(G, np.zeros(n), m, variant, 16, breakdown="restart", breakdown_eps=eps, record_loo=False)
    rr = np.array(r.rratio)
    assert np.min(np.abs(rr / eps - 1.0)) > 1e-3          # every decision is far from the threshold
    bds = [i for i, f in enumerate(r.breakdown) if f]
    assert len(bds) >= 3 and not r.hard_error
    xs = [None, r.x1] + r.xs                              # xs[j] = x_j
    for j in bds:                                        # step i = j + 1 broke down
        i = j + 1
        assert np.array_equal(xs[i + 1], G(xs[i]))        # x_{i+1} = G(x_i) exactly
        nxt = next((q for q in bds if q > j), len(r.breakdown) - 1)
        steps = nxt - j                                   # steps until (and including) the next breakdown
        fresh = aa_variant(G, xs[i], m, variant, steps, breakdown="restart", breakdown_eps=eps,
                           record_loo=False)
        assert np.array_equal(fresh.x1, xs[i + 1])
        for q in range(steps):
            assert np.array_equal(fresh.xs[q], xs[i + 2 + q]), (i, q)
            assert fresh.breakdown[q] == r.breakdown[j + 1 + q]


def test_second_consecutive_breakdown_is_a_hard_error():
    """G(x) = x + u: f_i = u for every i, so Delta f = 0 at the first step (R_00 = 0) and again
    on the first step after the restart: the second consecutive breakdown stops the run
    (S:256).  Both degraded steps are plain fixed-point steps.  u holds small integers, so
    every iterate is an integer vector and f = (x + u) - x = u exactly in fp64."""
    n = 64
    u = np.arange(n, dtype=np.float64) - 32.0
    for variant in VARIANTS:
        r = aa_variant(lambda x: x + u, np.zeros(n), 3, variant, 10, breakdown="restart", record_loo=False)
        assert r.hard_error and r.iters == 2
        assert r.breakdown == [True, True]
        assert np.array_equal(r.xs[0], 2 * u) and np.array_equal(r.xs[1], 3 * u)
