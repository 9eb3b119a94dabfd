"""Pins for the CPU oracle (O1/O2) against what the paper and the mathematics fix.

Each test names the mistake it would catch.  No test compares the oracle with
itself or re-types its formulas; the references are GMRES, exact
rational normal equations, LAPACK Householder QR, the printed sync formulas
(tests/golden/spec_examples.json) and the SPEC worked examples.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import aa_inputs
from aa_inputs import problems
from oracle import (EPS, Ledger, QRState, Reducer, aa_definition, aa_variant, icwy_rebuild_T,
                    icwy_update_T_small, loss_of_orthogonality, lsp_solve, qradd, qrdelete_givens,
                    VARIANTS)
from tests._gmres import gmres_iterates

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _build(variant, A, shards=1, **kw):
    n, m = A.shape
    st, led, red = QRState(n, m), Ledger(), Reducer(shards)
    per_add = []
    for j in range(m):
        before = led.counts["qradd"]
        if j == 0:
            # Alg. 2 l.1-2 (first column): one norm reduction
            r = red.norm(A[:, 0]); led.sync("qradd")
            st.R[0, 0] = r; st.Q[:, 0] = A[:, 0] / r; st.T[0, 0] = 1.0; st.mi = 1
        else:
            qradd(variant, st, A[:, j], led, red, **kw)
        per_add.append(led.counts["qradd"] - before)
    return st, led, per_add


def _signfix(Q, R):
    s = np.sign(np.diag(R))
    s[s == 0] = 1
    return Q * s, (R.T * s).T


# ----------------------------------------------------------------------------- generators
def test_splitmix64_matches_reference_sequence():
    """The counter generator equals SplitMix64 (Steele et al.) computed with Python ints."""
    def ref(state):
        z = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
        return z ^ (z >> 31)
    ctr = np.array([0, 1, 12345, 2**63 + 7, 9667 + (1 << 48)], dtype=np.uint64)
    got = aa_inputs.splitmix64(ctr)
    for c, g in zip(ctr.tolist(), got.tolist()):
        assert g == ref(c)
    # first outputs of the canonical SplitMix64 stream seeded with 0
    assert int(aa_inputs.splitmix64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF
    u = aa_inputs.uniform(10000, -1.0, 1.0, stream=2)
    assert u.min() >= -1.0 and u.max() < 1.0 and abs(u.mean()) < 0.05
    # counter-based: an offset window equals the slice of the full stream
    assert np.array_equal(aa_inputs.uniform(5, 0, 1, stream=1, offset=7),
                          aa_inputs.uniform(12, 0, 1, stream=1)[7:])


def test_shard_bounds_remainder_to_leading_ranks():
    b = aa_inputs.shard_bounds(10, 4)
    assert b == [(0, 3), (3, 3), (6, 2), (8, 2)]


# ----------------------------------------------------------------------------- SPEC examples
def test_spec_hand_examples():
    g = GOLD
    red = Reducer(g["dot_unit"]["shards"])
    assert red.dot(np.array(g["dot_unit"]["a"], float), np.array(g["dot_unit"]["b"], float)) == 1.0
    red = Reducer(g["dot_hand"]["shards"])
    assert red.dot(np.array(g["dot_hand"]["a"], float), np.array(g["dot_hand"]["b"], float)) == 20.0
    Q = np.array(g["fused_multi_dot"]["Q"], float)
    assert np.array_equal(Reducer(1).matT_vec(Q, np.array(g["fused_multi_dot"]["v"], float)),
                          np.array(g["fused_multi_dot"]["value"]))
    assert Reducer(1).norm(np.array(g["norm_hand"]["v"], float)) == 5.0
    # Alg. 2 l.2 through the driver: a 1-iteration run whose Delta f_0 = (3,4,0,0)
    ex = g["first_column"]
    df = np.array(ex["df"], float)
    # choose x0 = 0, G(x0) = c so f0 = c; x1 = c, G(x1) = 2c + df  =>  f1 = c + df, Delta f = df
    c = np.array([1.0, -2.0, 0.5, 3.0])
    G = lambda x: c if not x.any() else 2 * c + df
    r = aa_variant(G, np.zeros(4), 3, "mgs", 1)
    st = r.state
    assert st.R[0, 0] == ex["r00"]
    assert np.allclose(st.Q[:, 0], ex["q"], atol=0, rtol=1e-15)
    assert r.ledgers[0]["qradd"] == 1


def test_mgs_add_e2_hand_case():
    ex = GOLD["mgs_add_e2"]
    A = np.stack([np.array(ex["q0"], float), np.array(ex["v"], float)], axis=1)
    for v in VARIANTS:
        st, led, per = _build(v, A)
        assert np.allclose(st.R[:2, 1], ex["rcol"], atol=1e-15)
        assert np.allclose(st.Q[:, :2], A, atol=1e-15)
    st, led, per = _build("mgs", A)
    assert per[1] == ex["ledger"]


def test_delete_two_column_hand_case():
    ex = GOLD["delete_two_columns"]
    A = np.stack([np.array(ex["v1"], float), np.array(ex["v2"], float)], axis=1)
    for v in VARIANTS:
        st, led, _ = _build(v, A)
        before = led.snapshot()
        qrdelete_givens(st)
        assert led.snapshot() == before            # no communication
        assert st.mi == 1
        assert np.allclose(st.Q[:, 0], ex["q"], atol=1e-15)
        assert abs(st.R[0, 0] - ex["r"]) < 1e-15


def test_scalar_linear_m1_all_variants():
    ex = GOLD["scalar_linear_m1"]
    G = lambda x: ex["a"] * x + ex["b"]
    outs = []
    for v in VARIANTS:
        r = aa_variant(G, np.zeros(1), 1, v, 4, tol=1e-14)
        assert abs(r.xs[0][0] - ex["x2"]) < 1e-15   # x_2 is the fixed point
        outs.append(np.array([x[0] for x in r.xs]))
    o1 = aa_definition(G, np.zeros(1), 1, 4, tol=1e-14)
    assert abs(o1.xs[0][0] - ex["x2"]) < 1e-15
    for o in outs[1:]:
        assert np.allclose(o[:1], outs[0][:1], rtol=1e-12)


def test_constant_map_converges_in_two():
    b = np.array(GOLD["constant_map"]["b"])
    G = lambda x: b.copy()
    for v in VARIANTS:
        r = aa_variant(G, np.zeros(3), 3, v, 10, tol=1e-12)
        assert r.converged and r.iters <= 2
        assert np.array_equal(r.x, b)
    r = aa_definition(G, np.zeros(3), 3, 10, tol=1e-12)
    assert r.converged and r.iters <= 2 and np.array_equal(r.x, b)


# ----------------------------------------------------------------------------- exact LS
def _rational_normal_equations(F, f):
    k = F.shape[1]
    A = [[sum(Fraction(int(F[r, i])) * Fraction(int(F[r, j])) for r in range(F.shape[0]))
          for j in range(k)] for i in range(k)]
    y = [sum(Fraction(int(F[r, i])) * Fraction(int(f[r])) for r in range(F.shape[0])) for i in range(k)]
    # Gauss-Jordan in exact arithmetic
    M = [row[:] + [y[i]] for i, row in enumerate(A)]
    for c in range(k):
        p = next(r for r in range(c, k) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        piv = M[c][c]
        M[c] = [v / piv for v in M[c]]
        for r in range(k):
            if r != c and M[r][c] != 0:
                fac = M[r][c]
                M[r] = [a - fac * b for a, b in zip(M[r], M[c])]
    return np.array([float(M[i][k]) for i in range(k)])


@pytest.mark.parametrize("seed", range(6))
def test_lsp_matches_exact_rational_normal_equations(seed):
    """gamma from O2's incremental QR + Alg. 2 l.9 and from O1 equals the exact
    normal-equation solution (catches a transposed R, a wrong back-substitution
    order or a dropped Q^T f term)."""
    rng = np.random.default_rng(seed)
    n, k = 7, 3
    F = rng.integers(-5, 6, size=(n, k)).astype(float)
    while np.linalg.matrix_rank(F) < k:
        F = rng.integers(-5, 6, size=(n, k)).astype(float)
    f = rng.integers(-9, 10, size=n).astype(float)
    exact = _rational_normal_equations(F, f)
    from oracle.aa import _householder_lsq
    assert np.allclose(_householder_lsq(F, f), exact, rtol=1e-12, atol=1e-13)
    for v in VARIANTS:
        st, led, _ = _build(v, F)
        gam = lsp_solve(st, f, Ledger(), Reducer(1))
        assert np.allclose(gam, exact, rtol=1e-11, atol=1e-12), v


# ----------------------------------------------------------------------------- QR kernels
@pytest.mark.parametrize("variant", VARIANTS)
def test_qradd_matches_householder(variant):
    """Alg. 3-6 reproduce LAPACK Householder QR (sign-normalised) on kappa <= 1e2
     and cost exactly the printed number of reductions per add."""
    for seed in range(10):
        A = problems.ortho_test_matrix(300, 8, 1e2, seed=seed)
        st, led, per = _build(variant, A)
        Qh, Rh = _signfix(*np.linalg.qr(A))
        assert np.max(np.abs(st.R - Rh)) <= 1e-10 * np.max(np.abs(Rh))
        assert np.max(np.abs(st.Q - Qh)) <= 1e-10
        want = {"mgs": [j + 1 for j in range(8)], "icwy": [1] + [2] * 7,
                "cgs2": [1] + [3] * 7, "dcgs2": [1] + [2] * 7}[variant]
        assert per == want


@pytest.mark.parametrize("opt", [dict(dcgs2_rscale=True), dict(dcgs2_cond=2)])
def test_dcgs2_options_match_householder(opt):
    """DCGS-2 with the consistent R update (reading A3) or reorthogonalising from m_i > 2
    (reading A2) still reproduces LAPACK Householder QR at kappa <= 1e2; cond = 2 costs 2
    reductions per add from the third column (the first two adds are unchanged)."""
    for seed in range(5):
        A = problems.ortho_test_matrix(300, 8, 1e2, seed=seed)
        st, led, per = _build("dcgs2", A, **opt)
        Qh, Rh = _signfix(*np.linalg.qr(A))
        assert np.max(np.abs(st.R - Rh)) <= 1e-10 * np.max(np.abs(Rh))
        assert np.max(np.abs(st.Q - Qh)) <= 1e-10
        assert per == [1] + [2] * 7


def test_dcgs2_rscale_keeps_the_factorisation_consistent():
    """Reading A3 (SURVEY Pr5): at kappa = 1e6 the printed update R += s leaves F != QR at a
    level far above rounding, while R += R_kk s keeps ||A - QR||/||A|| at rounding level;
    the loss of orthogonality is the same class for both (the R update does not touch Q)."""
    A = problems.ortho_test_matrix(1500, 30, 1e6, seed=2)
    res = lambda st: np.linalg.norm(A - st.Q @ st.R) / np.linalg.norm(A)
    st_v, _, _ = _build("dcgs2", A)
    st_r, _, _ = _build("dcgs2", A, dcgs2_rscale=True)
    assert res(st_r) <= 1e-14, res(st_r)
    assert res(st_v) >= 1e3 * res(st_r), (res(st_v), res(st_r))
    lv, lr = loss_of_orthogonality(st_v.Q), loss_of_orthogonality(st_r.Q)
    assert lv == lr


def test_dcgs2_verbatim_r_update_is_plus_s():
    """Pins Alg. 6 l.5 as printed, R_{0:k-2,k-1} += s (reading A3), against a wrong sign, a
    missing update or a scaled one -- by scale equivariance, not by retyping the formula.
    Scaling F by 2 scales every dot product, norm and R entry by exactly 2 and leaves Q (so
    s = Q^T q, from normalised columns) bitwise unchanged: for the verbatim update
    D = 2 R(F) - R(2F) is then exactly the s added to each column, the consistent update
    (R += R_kk s) gives D = 0, and the two runs differ by R_rscale - R_verbatim = (R_kk - 1) s
    = (R_kk - 1) D column by column.  F is scaled by 2^20 first (exact), so R_kk >> 1 and a
    wrong sign (which would give R_rscale - R_verbatim = -(R_kk + 1) D) is far off."""
    A = problems.ortho_test_matrix(600, 14, 1e8, seed=4) * 2.0 ** 20
    Qv, Rv = (lambda st: (st.Q, st.R))(_build("dcgs2", A)[0])
    Qv2, Rv2 = (lambda st: (st.Q, st.R))(_build("dcgs2", 2.0 * A)[0])
    Rr, Rr2 = _build("dcgs2", A, dcgs2_rscale=True)[0].R, _build("dcgs2", 2.0 * A, dcgs2_rscale=True)[0].R
    assert np.array_equal(Qv, Qv2)
    assert np.array_equal(2.0 * Rr, Rr2)   # the consistent update is scale-equivariant
    D, E = 2.0 * Rv - Rv2, Rr - Rv
    checked = 0
    for j in range(2, 13):   # columns updated by a later reorthogonalisation (m_i > 3)
        d, e, rkk = D[:j, j], E[:j, j], Rv[j, j]
        assert rkk == Rr[j, j]
        col = np.max(np.abs(Rv[:j, j]))
        if np.max(np.abs(d)) < 1e4 * EPS * col:   # s still at rounding level in this column
            continue
        assert np.max(np.abs(e - (rkk - 1.0) * d)) <= 1e-3 * np.max(np.abs(e)), j
        assert np.max(np.abs(e + (rkk + 1.0) * d)) >= 0.5 * np.max(np.abs(e)), j   # (discriminates)
        checked += 1
    assert checked >= 4, checked


@pytest.mark.parametrize("kappa", [1e1, 1e3, 1e6, 1e9])
def test_loss_of_orthogonality_classes(kappa):
    """S:211 with c = 100, n = 500, m = 20: MGS, ICWY <= c eps kappa;
    CGS-2 <= c eps; DCGS-2 <= c eps kappa^2."""
    A = problems.ortho_test_matrix(500, 20, kappa, seed=7)
    c = 100.0
    loo = {v: loss_of_orthogonality(_build(v, A)[0].Q) for v in VARIANTS}
    assert loo["mgs"] <= c * EPS * kappa
    assert loo["icwy"] <= c * EPS * kappa
    assert loo["cgs2"] <= c * EPS
    assert loo["dcgs2"] <= c * EPS * kappa ** 2
    if kappa >= 1e6:
        # the classes are distinct: MGS/ICWY really lose orthogonality, CGS-2 does not
        assert loo["mgs"] > 1e3 * loo["cgs2"]
        assert loo["icwy"] > 1e3 * loo["cgs2"]


def test_qrdelete_reproduces_retained_columns():
    """Givens QRDelete: Q'R' = F[:, 1:] to 1e-12 and equals Householder QR of the
    retained columns (positive diagonal); zero ledger increments."""
    A = problems.ortho_test_matrix(100, 5, 1e3, seed=3)
    for v in VARIANTS:
        st, led, _ = _build(v, A)
        before = led.snapshot()
        qrdelete_givens(st)
        assert led.snapshot() == before
        k = st.mi
        assert k == 4
        F = A[:, 1:]
        assert np.max(np.abs(st.Q[:, :k] @ st.R[:k, :k] - F)) <= 1e-12 * np.max(np.abs(F))
        assert np.all(np.diag(st.R[:k, :k]) > 0)
        assert np.allclose(np.triu(st.R[:k, :k]), st.R[:k, :k])
        Qh, Rh = _signfix(*np.linalg.qr(F))
        assert np.max(np.abs(st.R[:k, :k] - Rh)) <= 1e-10 * np.max(np.abs(Rh))


def test_icwy_T_rebuild():
    """Orthonormal Q => rebuilt T = I; rebuilt strict-lower equals the dense
    Q^T Q strict lower; exactly one qrdelete reduction."""
    A = problems.ortho_test_matrix(200, 6, 1e4, seed=1)
    st, led, _ = _build("icwy", A)
    qrdelete_givens(st)
    before = led.counts["qrdelete"]
    icwy_rebuild_T(st, led, Reducer(1))
    assert led.counts["qrdelete"] - before == 1
    k = st.mi
    Q = st.Q[:, :k]
    dense = Q.T @ Q
    for i in range(k):
        assert st.T[i, i] == 1.0
        for j in range(k):
            if j < i:
                assert abs(st.T[i, j] - dense[i, j]) <= 1e-14
            elif j > i:
                assert st.T[i, j] == 0.0
    st2 = QRState(50, 3)
    st2.Q[:, :3] = np.linalg.qr(np.random.default_rng(0).standard_normal((50, 3)))[0]
    st2.mi = 3
    icwy_rebuild_T(st2, Ledger(), Reducer(1))
    assert np.max(np.abs(st2.T - np.eye(3))) <= 1e-15


def test_icwy_small_update_equals_gram_of_rotated_q():
    """Reduction-free T update (variant): with unit-norm but
    NON-orthogonal Q and T = I + strict_lower(Q^T Q) on the known rows 0..m_i-2, the
    updated rows 0..k-2 equal the strict lower part of the explicit Gram of the rotated
    Q' that qrdelete_givens produced (the paper's rebuild), and row k-1 is the
    identity row.  Catches a wrong rotation sign or order, a transposed W, and an
    off-by-one in the rows of T it reads."""
    rng = np.random.default_rng(5)
    n, mi = 40, 7
    st = QRState(n, mi)
    Q = rng.standard_normal((n, mi)) + 0.8 * rng.standard_normal((n, 1))   # correlated
    Q /= np.linalg.norm(Q, axis=0)
    st.Q[:, :] = Q
    st.R[:, :] = np.triu(rng.standard_normal((mi, mi)))
    st.R[np.diag_indices(mi)] = np.abs(np.diag(st.R)) + 1.0
    G0 = Q.T @ Q
    st.T[:, :] = np.eye(mi)
    st.T[:mi - 1, :mi - 1] += np.tril(G0[:mi - 1, :mi - 1], -1)   # row mi-1 unknown
    st.mi = mi
    rots = qrdelete_givens(st)
    assert len(rots) == mi - 1
    icwy_update_T_small(st, rots)
    k = st.mi
    Qp = st.Q[:, :k]
    Gp = Qp.T @ Qp
    assert np.max(np.abs(G0 - np.eye(mi))) > 0.3          # the test is not vacuous
    for i in range(k):
        assert st.T[i, i] == 1.0
        for j in range(k):
            if i == k - 1 and j < i:
                assert st.T[i, j] == 0.0
            elif j < i:
                assert abs(st.T[i, j] - Gp[i, j]) <= 1e-14, (i, j, st.T[i, j], Gp[i, j])
            elif j > i:
                assert st.T[i, j] == 0.0


def test_icwy_small_update_aa_agrees_with_rebuild():
    """AA with the reduction-free update follows the paper's rebuild to rounding on a
    well-conditioned problem and needs no qrdelete reduction; on the SURVEY Pr6
    ill-conditioned window (d in U[0.9, 0.99], LOO ~ 0.3) both converge."""
    d, b = problems.diagonal(600, -0.9, 0.9)
    G = lambda x: d * x + b
    ra = aa_variant(G, np.zeros(600), 5, "icwy", 30)
    rs = aa_variant(G, np.zeros(600), 5, "icwy", 30, icwy_delete="small")
    for xa, xs in zip(ra.xs, rs.xs):
        assert np.linalg.norm(xa - xs) <= 1e-10 * np.linalg.norm(xa)
    assert ra.ledgers[-1]["qrdelete"] == 30 - 5 and rs.ledgers[-1]["qrdelete"] == 0
    assert ra.ledgers[-1]["qradd"] == rs.ledgers[-1]["qradd"]
    d2, b2 = problems.diagonal(4000, 0.9, 0.99, seed=11)
    G2 = lambda x: d2 * x + b2
    r2a = aa_variant(G2, np.zeros(4000), 20, "icwy", 80, record_x=False)
    r2s = aa_variant(G2, np.zeros(4000), 20, "icwy", 80, record_x=False, icwy_delete="small")
    f0 = r2a.f_norms[0]
    assert r2a.f_norms[-1] <= 1e-9 * f0 and r2s.f_norms[-1] <= 1e-9 * f0, (r2a.f_norms[-1], r2s.f_norms[-1])


# ----------------------------------------------------------------------------- AA driver
def test_aa_equals_gmres_on_linear_problem():
    """AA with an untruncated window is GMRES: x_{i+1} = M x_i^GMRES + b.
    Catches a wrong sign in f = G(x) - x, an off-by-one in the window, or a
    mis-paired Delta g / Delta f column."""
    n = 200
    M, b = problems.linear_dense(n, 0.95)
    G = lambda x: M @ x + b
    A = np.eye(n) - M
    K = 25
    xg = gmres_iterates(A, b, np.zeros(n), K)
    runs = [aa_definition(G, np.zeros(n), 30, K)]
    runs += [aa_variant(G, np.zeros(n), 30, v, K) for v in VARIANTS]
    for r in runs:
        for i in range(1, K + 1):
            pred = M @ xg[i] + b
            xi1 = r.xs[i - 1]                     # x_{i+1}
            assert np.linalg.norm(xi1 - pred) <= 1e-10 * np.linalg.norm(pred), i
    # with m = 5 the relation holds until the window truncates (i <= 5)
    r = aa_variant(G, np.zeros(n), 5, "cgs2", 8)
    for i in range(1, 6):
        pred = M @ xg[i] + b
        assert np.linalg.norm(r.xs[i - 1] - pred) <= 1e-10 * np.linalg.norm(pred)
    i = 7
    assert np.linalg.norm(r.xs[i - 1] - (M @ xg[i] + b)) > 1e-8 * np.linalg.norm(r.xs[i - 1])


def test_sync_counts_match_paper_formulas():
    """Ledger over the start-up phase equals P:536-540 exactly; recycle counts equal
    P:241-243, P:312-325, P:380-383, P:424-425 (catches a dropped or merged sync)."""
    g = GOLD["startup_syncs"]
    n = 120
    d, bb = problems.diagonal(n, -0.9, 0.9)
    G = lambda x: d * x + bb
    for mi_, m in enumerate(g["m"]):
        for v in VARIANTS:
            r = aa_variant(G, np.zeros(n), m, v, m + 3, record_loo=False)
            L = r.ledgers
            startup = L[m - 1]["qradd"] + L[m - 1]["qrdelete"]
            assert startup == g[v][mi_], (v, m)
            for it in (m, m + 1, m + 2):        # recycle iterations (0-based index it = i-1)
                dq = L[it]["qradd"] - L[it - 1]["qradd"]
                dd = L[it]["qrdelete"] - L[it - 1]["qrdelete"]
                want = GOLD["recycle_syncs"]["qradd"][v]
                want = m if want == "m" else want
                assert dq == want, (v, m)
                assert dd == GOLD["recycle_syncs"]["qrdelete"][v]
                assert L[it]["lsp_rhs"] - L[it - 1]["lsp_rhs"] == 1
                assert L[it]["norm_check"] - L[it - 1]["norm_check"] == 1


def test_o2_matches_o1_and_shards_on_config1_problem():
    """Config-1 family (n=1000, m=5, ||M||=0.95): every variant reproduces the
    definition oracle to 1e-12 over 30 truncated iterations, independent of the
    simulated shard count."""
    n = 1000
    M, b = problems.linear_dense(n, 0.95)
    G = lambda x: M @ x + b
    o1 = aa_definition(G, np.zeros(n), 5, 30)
    for v in VARIANTS:
        for p in (1, 4):
            r = aa_variant(G, np.zeros(n), 5, v, 30, shards=p, record_loo=(p == 1))
            for a, bref in zip(r.xs, o1.xs):
                assert np.linalg.norm(a - bref) <= 1e-12 * np.linalg.norm(bref)
            if p == 1:
                assert max(r.loo) < 1e-13


def test_iteration_count_config1():
    """Config 1 run (ii): tol 1e-6 on ||dx||_2 -> identical counts for every variant and O1."""
    n = 1000
    M, b = problems.linear_dense(n, 0.95)
    G = lambda x: M @ x + b
    o1 = aa_definition(G, np.zeros(n), 5, 200, tol=1e-6, record_x=False)
    assert o1.converged
    for v in VARIANTS:
        r = aa_variant(G, np.zeros(n), 5, v, 200, tol=1e-6, record_x=False, record_loo=False)
        assert r.converged and r.iters == o1.iters


def test_damping_identity():
    """Reading A13: g - G gamma - (1-beta)(f - F gamma) equals the textbook damped AA
    (1-beta)(x_i - X gamma) + beta (g_i - G gamma) with X the Delta x window."""
    n = 300
    M, b = problems.linear_dense(n, 0.9, seed=5)
    G = lambda x: M @ x + b
    beta = 0.6
    o1 = aa_definition(G, np.zeros(n), 4, 12, beta=beta)
    # textbook recursion with explicit Delta x window
    x0 = np.zeros(n)
    gprev = G(x0); fprev = gprev - x0; xprev = x0; x = gprev.copy()
    dX, dF, dG = [], [], []
    for i in range(1, 13):
        g = G(x); f = g - x
        dX.append(x - xprev); dF.append(f - fprev); dG.append(g - gprev)
        dX, dF, dG = dX[-4:], dF[-4:], dG[-4:]
        F = np.stack(dF, 1)
        gam = np.linalg.lstsq(F, f, rcond=None)[0]
        xn = (1 - beta) * (x - np.stack(dX, 1) @ gam) + beta * (g - np.stack(dG, 1) @ gam)
        assert np.linalg.norm(xn - o1.xs[i - 1]) <= 1e-10 * np.linalg.norm(xn)
        xprev, x, fprev, gprev = x, xn, f, g
    for v in VARIANTS:
        r = aa_variant(G, np.zeros(n), 4, v, 12, beta=beta, record_loo=False)
        for a, bref in zip(r.xs, o1.xs):
            assert np.linalg.norm(a - bref) <= 1e-11 * np.linalg.norm(bref)


def test_block_constant_reduction_property():
    """AA is invariant under the isometry y = sqrt(w) * x: a block-constant problem of
    size sum(w) has iterates equal to the weighted small problem's (used by the
    full-size GPU parity test)."""
    w, d, bb = problems.block_constant(5000, 40)
    big_d, big_b = np.repeat(d, w), np.repeat(bb, w)
    sw = np.sqrt(w.astype(float))
    Gbig = lambda x: big_d * x + big_b
    Gsmall = lambda y: d * y + sw * bb
    for v in ("mgs", "dcgs2"):
        rb = aa_variant(Gbig, np.zeros(5000), 5, v, 15, record_loo=False)
        rs = aa_variant(Gsmall, np.zeros(40), 5, v, 15, record_loo=False)
        for xb, ys in zip(rb.xs, rs.xs):
            assert np.linalg.norm(xb - np.repeat(ys / sw, w)) <= 1e-12 * np.linalg.norm(xb)


def test_loss_of_orthogonality_closed_forms():
    """||I - Q^T Q||_F on cases with closed forms: two unit columns at
    angle theta give sqrt(2) |cos theta|; a column of norm 2 gives |1 - 4| = 3; an exactly
    orthonormal Q (a permutation) gives 0."""
    from oracle.qr import loss_of_orthogonality
    for theta in (0.3, 1.0, np.pi / 2):
        Q = np.zeros((5, 2))
        Q[0, 0] = 1.0
        Q[0, 1], Q[1, 1] = np.cos(theta), np.sin(theta)
        assert abs(loss_of_orthogonality(Q) - np.sqrt(2.0) * abs(np.cos(theta))) <= 4 * EPS
    assert loss_of_orthogonality(2.0 * np.eye(3)[:, :1]) == 3.0
    assert loss_of_orthogonality(np.eye(6)[:, [3, 0, 5]]) == 0.0


def test_triangular_solves_match_a_library_routine():
    """The oracle's substitutions (LSP back-substitution, Alg. 2 l.9; ICWY's unit-lower
    forward solve with T, Alg. 4 l.4) against scipy's LAPACK trsv on random well-conditioned
    systems, and exactly on an integer unit-lower system with a known solution."""
    from scipy.linalg import solve_triangular
    from oracle.qr import back_substitution, forward_substitution_unit_lower
    rng = np.random.default_rng(11)
    for k in (1, 2, 7, 20):
        R = np.triu(rng.standard_normal((k, k))) + 4.0 * np.eye(k)
        c = rng.standard_normal(k)
        assert np.allclose(back_substitution(R, c), solve_triangular(R, c, lower=False), rtol=1e-13, atol=1e-14)
        T = np.tril(rng.standard_normal((k, k)), -1) * 0.3 + np.eye(k)
        s = rng.standard_normal(k)
        assert np.allclose(forward_substitution_unit_lower(T, s),
                           solve_triangular(T, s, lower=True, unit_diagonal=True), rtol=1e-13, atol=1e-14)
    T = np.array([[1.0, 0, 0], [2.0, 1.0, 0], [-1.0, 3.0, 1.0]])
    x = np.array([1.0, -2.0, 5.0])
    assert np.array_equal(forward_substitution_unit_lower(T, T @ x), x)


def test_sharded_reducer_is_exact_on_integers_and_splits_like_spec():
    """The simulated shards: on integer data every partial and total is
    exact, so p shards give the plain sums bitwise for every reduction shape; the shard
    bounds put the remainder rows on the leading ranks."""
    rng = np.random.default_rng(5)
    n, k = 1003, 6
    A = rng.integers(-50, 50, size=(n, k)).astype(np.float64)
    B = rng.integers(-50, 50, size=(n, 2)).astype(np.float64)
    v = rng.integers(-50, 50, size=n).astype(np.float64)
    exact_dot = int(sum(int(a) * int(b) for a, b in zip(v, A[:, 0])))
    for p in (1, 2, 3, 7, 1003):
        red = Reducer(p)
        assert red.dot(v, A[:, 0]) == exact_dot
        assert np.array_equal(red.matT_vec(A, v), A.T @ v)
        assert np.array_equal(red.matT_mat(A, B), A.T @ B)
        assert np.array_equal(red.gram(A), A.T @ A)
        bounds = list(red._bounds(n))
        lens = [hi - lo for lo, hi in bounds]
        assert bounds[0][0] == 0 and bounds[-1][1] == n and sum(lens) == n
        assert max(lens) - min(lens) <= 1 and lens == sorted(lens, reverse=True)
