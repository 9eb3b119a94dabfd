"""Heat + nonlinear term workload (§5.1) on the oracle: pins of the harness map G
and the AA behaviour the paper reports (bands; exact paper counts are 'parity unpinned':
the paper used PCG+PFMG at 1024^2, reading A19)."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from aa_inputs import problems as P
from oracle import aa_variant, VARIANTS


def _laplacian(N):
    h = 1.0 / (N + 1)
    T = sp.diags([np.ones(N - 1), -2 * np.ones(N), np.ones(N - 1)], [-1, 0, 1]) / h ** 2
    I = sp.identity(N)
    return (sp.kron(I, T) + sp.kron(T, I)).tocsc()


def test_dst_solve_equals_sparse_direct_solve():
    N = 15
    rng = np.random.default_rng(0)
    r = rng.standard_normal(N * N)
    A = _laplacian(N)
    assert np.allclose(P.laplacian_solve(r, N), spla.spsolve(A, r), rtol=1e-12, atol=1e-14)


def test_stencil_eigenpairs_and_hand_case():
    N = 15
    A = _laplacian(N)
    h = 1.0 / (N + 1)
    i = np.arange(1, N + 1) * h
    for k, l in ((1, 1), (3, 7)):
        v = np.outer(np.sin(l * np.pi * i), np.sin(k * np.pi * i)).ravel()   # rows = y (index l)
        lam = P.laplacian_eigs(N)[l - 1, k - 1]
        assert np.allclose(A @ v, lam * v, rtol=1e-12, atol=1e-9)
    # nx = ny = 3, u = e_center -> (-Laplacian) u has 4/h^2 at the centre, -1/h^2 at the cross
    A3 = _laplacian(3)
    e = np.zeros(9); e[4] = 1.0
    out = -(A3 @ e)
    h3 = 0.25
    assert np.isclose(out[4], 4 / h3 ** 2) and np.allclose(out[[1, 3, 5, 7]], -1 / h3 ** 2)


def test_discretisation_error_is_second_order():
    errs = []
    for N in (31, 63):
        b = P.heat_rhs(N, 1)
        u = P.heat_u_exact(N)
        # residual of the discrete system at u_exact: A u + c(u) - b
        res = _laplacian(N) @ u + P.heat_c(u, 1) - b
        errs.append(np.max(np.abs(res)))
    assert 3.0 < errs[0] / errs[1] < 5.0


def test_term1_and_term2_bands():
    N = 64
    for term, m, lo, hi in ((1, 5, 5, 16), (2, 10, 20, 60)):
        b = P.heat_rhs(N, term)
        G = lambda u: P.heat_G(u, N, term, b)
        counts = {}
        for v in VARIANTS:
            r = aa_variant(G, np.zeros(N * N), m, v, 300, tol=1e-8, record_x=False, record_loo=False)
            counts[v] = r.iters if r.converged else None
            if r.converged:
                # converged to the discrete solution, which is O(h^2) from u_exact
                assert np.max(np.abs(r.x - P.heat_u_exact(N))) < 5e-3
        for v in ("mgs", "icwy", "cgs2"):
            assert counts[v] is not None and lo <= counts[v] <= hi, (term, counts)
        if term == 1:
            assert counts["dcgs2"] is not None and lo <= counts["dcgs2"] <= hi


def test_bratu_band_and_dcgs2_readings():
    """Bratu (§5.2, lambda = 6.7, m = 30, tol 1e-10): every variant converges in
    < 30 iterations -- DCGS-2 only with the consistent R update of reading A3
    (R += R_kk s); the verbatim Alg. 6 l.5 (R += s) diverges on this problem and on heat
    term 2, contradicting the paper's reported results (reading A3)."""
    N = 64
    b = P.heat_rhs(N, 3)
    G = lambda u: P.heat_G(u, N, 3, b)
    for v in ("mgs", "icwy", "cgs2"):
        r = aa_variant(G, np.zeros(N * N), 30, v, 100, tol=1e-10, record_x=False, record_loo=False)
        assert r.converged and r.iters < 30
    r = aa_variant(G, np.zeros(N * N), 30, "dcgs2", 100, tol=1e-10, dcgs2_rscale=True,
                   record_x=False, record_loo=False)
    assert r.converged and r.iters < 30
    with np.errstate(all="ignore"):
        r = aa_variant(G, np.zeros(N * N), 30, "dcgs2", 60, tol=1e-10, record_x=False, record_loo=False)
    assert not r.converged
