"""O1 (definition) and O2 (variant) Anderson-acceleration drivers — Alg. 1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .qr import (Ledger, QRState, Reducer, _breakdown_check, back_substitution, icwy_rebuild_T,
                 icwy_update_T_small, loss_of_orthogonality, lsp_solve, qradd, qrdelete_givens)


@dataclass
class AAResult:
    x: np.ndarray                      # last iterate returned (x_{i+1})
    iters: int                         # Alg. 1 loop index i at return (reading A10)
    converged: bool
    xs: list = field(default_factory=list)        # x_2, x_3, ... (x_{i+1} for i = 1..)
    f_norms: list = field(default_factory=list)   # ||f_i||_2, i = 1..
    dx_norms: list = field(default_factory=list)  # ||x_{i+1} - x_i||_2
    gammas: list = field(default_factory=list)
    lsq_res: list = field(default_factory=list)   # ||f_i - F_i gamma||_2 (O1 only)
    loo: list = field(default_factory=list)       # ||I - Q^T Q||_F after the update (O2)
    ledgers: list = field(default_factory=list)   # cumulative ledger snapshot after each iteration
    breakdown: list = field(default_factory=list)
    rratio: list = field(default_factory=list)    # R_kk / ||Delta f|| of the step's QRAdd (O2)
    x1: np.ndarray | None = None


def _householder_lsq(F: np.ndarray, f: np.ndarray) -> np.ndarray:
    """gamma = argmin ||f - F gamma||_2 by unpivoted Householder QR (LAPACK geqrf via
    numpy.linalg.qr) and back-substitution (reading A23)."""
    Qh, Rh = np.linalg.qr(F, mode="reduced")
    return back_substitution(Rh, Qh.T @ f)


def aa_definition(G, x0: np.ndarray, m: int, max_iters: int, tol: float = 0.0,
                  beta: float = 1.0, record_x: bool = True) -> AAResult:
    """O1: Alg. 1 with an exact least-squares solve each iteration.

    Optional damping (not in the paper; reading A13):
    x_{i+1} = G(x_i) - G_i gamma - (1 - beta) (f_i - F_i gamma)."""
    x0 = np.asarray(x0, dtype=np.float64)
    g = G(x0)                                   # l.1  x_1 = G(x_0), f_0 = G(x_0) - x_0
    f_prev, g_prev = g - x0, g
    x = np.array(g, copy=True)
    res = AAResult(x=x, iters=0, converged=False, x1=x.copy())
    dF: deque = deque()
    dG: deque = deque()
    for i in range(1, max_iters + 1):
        g = G(x)                                # l.3  f_i = G(x_i) - x_i
        f = g - x
        dF.append(f - f_prev)                   # l.4-5: Delta f_{i-1}, Delta g_{i-1}
        dG.append(g - g_prev)
        mi = min(m, i)
        while len(dF) > mi:
            dF.popleft()
            dG.popleft()
        F = np.stack(dF, axis=1)
        Gm = np.stack(dG, axis=1)
        gamma = _householder_lsq(F, f)          # l.6
        x_new = g - Gm @ gamma                  # l.7
        if beta != 1.0:
            x_new = x_new - (1.0 - beta) * (f - F @ gamma)
        dx = float(np.linalg.norm(x_new - x))   # l.8 (2-norm, absolute; reading A9)
        res.f_norms.append(float(np.linalg.norm(f)))
        res.dx_norms.append(dx)
        res.gammas.append(gamma)
        res.lsq_res.append(float(np.linalg.norm(f - F @ gamma)))
        if record_x:
            res.xs.append(x_new.copy())
        x = x_new
        f_prev, g_prev = f, g
        res.iters = i
        if dx < tol:
            res.converged = True
            break
    res.x = x
    return res


def aa_variant(G, x0: np.ndarray, m: int, variant: str, max_iters: int, tol: float = 0.0,
               beta: float = 1.0, shards: int = 1, dcgs2_cond: int = 3,
               dcgs2_rscale: bool = False, record_x: bool = True, record_loo: bool = True,
               dfs_override=None, icwy_delete: str = "rebuild", breakdown: str = "record",
               breakdown_eps: float | None = None) -> AAResult:
    """O2: Alg. 1 + Alg. 2 with the paper's incremental QR (variant in mgs/icwy/cgs2/dcgs2).

    ``icwy_delete``: "rebuild" = the paper's T update after QRDelete, one reduction
    (reading A6); "small" = the reduction-free variant icwy_update_T_small
    (not in the paper).
    Ledger phases: qradd (Algs. 2 l.2, 3-6), qrdelete (ICWY rebuild),
    lsp_rhs (Alg. 2 l.9), norm_check (Alg. 1 l.8).
    Damping (reading A13): x_{i+1} = g_i - G_i gamma - (1-beta)(f_i - Q (Q^T f_i)).

    ``breakdown`` (reading A12; the paper is silent on linear dependence): a QRAdd breaks
    down when its new R_kk <= eps_a ||Delta f|| (eps_a = 10 eps sqrt(n) unless
    ``breakdown_eps`` is given).  "record" only records it (res.breakdown) and carries on
    with the factorisation as computed (stress runs, config 5).  "restart" is SPEC's policy
     as SURVEY.md §8(b) assigns it to the library and its caller: the
    breaking step degrades to gamma = 0, i.e. x_{i+1} = G(x_i) (Alg. 1 l.1 restarted from
    x_i), the window is emptied, the next iteration takes Alg. 2's i = 1 branch with
    Delta f = f_{i+1} - f_i; a breakdown on that first step after a restart is a hard error
    (res.hard_error, the run stops)."""
    if breakdown not in ("record", "restart"):
        raise ValueError(f"unknown breakdown policy {breakdown!r}")
    x0 = np.asarray(x0, dtype=np.float64)
    n = x0.shape[0]
    red = Reducer(shards)
    led = Ledger()
    st = QRState(n, m)
    g = G(x0)                                   # Alg. 1 l.1
    f_prev, g_prev = g - x0, g
    x = np.array(g, copy=True)
    res = AAResult(x=x, iters=0, converged=False, x1=x.copy())
    st.eps_a = breakdown_eps
    res.hard_error = False
    dG: deque = deque()
    restarted = False                           # the previous step broke down (policy "restart")
    for i in range(1, max_iters + 1):
        g = G(x)                                # Alg. 1 l.3
        f = g - x
        df = f - f_prev                         # l.5  Delta f_{i-1}
        dg = g - g_prev                         # l.4  Delta g_{i-1}
        st.breakdown = False
        if st.mi == 0:                          # Alg. 2 l.1-2 (i = 1, or the first step after a restart)
            r00 = red.norm(df)
            led.sync("qradd")
            _breakdown_check(st, r00, r00)      # Delta f = 0: R_00 = 0 (A12)
            st.R[0, 0] = r00
            with np.errstate(invalid="ignore", divide="ignore"):
                st.Q[:, 0] = df / r00
            st.T[0, 0] = 1.0
            st.mi = 1
        else:
            if st.mi == m:                      # Alg. 2 l.4-5  QRDelete (i > m)
                rots = qrdelete_givens(st)
                dG.popleft()
                if variant == "icwy":
                    if icwy_delete == "small":
                        icwy_update_T_small(st, rots)
                    else:
                        icwy_rebuild_T(st, led, red)
            qradd(variant, st, df, led, red, dcgs2_cond, dcgs2_rscale)   # Alg. 2 l.7
        dG.append(dg)
        k = st.mi
        if breakdown == "restart" and st.breakdown:
            # the step degrades to gamma = 0: x_{i+1} = G(x_i); the dependent column is not kept
            led.sync("lsp_rhs")                 # Q^T f_i rode in the step's reductions all the same
            gamma = np.zeros(k)
            x_new = np.array(g, copy=True)
        else:
            gamma = lsp_solve(st, f, led, red)  # Alg. 2 l.9
            Gm = np.stack(dG, axis=1)
            x_new = g - Gm @ gamma              # Alg. 1 l.7
            if beta != 1.0:
                c = st.Q[:, :k].T @ f
                x_new = x_new - (1.0 - beta) * (f - st.Q[:, :k] @ c)
        dx = red.norm(x_new - x)                # Alg. 1 l.8
        led.sync("norm_check")
        res.f_norms.append(red.norm(f))
        res.dx_norms.append(dx)
        res.gammas.append(gamma)
        res.breakdown.append(st.breakdown)
        res.rratio.append(st.last_ratio)
        if record_loo:
            res.loo.append(loss_of_orthogonality(st.Q[:, :k]))
        res.ledgers.append(led.snapshot())
        if record_x:
            res.xs.append(x_new.copy())
        x = x_new
        f_prev, g_prev = f, g
        res.iters = i
        if breakdown == "restart" and st.breakdown:
            if restarted:                       # second consecutive breakdown
                res.hard_error = True
                break
            restarted = True
            st = QRState(n, m)                  # empty the window (aa_reset)
            st.eps_a = breakdown_eps
            dG.clear()
        else:
            restarted = False
        if dx < tol:
            res.converged = True
            break
    res.x = x
    res.state = st
    return res


def startup_syncs(variant: str, m: int) -> int:
    """Sync formulas printed at P:536-540 (start-up: filling the window)."""
    return {"mgs": (m * m + m) // 2, "icwy": 2 * m - 1, "cgs2": 3 * m - 2,
            "dcgs2": 2 * m - 1}[variant]


def recycle_syncs(variant: str, m: int, include_delete: bool = True) -> int:
    """Per recycle iteration."""
    base = {"mgs": m, "icwy": 2, "cgs2": 3, "dcgs2": 2}[variant]
    return base + (1 if (include_delete and variant == "icwy") else 0)


def fp_solve(G, x0, max_iters: int, tol: float):
    """Plain fixed-point (Picard) iteration x_{i+1} = G(x_i)."""
    x = np.asarray(x0, dtype=np.float64)
    for i in range(1, max_iters + 1):
        xn = G(x)
        if math.sqrt(float((xn - x) @ (xn - x))) < tol:
            return xn, i
        x = xn
    return x, max_iters
