"""O2 building blocks: the paper's incremental QR update kernels, written out.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy, fp64, no
blocking/fusion/reordering beyond what each algorithm states.  Indexing follows
the paper's 0-based inclusive convention: with ``k`` existing
columns the new column has index ``k = m_i - 1`` and the existing ones are
``0 .. m_i - 2``.
"""
from __future__ import annotations

import math

import numpy as np

EPS = float(np.finfo(np.float64).eps)
VARIANTS = ("mgs", "icwy", "cgs2", "dcgs2")


class Ledger:
    """Counts global reductions by phase.

    One fused multi-dot of any width, or a delayed reduction merged with a later
    one, counts exactly once."""

    PHASES = ("qradd", "qrdelete", "lsp_rhs", "norm_check", "other")

    def __init__(self):
        self.counts = dict.fromkeys(self.PHASES, 0)

    def sync(self, phase: str) -> None:
        self.counts[phase] += 1

    def snapshot(self) -> dict:
        return dict(self.counts)


class Reducer:
    """Global reductions over ``p`` simulated contiguous row shards:
    per-shard partial sums, then a fixed-order (ascending rank) sum.  p = 1 is a
    plain numpy dot."""

    def __init__(self, p: int = 1):
        self.p = p

    def _bounds(self, n):
        base, rem = divmod(n, self.p)
        off = 0
        for r in range(self.p):
            ln = base + (1 if r < rem else 0)
            yield off, off + ln
            off += ln

    def dot(self, a: np.ndarray, b: np.ndarray) -> float:
        if self.p == 1:
            return float(a @ b)
        tot = 0.0
        for lo, hi in self._bounds(a.shape[0]):
            tot += float(a[lo:hi] @ b[lo:hi])
        return tot

    def matT_vec(self, A: np.ndarray, v: np.ndarray) -> np.ndarray:
        """A^T v as one fused multi-dot ("fused dot product")."""
        if A.shape[1] == 0:
            return np.zeros(0)
        if self.p == 1:
            return A.T @ v
        tot = np.zeros(A.shape[1])
        for lo, hi in self._bounds(A.shape[0]):
            tot = tot + A[lo:hi].T @ v[lo:hi]
        return tot

    def matT_mat(self, A: np.ndarray, B: np.ndarray) -> np.ndarray:
        """A^T B (several right-hand sides) as ONE fused reduction: the merged
        "Delayed Sync" + "Sync" of Alg. 4 l.1-2 and Alg. 6 l.1/l.3."""
        if self.p == 1:
            return A.T @ B
        tot = np.zeros((A.shape[1], B.shape[1]))
        for lo, hi in self._bounds(A.shape[0]):
            tot = tot + A[lo:hi].T @ B[lo:hi]
        return tot

    def gram(self, A: np.ndarray) -> np.ndarray:
        if self.p == 1:
            return A.T @ A
        tot = np.zeros((A.shape[1], A.shape[1]))
        for lo, hi in self._bounds(A.shape[0]):
            tot = tot + A[lo:hi].T @ A[lo:hi]
        return tot

    def norm(self, v: np.ndarray) -> float:
        return math.sqrt(self.dot(v, v))


class QRState:
    """The AA iteration space: Q (n x m, column-oriented), R (m x m upper
    triangular), T (m x m unit lower, ICWY only, stored as I + L per reading A5),
    and the active column count m_i."""

    def __init__(self, n: int, m: int):
        self.n, self.m = n, m
        self.Q = np.zeros((n, m), order="F")
        self.R = np.zeros((m, m))
        self.T = np.zeros((m, m))
        self.mi = 0
        self.breakdown = False
        self.eps_a = None        # breakdown threshold; None = 10 eps sqrt(n) (reading A12)


# --------------------------------------------------------------------------------------
# small dense helpers (written as plain loops)
# --------------------------------------------------------------------------------------

def forward_substitution_unit_lower(T: np.ndarray, s: np.ndarray) -> np.ndarray:
    """Solve T r = s with T unit lower triangular (Alg. 4 l.4, "T^{-1} R"; reading A5)."""
    k = s.shape[0]
    r = np.array(s, dtype=np.float64, copy=True)
    for j in range(k):
        for l in range(j):
            r[j] -= T[j, l] * r[l]
    return r


def back_substitution(R: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Solve R gamma = c with R upper triangular (Alg. 2 l.9)."""
    k = c.shape[0]
    g = np.zeros(k)
    for j in range(k - 1, -1, -1):
        acc = c[j]
        for l in range(j + 1, k):
            acc -= R[j, l] * g[l]
        g[j] = acc / R[j, j]
    return g


def loss_of_orthogonality(Q: np.ndarray) -> float:
    """||I - Q^T Q||_F over the active columns (P:156 metric)."""
    k = Q.shape[1]
    return float(np.linalg.norm(np.eye(k) - Q.T @ Q, "fro"))


def breakdown_eps_default(n: int) -> float:
    """eps_a = 10 eps sqrt(n), n the GLOBAL vector length (reading A12)."""
    return 10.0 * EPS * math.sqrt(n)


def _breakdown_check(st: QRState, rkk: float, vnorm0: float) -> None:
    """Reading A12 (paper silent): breakdown if R_kk <= eps_a ||v_orig||,
    v_orig the column before projection.  NaN counts as a breakdown (not R_kk > threshold).
    Recorded here; the driver's policy acts on it (oracle.aa_variant ``breakdown``)."""
    eps_a = st.eps_a if st.eps_a is not None else breakdown_eps_default(st.n)
    st.last_ratio = rkk / vnorm0 if vnorm0 > 0.0 else 0.0
    if not (rkk > eps_a * vnorm0):
        st.breakdown = True


# --------------------------------------------------------------------------------------
# QRAdd variants (Algs. 3-6).  ``v`` is Delta f_{i-1}; k = st.mi existing columns.
# --------------------------------------------------------------------------------------

def _normalise_new_column(st, v, k, led, red, vnorm0):
    # "R_{m_i-1,m_i-1} <- ||Delta f||_2  (Sync);  Q_{:,m_i-1} <- Delta f / R_{m_i-1,m_i-1}"
    rkk = red.norm(v)
    led.sync("qradd")
    _breakdown_check(st, rkk, vnorm0)
    st.R[k, k] = rkk
    with np.errstate(invalid="ignore", divide="ignore"):
        st.Q[:, k] = v / rkk
    st.mi = k + 1


def qradd_mgs(st: QRState, v: np.ndarray, led: Ledger, red: Reducer, vnorm0: float) -> None:
    """Alg. 3 QRAdd_MGS: m_i - 1 dependent dot/axpy pairs, then the norm."""
    k = st.mi
    v = np.array(v, copy=True)
    for j in range(k):                                   # l.1 for j = 0 .. m_i-2
        st.R[j, k] = red.dot(st.Q[:, j], v)              # l.2 (Sync)
        led.sync("qradd")
        v = v - st.R[j, k] * st.Q[:, j]                  # l.3
    _normalise_new_column(st, v, k, led, red, vnorm0)    # l.5-6


def qradd_icwy(st: QRState, v: np.ndarray, led: Ledger, red: Reducer, vnorm0: float) -> None:
    """Alg. 4 QRAdd_ICWY: l.1 (Delayed Sync) and l.2 (Sync) are one reduction."""
    k = st.mi
    v = np.array(v, copy=True)
    if k >= 1:
        Qk = st.Q[:, :k]
        # l.1: T_{m_i-2, 0:m_i-2} <- Q_{:,0:m_i-2}^T Q_{:,m_i-2}      (Delayed Sync)
        # l.2: R_{0:m_i-2, m_i-1} <- Q_{:,0:m_i-2}^T Delta f          (Sync)
        # merged into one reduction: Q^T [q_{m_i-2}, Delta f]
        both = red.matT_mat(Qk, np.stack([st.Q[:, k - 1], v], axis=1))
        row, rcol = both[:, 0], both[:, 1]
        led.sync("qradd")
        st.T[k - 1, :k] = row
        st.T[k - 1, k - 1] = 1.0                          # l.3
        rcol = forward_substitution_unit_lower(st.T[:k, :k], rcol)   # l.4
        v = v - Qk @ rcol                                 # l.5
        st.R[:k, k] = rcol
    else:
        st.T[0, 0] = 1.0
    _normalise_new_column(st, v, k, led, red, vnorm0)     # l.6-7


def qradd_cgs2(st: QRState, v: np.ndarray, led: Ledger, red: Reducer, vnorm0: float) -> None:
    """Alg. 5 QRAdd_CGS2: three reductions."""
    k = st.mi
    v = np.array(v, copy=True)
    if k >= 1:
        Qk = st.Q[:, :k]
        s = red.matT_vec(Qk, v)                           # l.1 (Sync)
        led.sync("qradd")
        y = v - Qk @ s                                    # l.2
        z = red.matT_vec(Qk, y)                           # l.3 (Sync)
        led.sync("qradd")
        v = y - Qk @ z                                    # l.4
        st.R[:k, k] = s + z                               # l.5
    _normalise_new_column(st, v, k, led, red, vnorm0)     # l.6-7


def qradd_dcgs2(st: QRState, v: np.ndarray, led: Ledger, red: Reducer, vnorm0: float,
                cond: int = 3, rscale: bool = False) -> None:
    """Alg. 6 QRAdd_DCGS2, verbatim per readings A1-A4.

    ``cond``: reorthogonalise when m_i > cond (paper: 3; option 2, reading A2).
    ``rscale``: R_{0:m_i-3,m_i-2} += R_{m_i-2,m_i-2} s instead of += s (reading A3)."""
    k = st.mi
    v = np.array(v, copy=True)
    mi_new = k + 1
    if k >= 1:
        Qk = st.Q[:, :k]
        reortho = mi_new > cond and k >= 2                # l.2 "if m_i > 3"
        # l.1 (Delayed Sync) and l.3 (Sync) in ONE reduction:
        # Q_{0:m_i-2}^T [Delta f, q_{m_i-2}]; s is the first m_i-2 entries of column 2
        if reortho:
            both = red.matT_mat(Qk, np.stack([v, st.Q[:, k - 1]], axis=1))
            rcol = both[:, 0]
        else:
            rcol = red.matT_vec(Qk, v)                    # l.1 alone
        if reortho:
            s = both[:k - 1, 1]                           # l.3: Q_{:,0:m_i-3}^T Q_{:,m_i-2}
            # l.4 read as Q_{:,m_i-2} <- Q_{:,m_i-2} - Q_{:,0:m_i-3} s  (reading A1)
            st.Q[:, k - 1] = st.Q[:, k - 1] - st.Q[:, :k - 1] @ s
            if rscale:
                st.R[:k - 1, k - 1] += st.R[k - 1, k - 1] * s
            else:
                st.R[:k - 1, k - 1] += s                  # l.5 verbatim (reading A3)
        led.sync("qradd")                                 # the single merged reduction of l.1/l.3
        st.R[:k, k] = rcol                                # pre-reortho coefficients (reading A4)
        v = v - st.Q[:, :k] @ rcol                        # l.7 with the updated Q_{:,m_i-2}
    _normalise_new_column(st, v, k, led, red, vnorm0)     # l.8-9


def qradd(variant: str, st: QRState, v: np.ndarray, led: Ledger, red: Reducer,
          dcgs2_cond: int = 3, dcgs2_rscale: bool = False) -> None:
    vnorm0 = red.norm(v)   # breakdown reference; rides in the first reduction (not counted)
    if variant == "mgs":
        qradd_mgs(st, v, led, red, vnorm0)
    elif variant == "icwy":
        qradd_icwy(st, v, led, red, vnorm0)
    elif variant == "cgs2":
        qradd_cgs2(st, v, led, red, vnorm0)
    elif variant == "dcgs2":
        qradd_dcgs2(st, v, led, red, vnorm0, dcgs2_cond, dcgs2_rscale)
    else:
        raise ValueError(f"unknown QRAdd variant {variant!r}")


# --------------------------------------------------------------------------------------
# QRDelete (reading A7) and the ICWY T rebuild (A6)
# --------------------------------------------------------------------------------------

def qrdelete_givens(st: QRState) -> list:
    """Remove the oldest column of F = QR: drop R's first column (upper Hessenberg),
    re-triangularise with m_i - 1 Givens rotations of adjacent rows, apply the same
    rotations to Q's columns, drop Q's last column.  No communication.
    Returns the rotations [(c_j, s_j)] in the order applied."""
    mi = st.mi
    if mi == 0:
        raise ValueError("qrdelete on an empty factorisation")
    H = np.array(st.R[:mi, 1:mi], copy=True)           # mi x (mi-1) upper Hessenberg
    Q = np.array(st.Q[:, :mi], copy=True)
    rots = []
    for j in range(mi - 1):
        a, b = H[j, j], H[j + 1, j]
        rho = math.hypot(a, b)
        if rho > 0.0:
            c, s = a / rho, b / rho
        else:
            c, s = 1.0, 0.0
        hj, hj1 = H[j, j:].copy(), H[j + 1, j:].copy()
        H[j, j:] = c * hj + s * hj1
        H[j + 1, j:] = -s * hj + c * hj1
        H[j, j] = rho                                   # diagonal kept >= 0
        H[j + 1, j] = 0.0
        rots.append((c, s))
        qj, qj1 = Q[:, j].copy(), Q[:, j + 1].copy()
        Q[:, j] = c * qj + s * qj1
        Q[:, j + 1] = -s * qj + c * qj1
    st.R[:, :] = 0.0
    st.R[:mi - 1, :mi - 1] = H[:mi - 1, :]
    st.Q[:, :mi - 1] = Q[:, :mi - 1]
    st.Q[:, mi - 1:] = 0.0
    st.mi = mi - 1
    return rots


def icwy_rebuild_T(st: QRState, led: Ledger, red: Reducer) -> None:
    """After a delete, T <- I + strict_lower(Q^T Q) over the retained columns in ONE
    reduction ("updated by introducing a single reduction"; reading A6)."""
    k = st.mi
    G = red.gram(st.Q[:, :k])
    led.sync("qrdelete")
    st.T[:, :] = 0.0
    st.T[:k, :k] = np.eye(k) + np.tril(G, -1)


def icwy_update_T_small(st: QRState, rots: list) -> None:
    """VARIANT, not in the paper (reading A6b): after a
    delete, update T without a reduction.  The delete replaced Q by Q' = Q W, W the first
    m_i - 1 columns of the product of the rotations (applied to the identity exactly as
    qrdelete_givens applies them to Q's columns), so Q'^T Q' = W^T (Q^T Q) W, and Q^T Q is
    taken as S = T + T^T - I (unit diagonal) from the known rows of the pre-delete T.

    Called after qrdelete_givens (st.mi = k retained columns).  Rows 0..k-2 of the new T
    are set; row k-1 is left as the identity row because QRAdd (Alg. 4 l.1) recomputes it
    before any use, and it would need the unknown T row of the newest pre-delete column."""
    k = st.mi
    mi = k + 1
    W = np.eye(mi)
    for j, (c, s) in enumerate(rots):
        wj, wj1 = W[:, j].copy(), W[:, j + 1].copy()
        W[:, j] = c * wj + s * wj1
        W[:, j + 1] = -s * wj + c * wj1
    Tk = st.T[:k, :k]                                    # known rows 0..k-1 (pre-delete)
    S = Tk + Tk.T - np.eye(k)
    Wp = W[:k, :k - 1]                                   # rows 0..k-1 suffice (column l uses rows <= l+1)
    Sp = Wp.T @ S @ Wp
    T = np.eye(k)
    T[:k - 1, :k - 1] += np.tril(Sp, -1)
    st.T[:, :] = 0.0
    st.T[:k, :k] = T


# --------------------------------------------------------------------------------------
# LSP solve (Alg. 2)
# --------------------------------------------------------------------------------------

def lsp_solve(st: QRState, f: np.ndarray, led: Ledger, red: Reducer) -> np.ndarray:
    """Alg. 2 l.9: solve R gamma = Q^T f_i (one fused reduction, phase lsp_rhs)."""
    k = st.mi
    c = red.matT_vec(st.Q[:, :k], f)
    led.sync("lsp_rhs")
    return back_substitution(st.R[:k, :k], c)
