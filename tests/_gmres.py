"""Textbook GMRES (Saad & Schultz) used only as an independent pin for the oracle.

AA with an unbounded window applied to the linear map G(x) = M x + b is
equivalent to GMRES on (I - M) x = b (Walker & Ni 2011):
x_{i+1}^{AA} = G(x_i^{GMRES}).  Arnoldi with a second Gram-Schmidt pass, then the
small Hessenberg least-squares problem solved with numpy.linalg.lstsq.
Shares no code with oracle/.
"""
import numpy as np


def gmres_iterates(A, b, x0, kmax):
    """Return [x_0, x_1, ..., x_kmax] of full (unrestarted) GMRES."""
    n = b.shape[0]
    r0 = b - A @ x0
    beta = np.linalg.norm(r0)
    V = np.zeros((n, kmax + 1))
    H = np.zeros((kmax + 1, kmax))
    V[:, 0] = r0 / beta
    xs = [x0.copy()]
    for j in range(kmax):
        w = A @ V[:, j]
        for _ in range(2):                       # classical GS, twice
            h = V[:, :j + 1].T @ w
            w = w - V[:, :j + 1] @ h
            H[:j + 1, j] += h
        H[j + 1, j] = np.linalg.norm(w)
        if H[j + 1, j] > 0:
            V[:, j + 1] = w / H[j + 1, j]
        e1 = np.zeros(j + 2)
        e1[0] = beta
        y, *_ = np.linalg.lstsq(H[:j + 2, :j + 1], e1, rcond=None)
        xs.append(x0 + V[:, :j + 1] @ y)
    return xs
