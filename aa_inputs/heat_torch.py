"""The heat workload's map G on the device (torch; the caller's side of Alg. 1, not the
AA path): u -> A^{-1}(b - c(u)) with A^{-1} applied exactly by 2-D DST-I through FFTs of
the odd extension, optionally slab-distributed over ranks (rows split, two all-to-all
transposes per application).  Mirrors aa_inputs.problems.laplacian_solve (scipy)."""
from __future__ import annotations

import math

import torch


def dst1_lastdim(x: torch.Tensor) -> torch.Tensor:
    """Orthonormal DST-I along the last axis: y_k = sqrt(2/(N+1)) sum_j x_j sin(pi j k/(N+1))."""
    N = x.shape[-1]
    z = torch.zeros(*x.shape[:-1], 2 * N + 2, dtype=x.dtype, device=x.device)
    z[..., 1:N + 1] = x
    z[..., N + 2:] = -torch.flip(x, dims=[-1])
    Z = torch.fft.rfft(z, dim=-1)
    return -Z.imag[..., 1:N + 1] * (0.5 * math.sqrt(2.0 / (N + 1)))


def laplacian_eigs(N: int, device, dtype=torch.float64) -> torch.Tensor:
    h = 1.0 / (N + 1)
    s = torch.sin(torch.arange(1, N + 1, device=device, dtype=dtype) * (math.pi * h / 2)) ** 2
    return -(4.0 / h ** 2) * (s[:, None] + s[None, :])


BRATU_LAMBDA = 6.7


def heat_c(u: torch.Tensor, term: int) -> torch.Tensor:
    if term == 1:
        e = torch.exp(u)
        return u + u * e + u / e + (u - e) ** 2
    if term == 3:   # Bratu (§5.2): A u + lambda e^u = 0
        return BRATU_LAMBDA * torch.exp(u)
    return 100.0 * (u - u * u)


class HeatG:
    """G(u) = A^{-1}(b - c(u)) for this rank's row slab of the N x N grid."""

    def __init__(self, N: int, term: int, b_local: torch.Tensor, rank: int = 0, world: int = 1, dist=None):
        assert N % world == 0
        self.N, self.term, self.rank, self.world, self.dist = N, term, rank, world, dist
        self.Nl = N // world
        self.b = b_local.view(self.Nl, N)
        lam = laplacian_eigs(N, b_local.device)
        # transposed slab layout holds columns [rank*Nl, (rank+1)*Nl) of the mode grid
        self.lam_t = lam[:, rank * self.Nl:(rank + 1) * self.Nl].contiguous() if world > 1 else lam

    def _to_cols(self, A):   # (Nl, N) row slab -> (N, Nl) column slab
        p, Nl = self.world, self.Nl
        send = A.reshape(Nl, p, Nl).permute(1, 0, 2).contiguous()
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send)
        return recv.reshape(p * Nl, Nl)

    def _to_rows(self, B):   # (N, Nl) column slab -> (Nl, N) row slab
        p, Nl = self.world, self.Nl
        send = B.reshape(p, Nl, Nl).contiguous()
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send)
        return recv.permute(1, 0, 2).reshape(Nl, p * Nl)

    def __call__(self, u: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        r = self.b - heat_c(u.view(self.Nl, self.N), self.term)
        y = dst1_lastdim(r)                              # along x (contiguous)
        if self.world == 1:
            y = dst1_lastdim(y.t().contiguous())         # along y
            y = dst1_lastdim(y / self.lam_t.t())
            y = dst1_lastdim(y.t().contiguous())
        else:
            B = self._to_cols(y)                          # (N, Nl): y index first
            B = dst1_lastdim(B.t().contiguous())          # (Nl, N): along y
            B = dst1_lastdim(B / self.lam_t.t())          # divide in mode space, back along y
            y = dst1_lastdim(self._to_rows(B.t().contiguous()))
        if out is None:
            return y.reshape(-1)
        out.copy_(y.reshape(-1))
        return out
