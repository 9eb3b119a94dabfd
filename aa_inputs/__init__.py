"""Seeded synthetic inputs shared by the oracle tests and the GPU path.

This module holds NONE of the method's arithmetic (no QR, no least squares,
no AA update).  It only produces the numbers both sides consume:

* ``uniform`` — a counter-based SplitMix64 stream ("Input
  generator"): value_i = a + (b - a) * u_i with
  u_i = (splitmix64(seed + stream * 2**48 + i) >> 11) * 2**-53.
  The libaa test utility ``aa_fill_uniform`` (include/aa_testing.h) implements
  the same generator on the device with ``__dmul_rn``/``__dadd_rn`` so host and
  device values are bitwise identical (no FMA contraction on either side).
* ``problems`` — the fixed-point maps G the harness (the "caller") evaluates.

Seed 9667 is the default; streams: 1 = d, 2 = b, 3 = x0, 5 = config-5a Gaussian.
"""
from __future__ import annotations

import numpy as np

SEED = 9667
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser applied elementwise to uint64 counters (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64, copy=True) + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(n: int, lo: float, hi: float, *, stream: int, seed: int = SEED,
            offset: int = 0) -> np.ndarray:
    """Entries ``offset .. offset+n-1`` of the counter-based uniform stream on [lo, hi)."""
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = np.uint64(seed) + np.uint64(stream) * np.uint64(1 << 48) + idx
    z = splitmix64(ctr)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    # separate multiply then add (no FMA), exactly as the device side does
    scaled = np.multiply(np.float64(hi - lo), u)
    return np.add(np.float64(lo), scaled)


def shard_bounds(n: int, p: int) -> list[tuple[int, int]]:
    """Contiguous row partition of n rows over p ranks, remainder to the leading ranks
    (§4 "each process ... contains n/p contiguous rows"; SPEC.md ShardLayout)."""
    base, rem = divmod(n, p)
    out, off = [], 0
    for r in range(p):
        ln = base + (1 if r < rem else 0)
        out.append((off, ln))
        off += ln
    return out


from . import problems  # noqa: E402,F401
