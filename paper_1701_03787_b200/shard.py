"""Multi-GPU decomposition of the wavenumber plane.

Every (kx, kz) system is independent, so the plane of shape (n_y, n_z//2+1)
is split into contiguous kx slabs -- ranges of axis 1 of the reference's
(n_modes, n_y, n_z//2+1) spectral arrays -- one per rank.  For each mode row
a slab is one contiguous chunk of kx_rows * (n_z//2+1) values, so a rank's
RHS/solution is itself a (n_modes, slab) array the single-GPU solvers take
unchanged.  No collective is needed on the data path; the only
communication is the barrier and the max-over-ranks time reduction in
bench.py.
"""

from __future__ import annotations

import numpy as np

__all__ = ["kx_slab", "slab_of", "assemble_slabs"]


def kx_slab(n_y: int, rank: int, world: int) -> tuple:
    """[lo, hi) kx rows of `rank`: balanced contiguous split (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return (n_y * rank) // world, (n_y * (rank + 1)) // world


def slab_of(a: np.ndarray, n_y: int, rank: int, world: int, axis: int = 1) -> np.ndarray:
    """The rank's slab of an array whose `axis` is the kx axis."""
    lo, hi = kx_slab(n_y, rank, world)
    idx = [slice(None)] * a.ndim
    idx[axis] = slice(lo, hi)
    return a[tuple(idx)]


def assemble_slabs(parts, axis: int = 1) -> np.ndarray:
    """Inverse of slab_of over ranks 0..world-1 (rank order)."""
    return np.concatenate(list(parts), axis=axis)
