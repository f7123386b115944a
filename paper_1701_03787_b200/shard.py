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

__all__ = ["kx_slab", "kx_rows_folded", "slab_of", "assemble_slabs"]


def kx_slab(n_y: int, rank: int, world: int) -> tuple:
    """[lo, hi) kx rows of `rank`: balanced contiguous split (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return (n_y * rank) // world, (n_y * (rank + 1)) // world


def kx_rows_folded(n_y: int, rank: int, world: int) -> np.ndarray:
    """kx rows of `rank` in a folded decomposition: each rank holds whole
    mirror pairs (m, n_y - m), which have identical z2, so the biharmonic
    stream solve can run one factor recurrence per pair on every rank
    (solvers.mirror_pairs; SURVEY.md 8(e) "folded slabs").  Pairs are split
    in balanced contiguous ranges of m; the two self-mirrored rows (0 and
    n_y/2) go to the first and last rank.  Rows are returned in ascending
    order (for one rank: the plain plane), which puts partners a varying
    distance apart: at config 4 that measured 22.5 ms for the biharmonic
    against 25.2 ms with partners adjacent and 23.7 ms with partners a
    constant half-slab apart (the two row streams of a warp then meet on the
    same DRAM channels)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    if n_y < 4 or n_y % 2:
        lo, hi = kx_slab(n_y, rank, world)
        return np.arange(lo, hi)
    pairs = np.arange(1, n_y // 2)  # m; partner n_y - m
    lo, hi = (len(pairs) * rank) // world, (len(pairs) * (rank + 1)) // world
    rows = [0] if rank == 0 else []
    rows += [int(m) for m in pairs[lo:hi]]
    rows += [int(n_y - m) for m in pairs[lo:hi]]
    if rank == world - 1:
        rows.append(n_y // 2)
    return np.sort(np.asarray(rows, dtype=np.int64))


def slab_of(a: np.ndarray, n_y: int, rank: int, world: int, axis: int = 1) -> np.ndarray:
    """The rank's slab of an array whose `axis` is the kx axis."""
    lo, hi = kx_slab(n_y, rank, world)
    idx = [slice(None)] * a.ndim
    idx[axis] = slice(lo, hi)
    return a[tuple(idx)]


def assemble_slabs(parts, axis: int = 1) -> np.ndarray:
    """Inverse of slab_of over ranks 0..world-1 (rank order)."""
    return np.concatenate(list(parts), axis=axis)
