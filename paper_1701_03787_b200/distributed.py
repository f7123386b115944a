"""Slab-decomposed 3-D Shen transforms over several GPUs.

The solves need no communication (kx slabs, ``shard.py``).  A 3-D transform
does: the periodic FFTs want whole (y, z) planes, the wall-normal stage wants
whole x columns.  The paper's slab decomposition (one all-to-all per
transform) is used:

forward   physical x-planes [p0, p1) of rank r  --rfft2 over (y, z)-->
          (planes_r, n_y, n_z/2+1)  --all-to-all-->  (N, kx rows_r, n_z/2+1)
          --wall-normal stage (transforms.wall_forward)-->
          (n_modes, kx rows_r, n_z/2+1): exactly the rank's solver slab.
inverse   the mirror image.

The kx rows of rank r are ``shard.kx_rows_folded(n_y, r, world)`` -- the
same folded row set bench.py and the multi-GPU solves use (whole (m, -m)
mirror pairs per rank, ascending), so the exchange hands the solver the rows
its LU objects were built on and the mirror-pair kernels apply on every rank.
A caller-supplied ``rows_of(n_y, rank, world)`` selects another split
(``shard.kx_slab`` rows for contiguous slabs).

With NCCL the exchange is ``all_to_all_single`` over NVLink on device
tensors; the same code runs on CPU tensors under ``gloo`` (exchange tests).
Plane split: balanced contiguous (sizes differ by at most one).
"""

from __future__ import annotations

from .shard import kx_rows_folded
from .transforms import plane_irfft2, plane_rfft2

__all__ = ["plane_slab", "kx_rows", "planes_to_kx", "kx_to_planes", "forward_transform_slab", "inverse_transform_slab"]


def plane_slab(n_planes: int, rank: int, world: int) -> tuple:
    """[lo, hi) physical x-planes of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return (n_planes * rank) // world, (n_planes * (rank + 1)) // world


def _world(group):
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _all_to_all(recv, send, recv_sizes, send_sizes, group):
    """all_to_all_single; with a gloo group, device tensors go through host
    buffers (gloo has no CUDA all-to-all) -- the multi-rank path then also
    runs with several ranks on one GPU (tests) or on CPU-only hosts."""
    import torch.distributed as dist

    if send.is_cuda and dist.get_backend(group) == "gloo":
        r = recv.cpu()
        dist.all_to_all_single(r, send.cpu(), recv_sizes, send_sizes, group=group)
        recv.copy_(r)
    else:
        dist.all_to_all_single(recv, send, recv_sizes, send_sizes, group=group)


def kx_rows(n_y: int, rank: int, world: int, rows_of=None):
    """The kx rows (ascending int64 array) rank `rank` holds after the exchange."""
    import numpy as np

    f = rows_of or kx_rows_folded
    return np.asarray(f(n_y, rank, world), dtype=np.int64)


def planes_to_kx(x, n_planes: int, group=None, rows_of=None):
    """(planes_r, n_y, K) on rank r -> (n_planes, len(rows_r), K): all-to-all
    of the rank's planes to the kx rows of every rank (folded by default)."""
    import torch
    import torch.distributed as dist

    rank, world = _world(group)
    p, n_y, K = x.shape
    if world == 1:
        return x.contiguous()
    lo_p, hi_p = plane_slab(n_planes, rank, world)
    if hi_p - lo_p != p:
        raise ValueError(f"rank {rank} holds {p} planes, expected {hi_p - lo_p}")
    blocks = []
    send_sizes = []
    for q in range(world):
        idx = torch.from_numpy(kx_rows(n_y, q, world, rows_of)).to(x.device)
        blocks.append(x.index_select(1, idx).reshape(-1))
        send_sizes.append(p * int(idx.numel()) * K)
    send = torch.cat(blocks)
    m = len(kx_rows(n_y, rank, world, rows_of))
    recv_sizes = [(plane_slab(n_planes, q, world)[1] - plane_slab(n_planes, q, world)[0]) * m * K
                  for q in range(world)]
    recv = torch.empty(sum(recv_sizes), dtype=x.dtype, device=x.device)
    _all_to_all(recv, send, recv_sizes, send_sizes, group)
    # blocks arrive in rank order = plane order: already (n_planes, rows_r, K)
    return recv.view(n_planes, m, K)


def kx_to_planes(y, n_y: int, group=None, rows_of=None):
    """(n_planes, len(rows_r), K) -> (planes_r, n_y, K): inverse of planes_to_kx."""
    import torch
    import torch.distributed as dist

    rank, world = _world(group)
    n_planes, m, K = y.shape
    if world == 1:
        return y.contiguous()
    y = y.contiguous()
    send_sizes = []
    for q in range(world):
        lo, hi = plane_slab(n_planes, q, world)
        send_sizes.append((hi - lo) * m * K)  # axis-0 ranges are contiguous chunks
    lo_p, hi_p = plane_slab(n_planes, rank, world)
    p = hi_p - lo_p
    rows = [kx_rows(n_y, q, world, rows_of) for q in range(world)]
    recv_sizes = [p * len(r) * K for r in rows]
    recv = torch.empty(sum(recv_sizes), dtype=y.dtype, device=y.device)
    _all_to_all(recv, y.view(-1), recv_sizes, send_sizes, group)
    out = torch.empty((p, n_y, K), dtype=y.dtype, device=y.device)
    for part, r in zip(torch.split(recv, recv_sizes), rows):
        out.index_copy_(1, torch.from_numpy(r).to(y.device), part.view(p, len(r), K))
    return out


def forward_transform_slab(u_planes, mesh, space, group=None, solve_mass: bool = True, rows_of=None):
    """Rank's physical planes (planes_r, n_y, n_z) (torch CUDA, float64) ->
    rank's kx rows of the coefficients (n_modes, rows_r, n_z/2+1), complex128.
    ``solve_mass=False`` stops at the scalar products (forward_scalar_product)."""
    import torch

    from .mesh import family_code, space_code
    from .transforms import wall_forward

    N = mesh.n_x + 1
    fourier = plane_rfft2(u_planes.to(torch.float64))
    cols = planes_to_kx(fourier, N, group, rows_of)
    m, K = cols.shape[1], cols.shape[2]
    out = wall_forward(cols.reshape(N, m * K), mesh.n_x, family_code(mesh.family), space_code(space), solve_mass)
    return out.reshape(out.shape[0], m, K)


def inverse_transform_slab(c_slab, mesh, space, group=None, rows_of=None):
    """Rank's kx rows of coefficients (n_modes, rows_r, n_z/2+1) -> the rank's
    physical planes (planes_r, n_y, n_z), float64."""
    import torch

    from .mesh import family_code, space_code
    from .transforms import wall_inverse

    n, m, K = c_slab.shape
    lines, norm = wall_inverse(c_slab.to(torch.complex128).reshape(n, m * K).contiguous(), mesh.n_x,
                               family_code(mesh.family), space_code(space), mesh.n_y * mesh.n_z)
    planes = kx_to_planes(lines.reshape(mesh.n_x + 1, m, K), mesh.n_y, group, rows_of)
    return plane_irfft2(planes, mesh.n_y, mesh.n_z, norm)
