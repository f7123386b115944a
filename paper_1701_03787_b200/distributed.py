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

``PeerExchange`` fuses the exchange into the plane FFT kernels instead (256 x
256 planes, up to 8 ranks of one box): every rank's kx-row buffer is opened
on every other rank through CUDA IPC, the forward rfft2 kernel stores each
spectrum row straight into its owner's buffer over NVLink and the inverse
irfft2 kernel loads each row from its owner's buffer.  No pack pass, no
all-to-all: one HBM round trip and one collective less per transform.  Ranks
order their accesses with a stream synchronise and a barrier on either side.
"""

from __future__ import annotations

from .shard import kx_rows_folded
from .transforms import plane_irfft2, plane_rfft2

__all__ = ["plane_slab", "kx_rows", "planes_to_kx", "kx_to_planes", "forward_transform_slab", "inverse_transform_slab",
           "PeerExchange"]


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


class PeerExchange:
    """The kx-row exchange of the slab transforms through peer memory.

    Collective constructor (every rank of ``group``): allocates this rank's
    (n_planes, rows_r, n_z/2+1) complex128 buffer ``cols`` -- the all-to-all's
    result layout -- and opens every peer's buffer here through CUDA IPC.
    ``scatter_rfft2`` / ``gather_irfft2`` are the fused forward / inverse
    plane transforms (``csrc/shen_plane_fft.cu``, ``rfft2_256_kernel<true>``,
    ``irfft2_256_kernel<true>``).  Only the plane sizes the cluster kernel
    supports (``shen_plane_fft_supported``), at most 8 ranks."""

    def __init__(self, n_planes: int, n_y: int, n_z: int, group=None, rows_of=None):
        import ctypes

        import numpy as np
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        from . import _lib
        from ._device import device

        self.group = group
        self.rank, self.world = _world(group)
        if self.world > 8:
            raise ValueError("PeerExchange: at most 8 ranks")
        if not _lib.lib().shen_plane_fft_supported(n_y, n_z):
            raise ValueError(f"PeerExchange: {n_y} x {n_z} planes are not supported by the plane FFT kernel")
        self.n_planes, self.n_y, self.n_z, self.K = n_planes, n_y, n_z, n_z // 2 + 1
        self.plane_lo, self.plane_hi = plane_slab(n_planes, self.rank, self.world)
        rows = [kx_rows(n_y, q, self.world, rows_of) for q in range(self.world)]
        owner = np.full(n_y, -1, dtype=np.int32)
        local = np.zeros(n_y, dtype=np.int32)
        for q, r in enumerate(rows):
            owner[r] = q
            local[r] = np.arange(len(r), dtype=np.int32)
        if (owner < 0).any():
            raise ValueError("PeerExchange: the row sets do not cover every kx row")
        self.rows = rows[self.rank]
        self.cols = torch.empty((n_planes, len(self.rows), self.K), dtype=torch.complex128, device=device())
        self._peers = [self.cols]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, reduce_tensor(self.cols), group=group)
            self._peers = []
            for q, (fn, args) in enumerate(handles):
                t = self.cols if q == self.rank else fn(*args)
                if t.device != self.cols.device:
                    _lib.check(_lib.lib().shen_enable_peer_access(t.device.index), "shen_enable_peer_access")
                self._peers.append(t)  # keeps the IPC mapping alive
        self._bases = (ctypes.c_void_p * self.world)(*[t.data_ptr() for t in self._peers])
        self._nrows = (ctypes.c_int64 * self.world)(*[len(r) for r in rows])
        self._owner = (ctypes.c_int * n_y)(*owner.tolist())
        self._local = (ctypes.c_int * n_y)(*local.tolist())

    def _fence(self):
        """This rank's kernels have finished and every rank has got here."""
        import torch
        import torch.distributed as dist

        torch.cuda.current_stream().synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)

    def scatter_rfft2(self, u_planes):
        """rfft2 of the rank's planes (planes_r, n_y, n_z), float64, with every
        spectrum row stored into its owner's ``cols``; returns this rank's
        ``cols`` (n_planes, rows_r, K) once every rank's rows have landed."""
        import torch

        from . import _lib
        from ._device import stream_handle

        u = u_planes.to(torch.float64).contiguous()
        if tuple(u.shape) != (self.plane_hi - self.plane_lo, self.n_y, self.n_z):
            raise ValueError(f"rank {self.rank} expects planes of shape "
                             f"{(self.plane_hi - self.plane_lo, self.n_y, self.n_z)}, got {tuple(u.shape)}")
        self._fence()  # nobody still reads the buffers' previous contents
        _lib.check(_lib.lib().shen_plane_rfft2_scatter(u.shape[0], self.n_y, self.n_z, u.data_ptr(), self.world,
                                                       self._bases, self._nrows, self._owner, self._local,
                                                       self.plane_lo, self.n_planes, stream_handle()),
                   "shen_plane_rfft2_scatter")
        self._fence()
        return self.cols

    def gather_irfft2(self, norm: str = "backward"):
        """irfft2 of the rank's planes with every spectrum row read from its
        owner's ``cols`` (which each rank has filled: ``wall_inverse(...,
        out=cols)``); returns (planes_r, n_y, n_z) float64."""
        import ctypes

        import numpy as np
        import torch

        from . import _lib
        from ._device import stream_handle

        p = self.plane_hi - self.plane_lo
        out = torch.empty((p, self.n_y, self.n_z), dtype=torch.float64, device=self.cols.device)
        scale = {"backward": 1.0 / (self.n_y * self.n_z), "forward": 1.0,
                 "ortho": 1.0 / np.sqrt(self.n_y * self.n_z)}[norm]
        self._fence()  # every rank's cols is complete
        _lib.check(_lib.lib().shen_plane_irfft2_gather(p, self.n_y, self.n_z, self.world, self._bases, self._nrows,
                                                       self._owner, self._local, self.plane_lo, self.n_planes,
                                                       out.data_ptr(), ctypes.c_double(scale), stream_handle()),
                   "shen_plane_irfft2_gather")
        self._fence()  # peers may rewrite their buffers only after everyone has read
        return out


def forward_transform_slab(u_planes, mesh, space, group=None, solve_mass: bool = True, rows_of=None, exchange=None):
    """Rank's physical planes (planes_r, n_y, n_z) (torch CUDA, float64) ->
    rank's kx rows of the coefficients (n_modes, rows_r, n_z/2+1), complex128.
    ``solve_mass=False`` stops at the scalar products (forward_scalar_product).
    ``exchange``: a ``PeerExchange`` for this mesh -- the exchange then runs
    inside the plane FFT kernel instead of as an all-to-all."""
    import torch

    from .mesh import family_code, space_code
    from .transforms import wall_forward

    N = mesh.n_x + 1
    if exchange is not None:
        cols = exchange.scatter_rfft2(u_planes)
    else:
        fourier = plane_rfft2(u_planes.to(torch.float64))
        cols = planes_to_kx(fourier, N, group, rows_of)
    m, K = cols.shape[1], cols.shape[2]
    out = wall_forward(cols.reshape(N, m * K), mesh.n_x, family_code(mesh.family), space_code(space), solve_mass)
    return out.reshape(out.shape[0], m, K)


def inverse_transform_slab(c_slab, mesh, space, group=None, rows_of=None, exchange=None):
    """Rank's kx rows of coefficients (n_modes, rows_r, n_z/2+1) -> the rank's
    physical planes (planes_r, n_y, n_z), float64.  ``exchange``: see
    ``forward_transform_slab``."""
    import torch

    from .mesh import family_code, space_code
    from .transforms import wall_inverse

    n, m, K = c_slab.shape
    if exchange is not None:
        if (m, K) != tuple(exchange.cols.shape[1:]):
            raise ValueError(f"coefficient slab {(m, K)} does not match the exchange buffer {tuple(exchange.cols.shape[1:])}")
        exchange._fence()  # nobody still gathers from cols
        _, norm = wall_inverse(c_slab.to(torch.complex128).reshape(n, m * K).contiguous(), mesh.n_x,
                               family_code(mesh.family), space_code(space), mesh.n_y * mesh.n_z,
                               out=exchange.cols.view(mesh.n_x + 1, m * K))
        return exchange.gather_irfft2(norm)
    lines, norm = wall_inverse(c_slab.to(torch.complex128).reshape(n, m * K).contiguous(), mesh.n_x,
                               family_code(mesh.family), space_code(space), mesh.n_y * mesh.n_z)
    planes = kx_to_planes(lines.reshape(mesh.n_x + 1, m, K), mesh.n_y, group, rows_of)
    return plane_irfft2(planes, mesh.n_y, mesh.n_z, norm)
