"""The multi-rank product path end to end on the device: two ranks (one
process each) on cuda:0, gloo for the exchange and the gathers (NCCL over
NVLink on a multi-GPU node).  Each rank holds its x-planes of a physical
field and runs the slab-decomposed pipeline (distributed.py):

    rfft2 (cuFFT) -> all-to-all to its folded kx rows -> fused wall-normal
    forward kernel -> Helmholtz / biharmonic solves of its rows (mirror-pair
    kernel) -> inverse wall-normal kernel -> all-to-all back -> irfft2.

Rank 0 gathers the pieces and checks them against the single-process
product pipeline to 1e-13 (cuFFT plans of other batch sizes may round
differently), and that the full-plane solve of the gathered coefficients
reproduces the gathered solutions bit for bit (the per-system arithmetic of
the solvers does not depend on the decomposition or the pairing).  No kernel of one
rank waits on another rank: the exchange is host-side."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch

    from paper_1701_03787_b200 import distributed as D, solvers as S, transforms as T
    from paper_1701_03787_b200.matrices import assemble
    from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    S.PAIRS_MIN = 1  # the mirror-pair kernel on every rank's rows
    mesh = build_mesh(64, 32, 24, 2 * np.pi, np.pi)
    mats = assemble(64, mesh.family)
    nu, dt = 1 / 2000, 1e-4
    g = torch.Generator(device="cuda").manual_seed(11)
    u = torch.rand(mesh.shape, generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    lo, hi = D.plane_slab(mesh.n_x + 1, rank, world)
    rows = D.kx_rows(mesh.n_y, rank, world)
    res = {}
    for space, build in ((Space.DIRICHLET, S.build_helmholtz), (Space.BIHARMONIC, S.build_biharmonic)):
        z2 = wavenumber_grid(mesh, space).z2()
        c = D.forward_transform_slab(u[lo:hi].contiguous(), mesh, space)            # (n_modes, rows_r, K)
        x = build(mats, nu, dt, z2[rows]).solve(c)
        back = D.inverse_transform_slab(x, mesh, space)                              # (planes_r, n_y, n_z)
        parts_c = [None] * world
        parts_x = [None] * world
        parts_b = [None] * world
        dist.all_gather_object(parts_c, (rows, c.cpu().numpy()))
        dist.all_gather_object(parts_x, x.cpu().numpy())
        dist.all_gather_object(parts_b, back.cpu().numpy())
        if rank == 0:
            full_c = T.forward_transform(T.PhysicalField(u, mesh), space).data
            full_x = build(mats, nu, dt, z2).solve(full_c)
            full_b = T.inverse_transform(T.SpectralField(full_x, wavenumber_grid(mesh, space), mesh)).data
            full_c, full_x, full_b = full_c.cpu().numpy(), full_x.cpu().numpy(), full_b.cpu().numpy()
            gc = np.empty_like(full_c)
            gx = np.empty_like(full_x)
            for (r_rows, cr), xr in zip(parts_c, parts_x):
                gc[:, r_rows] = cr
                gx[:, r_rows] = xr
            gb = np.concatenate(parts_b, axis=0)
            same_x = np.array_equal(build(mats, nu, dt, z2).solve(gc), gx)
            rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())  # noqa: E731
            res[space.name] = [rel(gc, full_c), rel(gx, full_x), rel(gb, full_b), bool(same_x)]
    if rank == 0:
        np.save(os.path.join(out_dir, "res.npy"), np.array([res], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_pipeline_one_gpu(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = np.load(tmp_path / "res.npy", allow_pickle=True)[0]
    for space, (err_c, err_x, err_b, same_x) in res.items():
        assert err_c < 1e-13 and err_x < 1e-13 and err_b < 1e-13, (space, err_c, err_x, err_b)
        assert same_x, f"{space}: slab solves differ from the full-plane solve of the same coefficients"
    assert set(res) == {"DIRICHLET", "BIHARMONIC"}


# ---------------------------------------------------------------- exchange fused into the plane FFT kernels
def _peer_worker(rank, world, port, out_dir):
    """Slab transforms with the kx-row exchange inside the plane FFT kernels
    (distributed.PeerExchange: every rank's buffer opened on the others by
    CUDA IPC; here all ranks share cuda:0) against the all-to-all route."""
    import torch

    from paper_1701_03787_b200 import distributed as D, transforms as T
    from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    mesh = build_mesh(16, 256, 256, 2 * np.pi, np.pi)
    N = mesh.n_x + 1
    g = torch.Generator(device="cuda").manual_seed(3)
    u = torch.rand(mesh.shape, generator=g, device="cuda", dtype=torch.float64) * 2 - 1
    lo, hi = D.plane_slab(N, rank, world)
    rows = D.kx_rows(mesh.n_y, rank, world)
    ex = D.PeerExchange(N, mesh.n_y, mesh.n_z)
    res = {}
    for space in (Space.DIRICHLET, Space.BIHARMONIC):
        c_a2a = D.forward_transform_slab(u[lo:hi].contiguous(), mesh, space)
        c_p2p = D.forward_transform_slab(u[lo:hi].contiguous(), mesh, space, exchange=ex)
        b_a2a = D.inverse_transform_slab(c_a2a, mesh, space)
        b_p2p = D.inverse_transform_slab(c_a2a, mesh, space, exchange=ex)
        # a second round on the same buffers (reuse ordering)
        c_again = D.forward_transform_slab(u[lo:hi].contiguous(), mesh, space, exchange=ex)
        same = [bool(torch.equal(c_a2a, c_p2p)), bool(torch.equal(b_a2a, b_p2p)), bool(torch.equal(c_again, c_p2p))]
        parts_c = [None] * world
        parts_b = [None] * world
        dist.all_gather_object(parts_c, (rows, c_p2p.cpu().numpy(), same))
        dist.all_gather_object(parts_b, b_p2p.cpu().numpy())
        if rank == 0:
            full_c = T.forward_transform(T.PhysicalField(u, mesh), space).data
            full_b = T.inverse_transform(T.SpectralField(full_c, wavenumber_grid(mesh, space), mesh)).data
            full_c, full_b = full_c.cpu().numpy(), full_b.cpu().numpy()
            gc = np.empty_like(full_c)
            for r_rows, cr, _ in parts_c:
                gc[:, r_rows] = cr
            gb = np.concatenate(parts_b, axis=0)
            rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())  # noqa: E731
            res[space.name] = [rel(gc, full_c), rel(gb, full_b), all(all(s) for _, _, s in parts_c)]
    if rank == 0:
        np.save(os.path.join(out_dir, "res.npy"), np.array([res], dtype=object), allow_pickle=True)
    dist.barrier()
    del ex
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_matches_all_to_all(tmp_path, world):
    mp.start_processes(_peer_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = np.load(tmp_path / "res.npy", allow_pickle=True)[0]
    assert set(res) == {"DIRICHLET", "BIHARMONIC"}
    for space, (err_c, err_b, same) in res.items():
        assert same, f"{space}: fused exchange and all-to-all routes differ bitwise"
        assert err_c < 1e-13 and err_b < 1e-13, (space, err_c, err_b)


def test_peer_exchange_single_rank_is_plain_rfft2():
    """world = 1: the scatter writes the plain (planes, n_y, K) spectrum and
    the gather reads it back."""
    import torch

    from paper_1701_03787_b200 import distributed as D, transforms as T

    g = torch.Generator(device="cuda").manual_seed(9)
    u = torch.rand((5, 256, 256), generator=g, device="cuda", dtype=torch.float64)
    ex = D.PeerExchange(5, 256, 256)
    cols = ex.scatter_rfft2(u)
    assert torch.equal(cols, T.plane_rfft2(u))
    back = ex.gather_irfft2()
    assert torch.equal(back, T.plane_irfft2(cols, 256, 256))
    assert float((back - u).abs().max()) < 1e-14
    with pytest.raises(ValueError):
        D.PeerExchange(5, 128, 256)
    with pytest.raises(ValueError):
        ex.scatter_rfft2(u[:4])
