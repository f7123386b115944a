"""Multi-rank host logic on CPU (gloo, world size 2): the kx-slab split used
by bench.py / multi-GPU runs covers the plane exactly, per-rank solves of the
slabs reassemble into the single-process result, and the timing reduction is
a max over ranks.  The per-rank solver here is the CPU oracle (the product has
no CPU path); on GPUs each rank runs the same slab through the B200 solver."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1701_03787_b200.shard import assemble_slabs, kx_rows_folded, kx_slab, slab_of


def test_kx_slab_partition():
    for n_y in (1, 7, 64, 2048):
        for world in (1, 2, 3, 8):
            spans = [kx_slab(n_y, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n_y
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        kx_slab(8, 2, 2)


def test_kx_rows_folded_partition_and_pairs():
    """Folded slabs (bench.py multi-GPU): every kx row on exactly one rank,
    balanced, and every rank's z2 rows form whole mirror pairs, so the
    biharmonic pair kernel applies on every rank."""
    from paper_1701_03787_b200.mesh import channel_z2
    from paper_1701_03787_b200.solvers import mirror_pairs

    for n_y in (8, 64, 2048):
        z2 = channel_z2(n_y, 16)
        for world in (1, 2, 3, 8):
            parts = [kx_rows_folded(n_y, r, world) for r in range(world)]
            allr = np.concatenate(parts)
            assert sorted(allr.tolist()) == list(range(n_y))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 3
            for rows in parts:
                if len([r for r in rows if r not in (0, n_y // 2)]) < 2:
                    continue  # more ranks than pairs: this rank holds no pair
                pr = mirror_pairs(z2[rows])
                assert pr is not None
                zf = z2[rows].reshape(-1)
                assert np.array_equal(zf[pr[0]], zf[pr[1]])
                assert sorted(np.concatenate([pr[0], pr[1][pr[1] != pr[0]]]).tolist()) == list(range(zf.size))
    assert list(kx_rows_folded(7, 0, 1)) == list(range(7))  # odd n_y: plain slab


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch

    from oracle import shen_oracle as O
    from paper_1701_03787_b200.matrices import assemble
    from paper_1701_03787_b200.mesh import channel_z2

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mats = assemble(32, 0)
    n_y, n_z = 12, 8
    z2 = channel_z2(n_y, n_z)
    rng = np.random.default_rng(0)
    f = rng.standard_normal((mats.n_bih,) + z2.shape) + 1j * rng.standard_normal((mats.n_bih,) + z2.shape)
    z2s = slab_of(z2, n_y, rank, world, axis=0)
    fs = np.ascontiguousarray(slab_of(f, n_y, rank, world, axis=1))
    xs = O.biharmonic_solve(O.biharmonic_factor(mats, 1e-3, 1e-3, z2s), fs)
    parts = [None] * world
    dist.all_gather_object(parts, xs)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = O.biharmonic_solve(O.biharmonic_factor(mats, 1e-3, 1e-3, z2), f)
        np.save(os.path.join(out_dir, "ok.npy"),
                np.array([np.array_equal(assemble_slabs(parts, axis=1), full), t.item() == world]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_solve_gloo(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    ok = np.load(tmp_path / "ok.npy")
    assert ok.all(), ok


def test_plane_slab_partition():
    from paper_1701_03787_b200.distributed import plane_slab

    for n in (1, 9, 257):
        for world in (1, 2, 3, 8):
            spans = [plane_slab(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def _exchange_worker(rank, world, port, out_dir):
    import torch

    from paper_1701_03787_b200.distributed import kx_rows, kx_to_planes, plane_slab, planes_to_kx

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oks = []
    # folded rows (the default: the solver's row set, whole (m, -m) pairs) and
    # contiguous slabs; uneven splits on both axes
    for n_planes, n_y, K, rows_of in ((9, 12, 5, None), (9, 7, 5, None),
                                      (9, 7, 5, lambda n, r, w: np.arange(*kx_slab(n, r, w)))):
        g = torch.Generator().manual_seed(4)
        full = torch.complex(torch.randn(n_planes, n_y, K, generator=g, dtype=torch.float64),
                             torch.randn(n_planes, n_y, K, generator=g, dtype=torch.float64))
        lo, hi = plane_slab(n_planes, rank, world)
        cols = planes_to_kx(full[lo:hi].clone(), n_planes, rows_of=rows_of)
        rows = kx_rows(n_y, rank, world, rows_of)
        if rows_of is None:
            oks.append(np.array_equal(rows, kx_rows_folded(n_y, rank, world)))
        oks.append(torch.equal(cols, full[:, torch.from_numpy(rows), :]))
        back = kx_to_planes(cols, n_y, rows_of=rows_of)
        oks.append(torch.equal(back, full[lo:hi]))
    np.save(os.path.join(out_dir, f"ex{rank}.npy"), np.array(oks))
    dist.destroy_process_group()


def test_transform_exchange_gloo(tmp_path):
    """The all-to-all of the slab-decomposed transforms (distributed.py):
    x-planes -> kx rows -> x-planes reproduces the global transpose exactly on
    uneven splits, for the folded rows the solver slabs use (the default) and
    for contiguous slabs (world size 2, gloo; NCCL over NVLink on GPUs)."""
    world = 2
    mp.spawn(_exchange_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.load(tmp_path / f"ex{r}.npy").all()
