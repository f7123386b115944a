"""Parity at the BASELINE sizes, on the paths the bench runs (SURVEY.md 8(d)
parity gate; reference metric tests/test_solvers.py:41-43).

* config 4 (n_x = 1024, the whole 2048 x 1025 plane built and solved on the
  device exactly as bench.py does): >= 4,096 random systems, every system of
  the self-paired kx rows 0 and 1024, the last items of the mirror-pair table
  (the partial last group) and the largest z^2, against the oracle;
  residuals in 80-bit arithmetic on the largest-z^2 systems;
* config 5: the full 512 x 257 batch for N <= 513, >= 4,096 systems above;
* config 3 transforms: the full 257 x 256 x 256 U(-1, 1) field (seed 0),
  forward / scalar product / inverse, both spaces, against the oracle;
* the reference's own 3-D transforms at n_x = 512 and 1024 (golden,
  tests/golden/big_transforms.npz), where the biharmonic forward map is the
  most ill-conditioned.

Gate: per-system (per Fourier line) max|x - ref| / max|ref| <= 1e-10; the
residual ||M x - f|| / ||f|| <= max(1e-12, 2 x the reference's own residual
on the same system) (the reference itself exceeds 1e-12 at
config-4 corners).
"""

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import solvers as S
from paper_1701_03787_b200 import transforms as T
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import PointFamily, Space, build_mesh, channel_z2

pytestmark = pytest.mark.gpu

TOL = 1e-10
NU4, DT4 = 1 / 2000, 1e-4


def _sample(lu, z2_flat, n_y, n_zh, n_random, seed):
    """System indices: n_random random ones, all systems of kx rows 0 and
    n_y/2 (self-paired rows of the mirror-pair kernels), the systems of the
    last 64 items of the pair table, and the 8 largest z^2."""
    rng = np.random.default_rng(seed)
    parts = [rng.choice(z2_flat.size, size=n_random, replace=False),
             np.arange(n_zh), (n_y // 2) * n_zh + np.arange(n_zh), np.argsort(z2_flat)[-8:]]
    pairs = getattr(lu, "_pairs", None)
    if pairs is not None:
        tail = pairs[:, -64:].cpu().numpy().reshape(-1)
        parts.append(tail[tail >= 0])
    return np.unique(np.concatenate(parts))


def _gather(t, idx):
    import torch

    return t.index_select(1, torch.from_numpy(idx).to(t.device)).cpu().numpy()


@pytest.mark.parametrize("op,method", [("h", "stream"), ("b", "stream")])
def test_config4_full_plane_sampled(op, method):
    import torch

    mats = assemble(1024, 0)
    z2 = channel_z2(2048, 2048)
    build = S.build_helmholtz if op == "h" else S.build_biharmonic
    lu = build(mats, NU4, DT4, z2, method=method)
    nm, B = lu.n_modes, z2.size
    gen = torch.Generator(device="cuda").manual_seed(99 if op == "h" else 98)
    f = torch.randn((nm, B), dtype=torch.complex128, device="cuda", generator=gen)
    x = torch.empty_like(f)
    lu.solve_into(f, x, True)
    torch.cuda.synchronize()
    zf = z2.reshape(-1)
    idx = _sample(lu, zf, 2048, 1025, 4096, 5)
    assert idx.size >= 4096 + 2 * 1025
    fs, xs = _gather(f, idx), _gather(x, idx)
    del f, x, lu
    torch.cuda.empty_cache()
    if op == "h":
        ref = O.helmholtz_solve(O.helmholtz_factor(mats, NU4, DT4, zf[idx]), fs)
        dense = O.dense_helmholtz
    else:
        ref = O.biharmonic_solve(O.biharmonic_factor(mats, NU4, DT4, zf[idx]), fs)
        dense = O.dense_biharmonic
    rel = O.max_rel_per_system(xs, ref)
    assert rel.max() <= TOL, (rel.max(), idx[np.argmax(rel)])
    worst = np.argsort(zf[idx])[-6:]
    for j in worst:
        m = dense(mats, NU4, DT4, zf[idx[j]])
        r_gpu = float(O.residual_longdouble(m, xs[:, j], fs[:, j]))
        r_ref = float(O.residual_longdouble(m, ref[:, j], fs[:, j]))
        assert r_gpu <= max(1e-12, 2.0 * r_ref), (zf[idx[j]], r_gpu, r_ref)


@pytest.mark.parametrize("N", [129, 257, 513, 1025, 2049])
@pytest.mark.parametrize("op,method", [("h", "stream"), ("b", "stream")])
def test_config5_batch(N, op, method):
    """Config 5 (512 x 257 wavenumbers): the whole batch for N <= 513, 4,096
    random systems plus the special rows above."""
    import torch

    mats = assemble(N - 1, 0)
    z2 = channel_z2(512, 512)
    build = S.build_helmholtz if op == "h" else S.build_biharmonic
    lu = build(mats, NU4, DT4, z2, method=method)
    nm, B = lu.n_modes, z2.size
    gen = torch.Generator(device="cuda").manual_seed(N)
    f = torch.randn((nm, B), dtype=torch.complex128, device="cuda", generator=gen)
    x = torch.empty_like(f)
    lu.solve_into(f, x, True)
    zf = z2.reshape(-1)
    idx = np.arange(B) if N <= 513 else _sample(lu, zf, 512, 257, 4096, N)
    fs, xs = _gather(f, idx), _gather(x, idx)
    fac, sol = (O.helmholtz_factor, O.helmholtz_solve) if op == "h" else (O.biharmonic_factor, O.biharmonic_solve)
    ref = sol(fac(mats, NU4, DT4, zf[idx]), fs)
    rel = O.max_rel_per_system(xs, ref)
    assert rel.max() <= TOL, (rel.max(), idx[np.argmax(rel)])


@pytest.fixture(scope="module")
def c3_field():
    return np.random.default_rng(0).uniform(-1, 1, (257, 256, 256))


def _line_rel(got, want):
    return O.max_rel_per_system(got, want).max()


@pytest.mark.parametrize("fi", [0, 1])
@pytest.mark.parametrize("sc", [1, 2])
def test_config3_transforms_full(c3_field, fi, sc):
    """Config 3 at full size on the default route: forward transform, scalar
    product and inverse against the oracle (per Fourier line for spectra,
    relative to the global max for physical values)."""
    import torch

    fam = (PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO)[fi]
    space = (Space.CHEBYSHEV, Space.DIRICHLET, Space.BIHARMONIC)[sc]
    mesh = build_mesh(256, 256, 256, 2 * np.pi, np.pi, fam)
    mats = assemble(256, fi)
    u = c3_field
    ud = torch.from_numpy(u).cuda()
    c = T.forward_transform(T.PhysicalField(ud, mesh), space).data.cpu().numpy()
    want = O.forward_transform(u, sc, fi == 1, mats)
    assert _line_rel(c, want) <= TOL
    s = T.forward_scalar_product(T.PhysicalField(ud, mesh), space).data.cpu().numpy()
    assert _line_rel(s, O.forward_scalar_product(u, sc, fi == 1)) <= TOL
    grid = T.SpectralField(torch.from_numpy(want).cuda(), T.wavenumber_grid(mesh, space), mesh)
    back = T.inverse_transform(grid).data.cpu().numpy()
    want_b = O.inverse_transform(want, sc, fi == 1, 256, 256, 256)
    assert np.abs(back - want_b).max() <= 1e-12 * np.abs(want_b).max()


@pytest.mark.parametrize("n_x", [512, 1024])
@pytest.mark.parametrize("fi", [0, 1])
def test_big_transforms_vs_reference_golden(golden, n_x, fi):
    """The reference's own forward / inverse transforms at n_x = 512, 1024."""
    g = golden("big_transforms.npz")
    fam = (PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO)[fi]
    mesh = build_mesh(n_x, 4, 2, 2 * np.pi, np.pi, fam)
    key = f"nx{n_x}_f{fi}"
    u = g[key + "_u"]
    for sc, space in ((1, Space.DIRICHLET), (2, Space.BIHARMONIC)):
        c = T.forward_transform(T.PhysicalField(u, mesh), space).data
        want = g[f"{key}_s{sc}_fwd"]
        assert _line_rel(c, want) <= TOL, (space, _line_rel(c, want))
        back = T.inverse_transform(T.SpectralField(want, T.wavenumber_grid(mesh, space), mesh)).data
        want_b = g[f"{key}_s{sc}_inv"]
        assert np.abs(back - want_b).max() <= 1e-12 * np.abs(want_b).max()


def test_slab_solves_equal_full_plane():
    """Multi-GPU bookkeeping with the product solver: each rank's folded kx
    rows (shard.kx_rows_folded, the rows bench.py gives every rank) solved on
    their own reassemble into the single-GPU full-plane solution bit for bit
    (ranks emulated one after another on this GPU; the per-rank work has no
    collective)."""
    import torch

    from paper_1701_03787_b200.shard import kx_rows_folded

    mats = assemble(64, 0)
    n_y, n_z = 64, 64
    z2 = channel_z2(n_y, n_z)
    rng = np.random.default_rng(17)
    f = rng.standard_normal((mats.n_bih,) + z2.shape) + 1j * rng.standard_normal((mats.n_bih,) + z2.shape)
    full = S.build_biharmonic(mats, NU4, DT4, z2).solve(f)
    for world in (2, 3, 8):
        got = np.empty_like(full)
        for r in range(world):
            rows = kx_rows_folded(n_y, r, world)
            lu = S.build_biharmonic(mats, NU4, DT4, np.ascontiguousarray(z2[rows]))
            got[:, rows] = lu.solve(np.ascontiguousarray(f[:, rows]))
        assert np.array_equal(got, full), world
    del torch
