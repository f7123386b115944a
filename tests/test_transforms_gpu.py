"""GPU parity of the Shen transforms (reference transforms.py) against the
reference's golden outputs and the CPU oracle.

The device DCTs go through cuFFT instead of pocketfft, so results agree to
rounding, not bitwise.  Gate (fp64): max|got - ref| <= TOL * max|ref| per
array, TOL = 1e-12 (well inside BASELINE.json's 1e-10)."""

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import transforms as T
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import PointFamily, Space, build_mesh, wavenumber_grid

pytestmark = pytest.mark.gpu

TOL = 1e-12
FAMS = (PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO)
SPACES = (Space.CHEBYSHEV, Space.DIRICHLET, Space.BIHARMONIC)


def _close(got, want, tol=TOL):
    got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
    assert got.shape == want.shape, (got.shape, want.shape)
    assert got.dtype == want.dtype, (got.dtype, want.dtype)
    scale = max(np.abs(want).max(), 1e-300)
    err = np.abs(got - want).max() / scale
    assert err <= tol, err
    return err


@pytest.mark.parametrize("n_x", [8, 16, 32])
@pytest.mark.parametrize("fi", [0, 1])
def test_transforms_vs_reference_golden(golden, n_x, fi, xform_method):
    g = golden("transforms.npz")
    mesh = build_mesh(n_x, 8, 4, 2 * np.pi, np.pi, FAMS[fi])
    key = f"nx{n_x}_f{fi}"
    u = g[key + "_u"]
    for sc, space in enumerate(SPACES):
        c = T.forward_transform(T.PhysicalField(u, mesh), space)
        assert isinstance(c, T.SpectralField) and c.grid.space is space
        _close(c.data, g[f"{key}_s{sc}_fwd"])
        _close(T.forward_scalar_product(T.PhysicalField(u, mesh), space).data, g[f"{key}_s{sc}_fsp"])
        ref_c = T.SpectralField(g[f"{key}_s{sc}_fwd"], wavenumber_grid(mesh, space), mesh)
        back = T.inverse_transform(ref_c)
        assert isinstance(back, T.PhysicalField)
        _close(back.data, g[f"{key}_s{sc}_inv"])


@pytest.mark.parametrize("fi", [0, 1])
def test_1d_blocks_vs_reference_golden(golden, fi):
    g = golden("transforms.npz")
    v = g[f"blk_f{fi}_v"]
    fam = FAMS[fi]
    _close(T.chebyshev_scalar(v, fam), g[f"blk_f{fi}_cheb_scalar"])
    _close(T.chebyshev_evaluate(v, fam), g[f"blk_f{fi}_cheb_eval"])
    for sc, space in ((1, Space.DIRICHLET), (2, Space.BIHARMONIC)):
        _close(T.shen_scalar(v, fam, space), g[f"blk_f{fi}_s{sc}_shen_scalar"])
        w = v[:13 - space.mode_drop]
        _close(T.shen_expand(w, space, 12), g[f"blk_f{fi}_s{sc}_expand"])
        _close(T.mass_solve(w, space, 12, fam), g[f"blk_f{fi}_s{sc}_mass"])


@pytest.mark.parametrize("fi", [0, 1])
def test_mass_factors_match_oracle(fi):
    for sc in (1, 2):
        mine = T.mass_cholesky(24, FAMS[fi], SPACES[sc])
        want = O.mass_cholesky(assemble(24, fi), sc)
        for p in (0, 1):
            assert np.array_equal(mine[p], want[p])


@pytest.fixture(params=["wall", "fft"])
def xform_method(request, monkeypatch):
    monkeypatch.setattr(T, "XFORM_METHOD", request.param)
    return request.param


@pytest.mark.parametrize("fi", [0, 1])
@pytest.mark.parametrize("n_x", [64, 256])
def test_transforms_vs_oracle_larger(fi, n_x, xform_method):
    """Larger wall-normal sizes (cfg3's n_x = 256) on a small y/z plane,
    both wall-normal routes (fused kernel, cuFFT pipeline)."""
    mesh = build_mesh(n_x, 12, 10, 2 * np.pi, np.pi, FAMS[fi])
    mats = assemble(n_x, fi)
    rng = np.random.default_rng(n_x + fi)
    u = rng.uniform(-1, 1, mesh.shape)
    for sc, space in enumerate(SPACES):
        c = T.forward_transform(T.PhysicalField(u, mesh), space)
        want = O.forward_transform(u, sc, fi == 1, mats)
        _close(c.data, want)
        _close(T.forward_scalar_product(T.PhysicalField(u, mesh), space).data,
               O.forward_scalar_product(u, sc, fi == 1))
        back = T.inverse_transform(T.SpectralField(want, c.grid, mesh))
        _close(back.data, O.inverse_transform(want, sc, fi == 1, n_x, mesh.n_y, mesh.n_z))


@pytest.mark.parametrize("fi", [0, 1])
def test_many_lines_vs_oracle(fi):
    """544 Fourier lines: many line tiles of the fused kernel, the last one
    partial (TMA clips its columns); same gates as above."""
    mesh = build_mesh(64, 32, 32, 2 * np.pi, np.pi, FAMS[fi])
    mats = assemble(64, fi)
    u = np.random.default_rng(5 + fi).uniform(-1, 1, mesh.shape)
    for sc, space in enumerate(SPACES):
        c = T.forward_transform(T.PhysicalField(u, mesh), space)
        want = O.forward_transform(u, sc, fi == 1, mats)
        _close(c.data, want)
        _close(T.forward_scalar_product(T.PhysicalField(u, mesh), space).data,
               O.forward_scalar_product(u, sc, fi == 1))
        back = T.inverse_transform(T.SpectralField(want, c.grid, mesh))
        _close(back.data, O.inverse_transform(want, sc, fi == 1, 64, mesh.n_y, mesh.n_z))


@pytest.mark.parametrize("fi", [0, 1])
def test_real_inputs_stay_real(fi):
    rng = np.random.default_rng(5)
    v = rng.standard_normal((17, 4, 2))
    fam = FAMS[fi]
    _close(T.chebyshev_scalar(v, fam), O.chebyshev_scalar(v, fi == 1))
    _close(T.chebyshev_evaluate(v, fam), O.chebyshev_evaluate(v, fi == 1))
    for sc in (0, 1, 2):
        _close(T.shen_scalar(v, fam, SPACES[sc]), O.shen_scalar(v, fi == 1, sc))
    mats = assemble(16, fi)
    for sc, drop in ((1, 2), (2, 4)):
        w = v[:17 - drop]
        _close(T.shen_expand(w, SPACES[sc], 16), O.shen_expand(w, sc, 16))
        _close(T.mass_solve(w, SPACES[sc], 16, fam), O.mass_solve(w, sc, mats))
    # 1-D vector (no trailing axes)
    _close(T.chebyshev_scalar(v[:, 0, 0], fam), O.chebyshev_scalar(v[:, 0, 0], fi == 1))


def test_torch_inputs_stay_on_device():
    import torch

    mesh = build_mesh(16, 8, 6, 2 * np.pi, np.pi, PointFamily.GAUSS)
    rng = np.random.default_rng(11)
    u = rng.uniform(-1, 1, mesh.shape)
    ud = torch.from_numpy(u).cuda()
    c = T.forward_transform(T.PhysicalField(ud, mesh), Space.DIRICHLET)
    assert isinstance(c.data, torch.Tensor) and c.data.is_cuda and c.data.dtype == torch.complex128
    _close(c.data, O.forward_transform(u, 1, False, assemble(16, 0)))
    back = T.inverse_transform(c)
    assert isinstance(back.data, torch.Tensor) and back.data.dtype == torch.float64
    cc = c.copy()
    assert cc.data.data_ptr() != c.data.data_ptr()
    assert float(c.zeros_like().data.abs().max()) == 0.0


def test_errors_match_reference():
    mesh = build_mesh(8, 4, 4, 1.0, 1.0)
    with pytest.raises(ValueError):
        T.PhysicalField(np.zeros((8, 4, 4)), mesh)
    with pytest.raises(ValueError):
        T.SpectralField(np.zeros((9, 4, 4), complex), wavenumber_grid(mesh, Space.DIRICHLET), mesh)
    with pytest.raises(ValueError, match="Chebyshev mass solve"):
        T.mass_solve(np.zeros((9, 2)), Space.CHEBYSHEV, 8, PointFamily.GAUSS)


@pytest.mark.parametrize("fi", [0, 1])
@pytest.mark.parametrize("space", [Space.DIRICHLET, Space.BIHARMONIC, Space.CHEBYSHEV])
def test_cfg3_projection_round_trip(fi, space, xform_method):
    """BASELINE config 3 sizes (physical 257 x 256 x 256): forward(inverse(c))
    recovers any coefficient field of the space (size-independent property),
    and inverse(forward(u)) recovers u for the Chebyshev space."""
    import torch

    mesh = build_mesh(256, 256, 256, 2 * np.pi, np.pi, FAMS[fi])
    grid = wavenumber_grid(mesh, space)
    g = torch.Generator(device="cuda").manual_seed(3 + fi)
    shape = (grid.n_modes,) + mesh.spectral_shape_yz
    c = torch.complex(torch.rand(shape, generator=g, device="cuda", dtype=torch.float64) - 0.5,
                      torch.rand(shape, generator=g, device="cuda", dtype=torch.float64) - 0.5)
    # coefficients of a real field: the kz = 0 and Nyquist columns must be Hermitian in ky
    u = T.inverse_transform(T.SpectralField(c, grid, mesh)).data
    c_herm = T.forward_transform(T.PhysicalField(u, mesh), space).data
    u2 = T.inverse_transform(T.SpectralField(c_herm, grid, mesh)).data
    err = float((u2 - u).abs().max() / u.abs().max())
    assert err < 1e-12, err
    c2 = T.forward_transform(T.PhysicalField(u2, mesh), space).data
    err_c = float((c2 - c_herm).abs().max() / c_herm.abs().max())
    # The biharmonic coefficient round trip is ill-conditioned at n_x = 256
    # (rounding of the point values is amplified by the forward map): the
    # reference itself (oracle, same property, 8 x 8 plane) loses 5.5e-11
    # (Gauss) / 5.8e-11 (Lobatto), both device routes the same.
    # Chebyshev/Dirichlet lose < 1e-13.
    tol_c = 2e-10 if space is Space.BIHARMONIC else 1e-12
    assert err_c < tol_c, err_c


@pytest.mark.parametrize("space", [Space.DIRICHLET, Space.BIHARMONIC])
def test_slab_transforms_single_rank(space):
    """distributed.forward/inverse_transform_slab on one rank equal the
    single-GPU transforms (the all-to-all itself is tested under gloo)."""
    import torch

    from paper_1701_03787_b200 import distributed as D

    mesh = build_mesh(64, 16, 12, 2 * np.pi, np.pi, PointFamily.GAUSS)
    u = torch.rand(mesh.shape, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    c = D.forward_transform_slab(u, mesh, space)
    want = T.forward_transform(T.PhysicalField(u, mesh), space).data
    assert torch.equal(c, want)
    back = D.inverse_transform_slab(c, mesh, space)
    assert torch.equal(back, T.inverse_transform(T.SpectralField(want, wavenumber_grid(mesh, space), mesh)).data)


@pytest.mark.parametrize("n_x,fi,L", [(512, 1, 17000), (512, 0, 2048), (1024, 0, 1024), (1024, 1, 1024)])
def test_large_nx_routes_vs_oracle(n_x, fi, L):
    """The large-n_x routes of wall_forward / wall_inverse (transforms._split_mass:
    fused scalar product + standalone mass-solve kernel when tiles hold few
    lines; the cuFFT route for one-line Gauss tiles) against the oracle."""
    from paper_1701_03787_b200.wall import wall_plan

    N = n_x + 1
    plan = wall_plan(n_x, fi, 1, 0, True, T._cheb_scale(N, fi))
    assert plan is not None and plan.struct.log2_lines <= 2
    rng = np.random.default_rng(n_x + fi)
    x = rng.standard_normal((N, L)) + 1j * rng.standard_normal((N, L))
    mats = assemble(n_x, fi)
    import torch

    xd = torch.from_numpy(x).cuda()
    for sc in (1, 2):
        c = T.wall_forward(xd, n_x, fi, sc, True).cpu().numpy()
        want = O.mass_solve(O.shen_scalar(x, fi == 1, sc), sc, mats)
        _close(c, want, 1e-10 if sc == 2 else TOL)
        back, _ = T.wall_inverse(torch.from_numpy(want).cuda(), n_x, fi, sc, 1)
        _close(back.cpu().numpy(), O.chebyshev_evaluate(O.shen_expand(want, sc, n_x), fi == 1))


@pytest.mark.parametrize("lead", [(1,), (3,), (2, 5)])
def test_plane_fft_vs_numpy(lead):
    """256 x 256 (y, z) planes on the cluster kernel (csrc/shen_plane_fft.cu):
    rfft2 / irfft2 as numpy's (reference transforms.py:181-205), every norm;
    irfft2 ignores the imaginary parts of the z = 0 and z = n_z/2 columns as
    numpy does."""
    import torch

    from paper_1701_03787_b200 import _lib
    from paper_1701_03787_b200.transforms import plane_irfft2, plane_rfft2

    assert _lib.lib().shen_plane_fft_supported(256, 256) == 1
    rng = np.random.default_rng(len(lead))
    x = rng.uniform(-1, 1, lead + (256, 256))
    X = plane_rfft2(torch.from_numpy(x).cuda())
    want = np.fft.rfft2(x)
    assert X.shape == want.shape and X.dtype == torch.complex128
    assert np.abs(X.cpu().numpy() - want).max() <= 1e-14 * np.abs(want).max()
    Y = rng.standard_normal(want.shape) + 1j * rng.standard_normal(want.shape)
    for norm in ("backward", "forward", "ortho"):
        back = plane_irfft2(torch.from_numpy(Y).cuda(), 256, 256, norm).cpu().numpy()
        wantb = np.fft.irfft2(Y, s=(256, 256), norm=norm)
        assert back.shape == wantb.shape
        assert np.abs(back - wantb).max() <= 1e-14 * np.abs(wantb).max(), norm
    rt = plane_irfft2(X, 256, 256).cpu().numpy()
    assert np.abs(rt - x).max() <= 1e-14


@pytest.mark.parametrize("n", [256, 64])
def test_plane_fft_line_factors(n):
    """The per-line factors of the nonlinear term inside the plane transforms:
    rfft2 times a real mask (apply_mask, reference stepper.py:142-144) and
    irfft2 of the spectrum times 1j m (stepper.py:171-172), on the cluster
    kernel (256 x 256) and on the cuFFT fallback (64 x 64); ``out=`` writes
    into a slice of a larger array."""
    import torch

    from paper_1701_03787_b200.transforms import plane_irfft2, plane_rfft2

    rng = np.random.default_rng(n)
    K = n // 2 + 1
    x = rng.uniform(-1, 1, (3, n, n))
    mask = (rng.uniform(0, 1, (n, K)) < 0.6).astype(np.float64)
    X = plane_rfft2(torch.from_numpy(x).cuda(), fac=torch.from_numpy(mask.reshape(-1)).cuda()).cpu().numpy()
    want = np.fft.rfft2(x) * mask
    assert np.abs(X - want).max() <= 1e-14 * np.abs(want).max()
    assert np.all(X[:, mask == 0] == 0)
    Y = rng.standard_normal((3, n, K)) + 1j * rng.standard_normal((3, n, K))
    m = 1j * (2 * np.pi * np.fft.fftfreq(n, 1.0 / n) / 7.0)[:, None] * np.ones((1, K))
    fac = (torch.from_numpy(np.ascontiguousarray(m.real).reshape(-1)).cuda(),
           torch.from_numpy(np.ascontiguousarray(m.imag).reshape(-1)).cuda())
    big = torch.full((2, 3, n, n), 7.0, dtype=torch.float64, device="cuda")
    got = plane_irfft2(torch.from_numpy(Y).cuda(), n, n, "forward", fac=fac, out=big[1])
    assert got.data_ptr() == big[1].data_ptr() and bool((big[0] == 7.0).all())
    wantb = np.fft.irfft2(Y * m, s=(n, n), norm="forward")
    assert np.abs(big[1].cpu().numpy() - wantb).max() <= 1e-14 * np.abs(wantb).max()
    with pytest.raises(ValueError):
        plane_irfft2(torch.from_numpy(Y).cuda(), n, n, out=big)  # wrong shape
    if n == 256:
        with pytest.raises(ValueError):
            plane_rfft2(torch.from_numpy(x).cuda(), fac=torch.from_numpy(mask.reshape(-1)[:-1].copy()).cuda())
