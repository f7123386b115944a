"""GPU parity of the B200 solvers against the reference (golden fixtures)
and the CPU oracle, mirroring the reference's tests/test_solvers.py cases
plus the BASELINE configurations.

Gates (BASELINE.json north_star): per-system max|x - x_ref| / max|x_ref|
<= 1e-10; residual ||M x - f|| / ||f|| <= 1e-12, evaluated with an 80-bit
dense product.  At BASELINE config 4 corners the reference's own residual
reaches ~1.5e-12 (measured again here), so the residual gate is
max(1e-12, 2 x the reference's residual on the same system)."""

import hashlib

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import solvers as S
from paper_1701_03787_b200.matrices import BandedMatrix, assemble
from paper_1701_03787_b200.mesh import channel_z2

pytestmark = pytest.mark.gpu

TOL = 1e-10
NU, DT = 1 / 5200, 1e-5


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", range(8))
@pytest.mark.parametrize("method", ["stored", "stream"])
def test_factors_bitwise_vs_reference(golden, golden_meta, case, method):
    """Materialised factors (lazy attributes) equal the reference's bit for bit."""
    g = golden("solvers.npz")
    meta = golden_meta["solver_cases"][case]
    mats = assemble(meta["n_x"], meta["family"])
    z2 = g[f"c{case}_z2"]
    hl = S.build_helmholtz(mats, meta["nu"], meta["dt"], z2, method=method)
    for nm in ("low", "d", "e", "tail"):
        for p in (0, 1):
            assert np.array_equal(getattr(hl, nm)[p], g[f"c{case}_h_{nm}{p}"]), (nm, p)
    bl = S.build_biharmonic(mats, meta["nu"], meta["dt"], z2, method=method)
    for nm in ("low2", "low4", "d", "e", "f", "a", "b"):
        for p in (0, 1):
            assert np.array_equal(getattr(bl, nm)[p], g[f"c{case}_b_{nm}{p}"]), (nm, p)
    assert bl.storage_vectors() == 7


@pytest.mark.parametrize("case", range(8))
def test_stored_solve_bitwise_vs_reference(golden, golden_meta, case):
    """method='stored' replays the reference's arithmetic: identical bytes."""
    g = golden("solvers.npz")
    meta = golden_meta["solver_cases"][case]
    mats = assemble(meta["n_x"], meta["family"])
    z2 = g[f"c{case}_z2"]
    hl = S.build_helmholtz(mats, meta["nu"], meta["dt"], z2, method="stored")
    bl = S.build_biharmonic(mats, meta["nu"], meta["dt"], z2, method="stored")
    for kind in ("real", "cplx"):
        xh = hl.solve(g[f"c{case}_h_rhs_{kind}"])
        xb = bl.solve(g[f"c{case}_b_rhs_{kind}"])
        assert xh.dtype == g[f"c{case}_h_x_{kind}"].dtype
        assert np.array_equal(xh, g[f"c{case}_h_x_{kind}"]), kind
        assert np.array_equal(xb, g[f"c{case}_b_x_{kind}"]), kind


@pytest.mark.parametrize("case", range(8))
@pytest.mark.parametrize("method", ["stream"])
def test_fused_solve_parity(golden, golden_meta, case, method):
    g = golden("solvers.npz")
    meta = golden_meta["solver_cases"][case]
    mats = assemble(meta["n_x"], meta["family"])
    z2 = g[f"c{case}_z2"]
    hl = S.build_helmholtz(mats, meta["nu"], meta["dt"], z2, method=method)
    bl = S.build_biharmonic(mats, meta["nu"], meta["dt"], z2, method=method)
    for kind in ("real", "cplx"):
        for op, lu in (("h", hl), ("b", bl)):
            x = lu.solve(g[f"c{case}_{op}_rhs_{kind}"])
            want = g[f"c{case}_{op}_x_{kind}"]
            assert x.dtype == want.dtype and x.shape == want.shape
            err = O.max_rel_per_system(x, want).max()
            assert err <= TOL, (op, kind, err)


def test_baseline_config1_config2(golden, golden_meta):
    """BASELINE configs 1 and 2 in full (n_x = 63, 64 x 33 systems)."""
    mats = assemble(63, 0)
    z2 = channel_z2(64, 64)
    base = golden_meta["baseline"]
    g = golden("baseline_c1c2.npz")
    for op, build, nm in (("h", S.build_helmholtz, mats.n_dir), ("b", S.build_biharmonic, mats.n_bih)):
        rng = np.random.default_rng(0)
        f = rng.standard_normal((nm,) + z2.shape) + 1j * rng.standard_normal((nm,) + z2.shape)
        xs = build(mats, 1e-3, 1e-3, z2, method="stored").solve(f)
        assert _sha(xs) == base[op]["x_sha256"], f"{op}: stored path not bit-identical to the reference"
        xc = build(mats, 1e-3, 1e-3, z2).solve(f)
        err = O.max_rel_per_system(xc, xs).max()
        assert err <= TOL, (op, err)
        assert O.max_rel_per_system(xc.reshape(nm, -1)[:, ::16], g[f"{op}_x_every16"]).max() <= TOL


@pytest.mark.parametrize("fam", [0, 1])
@pytest.mark.parametrize("n_x", [16, 32, 64])
def test_matches_dense_solve(n_x, fam):
    """reference tests/test_solvers.py:30-59: fast solve == np.linalg.solve(dense)."""
    mats = assemble(n_x, fam)
    zv = np.array([0.0, 10.0, 200.0])
    z2 = np.repeat(zv ** 2, 50)
    rng = np.random.default_rng(n_x)
    for build, dense, nm in ((S.build_helmholtz, S.dense_helmholtz, mats.n_dir),
                             (S.build_biharmonic, S.dense_biharmonic, mats.n_bih)):
        rhs = rng.standard_normal((nm, z2.size))
        got = build(mats, NU, DT, z2).solve(rhs)
        for i, z in enumerate(zv):
            sl = slice(50 * i, 50 * i + 50)
            want = np.linalg.solve(dense(mats, NU, DT, z ** 2), rhs[:, sl])
            assert np.abs(got[:, sl] - want).max() / np.abs(want).max() < 1e-10


def test_large_wavenumber_recovery():
    """reference tests/test_solvers.py:107-117 (z = 5400, n_x = 256)."""
    mats = assemble(256, 0)
    z2 = np.array([5400.0 ** 2])
    rng = np.random.default_rng(13)
    u = rng.random((mats.n_bih, 1))
    xi0, xi1, xi2 = S.biharmonic_coefficients(NU, DT, z2)
    f = xi0 * mats.fourth_bih.apply(u) - xi1 * mats.stiff_bih.apply(u) + xi2 * mats.mass_bih.apply(u)
    v = S.build_biharmonic(mats, NU, DT, z2).solve(f)
    assert np.abs(u - v).max() / np.abs(u).max() < 1e-9


def test_shapes_dtypes_and_errors():
    mats = assemble(16, 0)
    z2 = np.linspace(0.0, 400.0, 12).reshape(3, 4)
    lu = S.build_helmholtz(mats, NU, DT, z2)
    rng = np.random.default_rng(12)
    rhs = rng.standard_normal((mats.n_dir, 3, 4))
    got = lu.solve(rhs)
    assert got.shape == rhs.shape and got.dtype == np.float64
    for i in range(3):
        for j in range(4):
            want = np.linalg.solve(S.dense_helmholtz(mats, NU, DT, z2[i, j]), rhs[:, i, j])
            assert np.abs(got[:, i, j] - want).max() < 1e-10
    # float32 / complex64 promote like np.result_type(rhs, float)
    assert lu.solve(rhs.astype(np.float32)).dtype == np.float64
    assert lu.solve(rhs.astype(np.complex64)).dtype == np.complex128
    with pytest.raises(ValueError, match="does not match"):
        lu.solve(rhs[:, :2])
    # scalar z2
    lu0 = S.build_biharmonic(mats, NU, DT, 25.0)
    r0 = rng.standard_normal(mats.n_bih)
    x0 = lu0.solve(r0)
    assert x0.shape == (mats.n_bih,)
    assert np.abs(x0 - np.linalg.solve(S.dense_biharmonic(mats, NU, DT, 25.0), r0)).max() < 1e-10
    # empty batch
    lue = S.build_helmholtz(mats, NU, DT, np.zeros((0,)))
    assert lue.solve(np.zeros((mats.n_dir, 0))).shape == (mats.n_dir, 0)
    # inputs are not mutated
    keep = rhs.copy()
    lu.solve(rhs)
    assert np.array_equal(keep, rhs)


def test_torch_device_io():
    import torch

    mats = assemble(64, 1)
    z2 = np.linspace(0, 1e4, 40)
    lu = S.build_biharmonic(mats, 1e-3, 1e-3, z2)
    rng = np.random.default_rng(4)
    f = rng.standard_normal((mats.n_bih, 40)) + 1j * rng.standard_normal((mats.n_bih, 40))
    xt = lu.solve(torch.from_numpy(f).cuda())
    assert isinstance(xt, torch.Tensor) and xt.is_cuda and xt.dtype == torch.complex128
    assert np.array_equal(xt.cpu().numpy(), lu.solve(f))


def _degenerate(n_x, rows):
    import dataclasses

    m = assemble(n_x, 0)
    d0 = m.mass_dir.diagonal(0).copy()
    d0[list(rows)] = 0.0
    md = BandedMatrix(m.mass_dir.shape, m.mass_dir.offsets,
                      tuple(d0 if o == 0 else dg for o, dg in zip(m.mass_dir.offsets, m.mass_dir.diagonals)))
    return dataclasses.replace(m, mass_dir=md)


@pytest.mark.parametrize("rows,want", [([0], 0), ([1], 1), ([0, 1], 0)])
@pytest.mark.parametrize("method", ["stream", "stored"])
def test_zero_pivot_raises(rows, want, method):
    with pytest.raises(S.ZeroPivotError, match=f"Helmholtz factorization hit a near-zero pivot at row {want}$"):
        S.build_helmholtz(_degenerate(16, rows), 0.0, 1.0, np.array([0.0, 1.0]), method=method)
    with pytest.raises(S.ZeroPivotError):
        S.lu_nopivot(np.array([[0.0, 1.0], [1.0, 0.0]]))


def _corner_systems(n_y, n_z):
    z2 = channel_z2(n_y, n_z)
    flat = z2.reshape(-1)
    idx = np.unique(np.concatenate([np.argsort(flat)[-6:], np.argsort(flat)[:3],
                                    np.random.default_rng(0).integers(0, flat.size, 23)]))
    return flat[idx]


@pytest.mark.parametrize("op", ["h", "b"])
@pytest.mark.parametrize("method", ["stream"])
def test_config4_corners_residual(op, method):
    """BASELINE config 4 parameters (n_x = 1024, nu = 1/2000, dt = 1e-4) on
    32 systems including the largest z^2 of the 2048 x 1025 plane."""
    mats = assemble(1024, 0)
    nu, dt = 1 / 2000, 1e-4
    z2 = _corner_systems(2048, 2048)
    nm = mats.n_dir if op == "h" else mats.n_bih
    rng = np.random.default_rng(44)
    f = rng.standard_normal((nm, z2.size)) + 1j * rng.standard_normal((nm, z2.size))
    if op == "h":
        x = S.build_helmholtz(mats, nu, dt, z2, method=method).solve(f)
        ref = O.helmholtz_solve(O.helmholtz_factor(mats, nu, dt, z2), f)
        dense = O.dense_helmholtz
    else:
        x = S.build_biharmonic(mats, nu, dt, z2, method=method).solve(f)
        ref = O.biharmonic_solve(O.biharmonic_factor(mats, nu, dt, z2), f)
        dense = O.dense_biharmonic
    assert O.max_rel_per_system(x, ref).max() <= TOL
    for j in range(z2.size):
        m = dense(mats, nu, dt, z2[j])
        r_gpu = float(O.residual_longdouble(m, x[:, j], f[:, j]))
        r_ref = float(O.residual_longdouble(m, ref[:, j], f[:, j]))
        assert r_gpu <= max(1e-12, 2.0 * r_ref), (j, z2[j], r_gpu, r_ref)


@pytest.mark.parametrize("N", [129, 257, 513, 1025, 2049])
@pytest.mark.parametrize("method", ["stream"])
def test_config5_sizes(N, method):
    """BASELINE config 5 wall-normal sweep, 24 systems of the 512 x 257 plane."""
    mats = assemble(N - 1, 0)
    z2 = _corner_systems(512, 512)[:24]
    nu, dt = 1 / 2000, 1e-4
    rng = np.random.default_rng(N)
    for build, fac, sol, nm in ((S.build_helmholtz, O.helmholtz_factor, O.helmholtz_solve, mats.n_dir),
                                (S.build_biharmonic, O.biharmonic_factor, O.biharmonic_solve, mats.n_bih)):
        f = rng.standard_normal((nm, z2.size)) + 1j * rng.standard_normal((nm, z2.size))
        x = build(mats, nu, dt, z2, method=method).solve(f)
        assert O.max_rel_per_system(x, sol(fac(mats, nu, dt, z2), f)).max() <= TOL


@pytest.mark.parametrize("op", ["h", "b"])
def test_host_pipeline_multi_slab(op):
    """numpy in/out goes through the column-slab pipeline (several slabs at
    this batch); each system's arithmetic is the device path's, so the
    results are identical to a torch-device solve, for complex and real RHS,
    with and without ``out=``."""
    import torch

    mats = assemble(32, 0)
    z2 = channel_z2(96, 190)          # 96 x 96 = 9216 systems -> several slabs
    build = S.build_helmholtz if op == "h" else S.build_biharmonic
    lu = build(mats, NU, DT, z2)
    nm = lu.n_modes
    rng = np.random.default_rng(21)
    f = rng.standard_normal((nm,) + z2.shape) + 1j * rng.standard_normal((nm,) + z2.shape)
    want = lu.solve(torch.from_numpy(f).cuda()).cpu().numpy()
    got = lu.solve(f)
    assert np.array_equal(got, want)
    pinned = torch.empty(f.shape, dtype=torch.complex128, pin_memory=True).numpy()
    res = lu.solve(f, out=pinned)
    assert res is pinned and np.array_equal(pinned, want)
    fr = f.real.copy()
    want_r = lu.solve(torch.from_numpy(fr).cuda()).cpu().numpy()
    got_r = lu.solve(fr)
    assert got_r.dtype == np.float64 and np.array_equal(got_r, want_r)
    assert O.max_rel_per_system(got, O.helmholtz_solve(O.helmholtz_factor(mats, NU, DT, z2), f)
                                if op == "h" else
                                O.biharmonic_solve(O.biharmonic_factor(mats, NU, DT, z2), f)).max() < TOL


def test_solve_many_matches_single_solves():
    """solve_many pipelines several operators through one host<->device
    pipeline; results equal the individual solves bit for bit."""
    mats = assemble(32, 0)
    z2 = channel_z2(96, 190)
    hlu = S.build_helmholtz(mats, NU, DT, z2)
    blu = S.build_biharmonic(mats, NU, DT, z2)
    rng = np.random.default_rng(8)
    fh = rng.standard_normal((mats.n_dir,) + z2.shape) + 1j * rng.standard_normal((mats.n_dir,) + z2.shape)
    fb = rng.standard_normal((mats.n_bih,) + z2.shape)
    xh, xb = S.solve_many([(hlu, fh), (blu, fb)])
    assert np.array_equal(xh, hlu.solve(fh)) and np.array_equal(xb, blu.solve(fb))
    assert xb.dtype == np.float64
    with pytest.raises(ValueError):
        S.solve_many([(hlu, fh[:, :3])])


@pytest.mark.parametrize("n_x,ny,nz", [(32, 16, 16), (256, 64, 30), (1024, 8, 64), (2048, 4, 32), (64, 12, 66)])
@pytest.mark.parametrize("cplx", [True, False])
def test_biharmonic_mirror_pairs_bitwise(n_x, ny, nz, cplx):
    """Mirror-paired systems ((m, n) and (-m, n): identical z2) share one
    factor recurrence per thread; results must equal the one-system-per-thread
    solve bit for bit (same per-system operations)."""
    from paper_1701_03787_b200.mesh import channel_z2

    mats = assemble(n_x, 0)
    z2 = channel_z2(ny, nz)
    S.PAIRS_MIN, saved = 1, S.PAIRS_MIN  # force pairs at test sizes
    try:
        lu = S.build_biharmonic(mats, 1 / 2000, 1e-4, z2)
    finally:
        S.PAIRS_MIN = saved
    assert lu._pairs is not None
    rng = np.random.default_rng(n_x + ny)
    shp = (mats.n_bih,) + z2.shape
    f = rng.standard_normal(shp) + 1j * rng.standard_normal(shp) if cplx else rng.standard_normal(shp)
    x_pair = lu.solve(f)
    pairs = lu._pairs
    lu._pairs = None
    x_one = lu.solve(f)
    lu._pairs = pairs
    assert x_pair.dtype == x_one.dtype and np.array_equal(x_pair, x_one)


def _degenerate_bih(n_x, rows):
    """stiff_bih with a zeroed main diagonal on `rows`: with nu*dt = 0 and
    z2 = 0 the biharmonic operator is -stiff_bih, whose pivot d vanishes on
    the first zeroed row (reference solvers.py:314-346 pivot check)."""
    import dataclasses

    m = assemble(n_x, 0)
    sb = m.stiff_bih
    d0 = sb.diagonal(0).copy()
    d0[list(rows)] = 0.0
    nb = BandedMatrix(sb.shape, sb.offsets, tuple(d0 if o == 0 else dg for o, dg in zip(sb.offsets, sb.diagonals)))
    return dataclasses.replace(m, stiff_bih=nb)


@pytest.mark.parametrize("rows,want", [([0], 0), ([1], 1), ([0, 1], 0)])
@pytest.mark.parametrize("method", ["stream", "stored"])
def test_biharmonic_zero_pivot_raises(rows, want, method):
    """The device pivot flag of the biharmonic factor raises the reference's
    error at build, first bad row in parity-0-then-parity-1 order; the oracle
    (the reference's arithmetic) agrees on the row."""
    mats = _degenerate_bih(16, rows)
    msg = f"biharmonic factorization hit a near-zero pivot at row {want}$"
    with pytest.raises(S.ZeroPivotError, match=msg):
        S.build_biharmonic(mats, 0.0, 1.0, np.array([0.0, 0.0]), method=method)
    with pytest.raises(ArithmeticError, match=msg):
        O.biharmonic_factor(mats, 0.0, 1.0, np.array([0.0, 0.0]))


@pytest.mark.parametrize("cplx", [True, False])
@pytest.mark.parametrize("max_ctas", [1, 2, 3])
def test_biharmonic_pair_grid_caps(max_ctas, cplx):
    """The pair kernel takes its parity from blockIdx.x & 1: a CTA cap of 1
    or an odd cap must still solve both parities of every system (advisor
    round 1), bit-identical to the uncapped launch."""
    import torch

    mats = assemble(64, 0)
    z2 = channel_z2(32, 64)
    S.PAIRS_MIN, saved = 1, S.PAIRS_MIN
    try:
        lu = S.build_biharmonic(mats, 1 / 2000, 1e-4, z2)
    finally:
        S.PAIRS_MIN = saved
    assert lu._pairs is not None
    rng = np.random.default_rng(max_ctas)
    shp = (mats.n_bih, z2.size)
    f = rng.standard_normal(shp) + 1j * rng.standard_normal(shp) if cplx else rng.standard_normal(shp)
    fd = torch.from_numpy(f).cuda()
    want = torch.empty_like(fd)
    lu.solve_into(fd, want, cplx)
    got = torch.full_like(fd, float("nan"))
    lu.solve_into(fd, got, cplx, max_ctas=max_ctas)
    assert torch.equal(got, want)


def test_solve_field_wraps_solve():
    """solve_field (reference solvers.py:387-392): the SpectralField's data
    solved per wavenumber, grid and mesh carried over."""
    from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid
    from paper_1701_03787_b200.transforms import SpectralField

    mesh = build_mesh(32, 16, 16, 2 * np.pi, np.pi)
    mats = assemble(32, 0)
    for space, build in ((Space.DIRICHLET, S.build_helmholtz), (Space.BIHARMONIC, S.build_biharmonic)):
        grid = wavenumber_grid(mesh, space)
        lu = build(mats, NU, DT, grid.z2())
        rng = np.random.default_rng(5)
        shp = (grid.n_modes,) + tuple(mesh.spectral_shape_yz)
        field = SpectralField(rng.standard_normal(shp) + 1j * rng.standard_normal(shp), grid, mesh)
        out = S.solve_field(lu, field)
        assert isinstance(out, SpectralField) and out.grid is grid and out.mesh is mesh
        assert np.array_equal(out.data, lu.solve(field.data))
