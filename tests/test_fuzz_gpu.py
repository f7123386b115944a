"""Randomised sizes against the CPU oracle: the fixed-size parity tests use
round numbers, these draw odd and awkward ones (wall-normal sizes that are
not multiples of the checkpoint spacing, batches that end inside a warp or a
CTA group, planes with and without mirror pairs, real and complex right-hand
sides, both point families).  Same gates as the reference's own tests
(tests/test_solvers.py:41-43, tests/test_transforms.py:19-54): per-system max
relative difference <= 1e-10 for the solves, 1e-10 per line for the transforms
(1e-12 in the Dirichlet space)."""

import os

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import solvers as S
from paper_1701_03787_b200 import transforms as T
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import PointFamily, Space, build_mesh, channel_z2

pytestmark = pytest.mark.gpu

# SHEN_FUZZ_SEEDS=n widens both sweeps (a soak run; the default keeps the suite short)
_N = int(os.environ.get("SHEN_FUZZ_SEEDS", "0"))

FAMS = [PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO]
SPACES = [Space.CHEBYSHEV, Space.DIRICHLET, Space.BIHARMONIC]


def _solve_case(seed):
    rng = np.random.default_rng(1000 + seed)
    n_x = int(rng.choice([rng.integers(8, 40), rng.integers(40, 200), rng.integers(200, 700)]))  # assemble: n_x >= 8
    fam = int(rng.integers(0, 2))
    kind = int(rng.integers(0, 3))
    if kind == 0:  # a channel plane: mirror pairs, self-paired rows
        n_y, n_z = 2 * int(rng.integers(1, 24)), 2 * int(rng.integers(1, 40))
        z2 = channel_z2(n_y, n_z, float(rng.uniform(1, 8)), float(rng.uniform(1, 4)))
    elif kind == 1:  # an arbitrary flat batch (no pairs), odd length for complex RHS
        z2 = rng.uniform(0.0, 4e4, int(rng.integers(1, 3000)))
    else:  # a 2-D batch with repeated rows that are not a channel plane
        r, c = int(rng.integers(1, 9)), int(rng.integers(1, 130))
        z2 = np.repeat(rng.uniform(0.0, 1e4, (1, c)), r, axis=0) + (rng.integers(0, 2, (r, 1)) * 3.0)
    nu, dt = float(10 ** rng.uniform(-4, -2)), float(10 ** rng.uniform(-5, -2))
    cplx = bool(rng.integers(0, 2)) or (z2.size % 2 == 1)  # real RHS needs an even batch (16-B row pieces)
    return rng, n_x, fam, z2, nu, dt, cplx


@pytest.mark.parametrize("seed", range(_N or 24))
def test_random_solves_vs_oracle(seed):
    rng, n_x, fam, z2, nu, dt, cplx = _solve_case(seed)
    mats = assemble(n_x, fam)
    for build, fac, sol, nm in ((S.build_helmholtz, O.helmholtz_factor, O.helmholtz_solve, mats.n_dir),
                                (S.build_biharmonic, O.biharmonic_factor, O.biharmonic_solve, mats.n_bih)):
        shape = (nm,) + z2.shape
        f = rng.standard_normal(shape)
        if cplx:
            f = f + 1j * rng.standard_normal(shape)
        keep = f.copy()
        x = build(mats, nu, dt, z2).solve(f)
        assert np.array_equal(f, keep)  # the input is never mutated
        assert x.shape == shape and x.dtype == (np.complex128 if cplx else np.float64)
        want = sol(fac(mats, nu, dt, z2.reshape(-1)), f.reshape(nm, -1)).reshape(shape)
        err = O.max_rel_per_system(x.reshape(nm, -1), want.reshape(nm, -1)).max()
        assert err <= 1e-10, (seed, n_x, fam, z2.shape, cplx, build.__name__, err)


@pytest.mark.parametrize("seed", range(_N // 2 or 12))
def test_random_transforms_vs_oracle(seed):
    rng = np.random.default_rng(2000 + seed)
    n_x = 2 * int(rng.choice([rng.integers(4, 33), rng.integers(33, 130), rng.integers(130, 330)]))  # build_mesh: even
    fi = int(rng.integers(0, 2))
    n_y, n_z = 2 * int(rng.integers(1, 20)), 2 * int(rng.integers(1, 20))
    mesh = build_mesh(n_x, n_y, n_z, 2 * np.pi, np.pi, FAMS[fi])
    mats = assemble(n_x, fi)
    u = rng.uniform(-1, 1, mesh.shape)
    for sc, space in enumerate(SPACES):
        tol = 1e-10 if sc == 2 else 1e-12
        c = T.forward_transform(T.PhysicalField(u, mesh), space)
        want = O.forward_transform(u, sc, fi == 1, mats)
        scale = np.abs(want).max()
        assert np.abs(c.data - want).max() <= tol * scale, (seed, n_x, fi, n_y, n_z, sc, "forward")
        sp = T.forward_scalar_product(T.PhysicalField(u, mesh), space).data
        wsp = O.forward_scalar_product(u, sc, fi == 1)
        assert np.abs(sp - wsp).max() <= 1e-12 * np.abs(wsp).max(), (seed, n_x, fi, sc, "scalar product")
        back = T.inverse_transform(T.SpectralField(want, c.grid, mesh)).data
        wb = O.inverse_transform(want, sc, fi == 1, n_x, mesh.n_y, mesh.n_z)
        assert np.abs(back - wb).max() <= 1e-12 * np.abs(wb).max(), (seed, n_x, fi, sc, "inverse")


# ---------------------------------------------------------------- the stepper's callers
APPLY_NAMES = ("mass_dir", "mass_bih", "mixed_mass", "stiff_dir", "stiff_bih", "fourth_bih", "deriv_dir_to_bih",
               "deriv_bih_to_dir", "deriv_dir_to_cheb")


@pytest.mark.parametrize("seed", range(_N // 4 or 8))
def test_random_rhs_recover_apply_vs_oracle(seed):
    """RHS assembly and structured apply bit-identical, velocity recovery to
    1e-12, on random meshes (n_x even as build_mesh asks, line counts on both
    sides of the kernels' 4096-line switch)."""
    from paper_1701_03787_b200 import operators as P, recover as R, rhs as H
    from paper_1701_03787_b200.mesh import wavenumber_grid

    rng = np.random.default_rng(3000 + seed)
    n_x = 2 * int(rng.choice([rng.integers(4, 20), rng.integers(20, 100), rng.integers(100, 300)]))
    fi = int(rng.integers(0, 2))
    n_y, n_z = 2 * int(rng.integers(1, 40)), 2 * int(rng.integers(1, 60))
    mesh = build_mesh(n_x, n_y, n_z, float(rng.uniform(2, 14)), float(rng.uniform(1, 7)), FAMS[fi])
    grid = wavenumber_grid(mesh, Space.DIRICHLET)
    m, n, z2 = grid.m_scaled[:, None], grid.n_scaled[None, :], grid.z2()
    mats = assemble(n_x, fi)
    nu, dt = float(10 ** rng.uniform(-4, -2)), float(10 ** rng.uniform(-5, -2))
    shp_d, shp_b = (mats.n_dir,) + z2.shape, (mats.n_bih,) + z2.shape

    def c(shp):
        return rng.standard_normal(shp) + 1j * rng.standard_normal(shp)

    u, g = c(shp_b), c(shp_d)
    hc, hp = [c(shp_d) for _ in range(3)], [c(shp_d) for _ in range(3)]
    hab = O.ab2(hc, hp)
    asm = H.RhsAssembler(mats, nu, dt, z2, m, n)
    tag = (seed, n_x, fi, n_y, n_z)
    assert np.array_equal(asm.rhs_u(u, hc, hp), O.assemble_rhs_u(mats, nu, dt, z2, m, n, u, hab)), tag
    assert np.array_equal(asm.rhs_g(g, hc, hp), O.assemble_rhs_g(mats, nu, dt, z2, m, n, g, hab)), tag
    want_v, want_w = O.recover_velocity(mats, z2, m, n, u, g)
    v, w = R.VelocityRecovery(mats, z2, m, n)(u, g)
    assert np.abs(v - want_v).max() <= 1e-12 * np.abs(want_v).max(), tag
    assert np.abs(w - want_w).max() <= 1e-12 * np.abs(want_w).max(), tag
    name = APPLY_NAMES[seed % len(APPLY_NAMES)]
    M = getattr(mats, name)
    x = c((M.shape[1],) + z2.shape) if seed % 2 else rng.standard_normal((M.shape[1],) + z2.shape)
    assert np.array_equal(P.apply(M, x), M.apply(x)), tag + (name,)
