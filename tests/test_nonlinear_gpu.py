"""Device nonlinear term (nonlinear.py) against the reference's
ChannelStepper.compute_nonlinear (golden) and the oracle restatement.
Rounding differs from pocketfft/LAPACK: gate 1e-12 of each field's max."""

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import nonlinear as NL
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import PointFamily, Space, build_mesh, wavenumber_grid

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _close(got, want):
    got = got.cpu().numpy() if hasattr(got, "cpu") else got
    assert got.shape == want.shape and got.dtype == want.dtype
    err = np.abs(got - want).max() / max(np.abs(want).max(), 1e-300)
    assert err <= TOL, err


@pytest.mark.parametrize("fi", [0, 1])
def test_nonlinear_vs_reference_golden(golden, fi):
    g = golden("rhs.npz")
    k = f"f{fi}"
    mesh = build_mesh(16, 8, 8, 2 * np.pi, np.pi, (PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO)[fi])
    term = NL.NonlinearTerm(assemble(16, fi), mesh, g[k + "_m"], g[k + "_n"], g[k + "_mask"])
    out = term(g[k + "_u"], g[k + "_v"], g[k + "_w"], g[k + "_g"])
    for i in range(3):
        _close(out[i], g[f"{k}_nl{i}"])


@pytest.mark.parametrize("n_x,n_y,n_z", [(64, 16, 12), (128, 32, 32), (16, 256, 256)])
@pytest.mark.parametrize("fi", [0, 1])
def test_nonlinear_vs_oracle_larger(n_x, n_y, n_z, fi):
    import torch

    mesh = build_mesh(n_x, n_y, n_z, 2 * np.pi, np.pi, (PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO)[fi])
    gd, gb = wavenumber_grid(mesh, Space.DIRICHLET), wavenumber_grid(mesh, Space.BIHARMONIC)
    m, n = gd.m_scaled[:, None], gd.n_scaled[None, :]
    mi = np.fft.fftfreq(n_y, 1.0 / n_y).astype(int)[:, None]
    ni = np.arange(n_z // 2 + 1)[None, :]
    mask = (np.abs(mi) != n_y // 2) & (ni != n_z // 2) & (np.abs(mi) < max(n_y // 3, 1)) & (ni < max(n_z // 3, 1))
    mats = assemble(n_x, fi)
    rng = np.random.default_rng(n_x)

    def c(grid):
        shp = (grid.n_modes,) + mesh.spectral_shape_yz
        return rng.standard_normal(shp) + 1j * rng.standard_normal(shp)

    u, v, w, gg = c(gb), c(gd), c(gd), c(gd)
    want = O.compute_nonlinear(mats, fi == 1, n_y, n_z, m, n, mask, u, v, w, gg)
    term = NL.NonlinearTerm(mats, mesh, m, n, mask)
    got = term(u, v, w, gg)
    for i in range(3):
        _close(got[i], want[i])
    gt = term(*(torch.from_numpy(x).cuda() for x in (u, v, w, gg)))
    assert gt[0].is_cuda
    _close(gt[2], want[2])
