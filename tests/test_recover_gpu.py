"""Device velocity recovery (recover.py) against the reference's
stepper.py:296-303 (golden, computed with the reference's own functions)
and the oracle at larger sizes.  LAPACK's banded Cholesky solve rounds
differently: gate 1e-12 of each field's max."""

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import recover as R
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _close(got, want):
    got = got.cpu().numpy() if hasattr(got, "cpu") else got
    assert got.shape == want.shape and got.dtype == want.dtype
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err <= TOL, err


@pytest.mark.parametrize("fi", [0, 1])
def test_recover_vs_reference_golden(golden, fi):
    g = golden("rhs.npz")
    k = f"f{fi}"
    rec = R.VelocityRecovery(assemble(16, fi), g[k + "_z2"], g[k + "_m"], g[k + "_n"])
    v, w = rec(g[k + "_u"], g[k + "_g"])
    _close(v, g[k + "_vrec"])
    _close(w, g[k + "_wrec"])


@pytest.mark.parametrize("n_x", [64, 256])
@pytest.mark.parametrize("fi", [0, 1])
def test_recover_vs_oracle_larger(n_x, fi):
    import torch

    from paper_1701_03787_b200.mesh import PointFamily

    mesh = build_mesh(n_x, 24, 16, 2 * np.pi, np.pi, (PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO)[fi])
    gd = wavenumber_grid(mesh, Space.DIRICHLET)
    m, n, z2 = gd.m_scaled[:, None], gd.n_scaled[None, :], gd.z2()
    mats = assemble(n_x, fi)
    rng = np.random.default_rng(n_x)
    u = rng.standard_normal((mats.n_bih,) + z2.shape) + 1j * rng.standard_normal((mats.n_bih,) + z2.shape)
    gg = rng.standard_normal((mats.n_dir,) + z2.shape) + 1j * rng.standard_normal((mats.n_dir,) + z2.shape)
    want = O.recover_velocity(mats, z2, m, n, u, gg)
    rec = R.VelocityRecovery(mats, z2, m, n)
    v, w = rec(u, gg)
    _close(v, want[0])
    _close(w, want[1])
    vt, wt = rec(torch.from_numpy(u).cuda(), torch.from_numpy(gg).cuda())
    assert vt.is_cuda
    _close(wt, want[1])
    with pytest.raises(ValueError):
        rec(u[:-1], gg)
