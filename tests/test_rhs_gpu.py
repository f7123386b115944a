"""Fused right-hand-side assembly (rhs.py / csrc/shen_rhs.cu) against the
reference's ChannelStepper (golden) and the oracle: bit-identical."""

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import rhs as H
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fi", [0, 1])
def test_rhs_vs_reference_golden(golden, fi):
    g = golden("rhs.npz")
    k = f"f{fi}"
    mats = assemble(16, fi)
    hc = [g[f"{k}_hc{i}"] for i in range(3)]
    hp = [g[f"{k}_hp{i}"] for i in range(3)]
    asm = H.RhsAssembler(mats, 1e-2, 1e-3, g[k + "_z2"], g[k + "_m"], g[k + "_n"])
    ru = asm.rhs_u(g[k + "_u"], hc, hp)
    rg = asm.rhs_g(g[k + "_g"], hc, hp)
    assert ru.dtype == np.complex128 and ru.shape == g[k + "_rhs_u"].shape
    assert np.array_equal(ru, g[k + "_rhs_u"])
    assert np.array_equal(rg, g[k + "_rhs_g"])


@pytest.mark.parametrize("n_x", [64, 256])
@pytest.mark.parametrize("fi", [0, 1])
def test_rhs_vs_oracle_larger(n_x, fi):
    import torch

    from paper_1701_03787_b200.mesh import PointFamily

    mesh = build_mesh(n_x, 16, 12, 2 * np.pi, np.pi, (PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO)[fi])
    grid = wavenumber_grid(mesh, Space.DIRICHLET)
    m, n, z2 = grid.m_scaled[:, None], grid.n_scaled[None, :], grid.z2()
    mats = assemble(n_x, fi)
    rng = np.random.default_rng(n_x)
    shp_d, shp_b = (mats.n_dir,) + z2.shape, (mats.n_bih,) + z2.shape

    def c(shp):
        return rng.standard_normal(shp) + 1j * rng.standard_normal(shp)

    u, g = c(shp_b), c(shp_d)
    hc = [c(shp_d) for _ in range(3)]
    hp = [c(shp_d) for _ in range(3)]
    hab = O.ab2(hc, hp)
    nu, dt = 1 / 2000, 1e-4
    asm = H.RhsAssembler(mats, nu, dt, z2, m, n)
    assert np.array_equal(asm.rhs_u(u, hc, hp), O.assemble_rhs_u(mats, nu, dt, z2, m, n, u, hab))
    assert np.array_equal(asm.rhs_g(g, hc, hp), O.assemble_rhs_g(mats, nu, dt, z2, m, n, g, hab))
    # torch in -> torch out, on the device
    td = asm.rhs_g(torch.from_numpy(g).cuda(), [torch.from_numpy(h).cuda() for h in hc],
                   [torch.from_numpy(h).cuda() for h in hp])
    assert td.is_cuda and np.array_equal(td.cpu().numpy(), O.assemble_rhs_g(mats, nu, dt, z2, m, n, g, hab))
    with pytest.raises(ValueError):
        asm.rhs_g(g[:-1], hc, hp)
