"""A whole reference time step composed of the device pieces
(stepper.DeviceStepper) against the reference's ChannelStepper.step on the
same state (golden), both forcings.  Pieces round differently from
pocketfft/LAPACK: gate 1e-11 of each field's max."""

import numpy as np
import pytest

from paper_1701_03787_b200.checkpoint import FlowState
from paper_1701_03787_b200.mesh import PointFamily, Space, build_mesh, wavenumber_grid
from paper_1701_03787_b200.stepper import DeviceStepper
from paper_1701_03787_b200.transforms import SpectralField

pytestmark = pytest.mark.gpu
TOL = 1e-11


class _Cfg:
    def __init__(self, forcing, beta=0.0, target_flux=0.0):
        self.nu, self.dt, self.forcing, self.beta, self.target_flux, self.dealias = 1e-2, 1e-3, forcing, beta, \
            target_flux, True


def _close(got, want):
    got = got.cpu().numpy()
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err <= TOL, err


@pytest.mark.parametrize("fi", [0, 1])
@pytest.mark.parametrize("tag", ["fb", "cf"])
def test_step_vs_reference_golden(golden, fi, tag):
    g = golden("rhs.npz")
    k = f"f{fi}"
    mesh = build_mesh(16, 8, 8, 2 * np.pi, np.pi, (PointFamily.GAUSS, PointFamily.GAUSS_LOBATTO)[fi])
    gd, gb = wavenumber_grid(mesh, Space.DIRICHLET), wavenumber_grid(mesh, Space.BIHARMONIC)
    cfg = _Cfg("fixed-beta", beta=0.5) if tag == "fb" else _Cfg("constant-flux", target_flux=0.3)
    stp = DeviceStepper(mesh, cfg)

    def sf(x, grid):
        return SpectralField(x, grid, mesh)

    state = FlowState(sf(g[k + "_u"], gb), sf(g[k + "_v"], gd), sf(g[k + "_w"], gd), sf(g[k + "_g"], gd),
                      tuple(sf(g[f"{k}_hc{i}"], gd) for i in range(3)), tuple(sf(g[f"{k}_hp{i}"], gd) for i in range(3)),
                      0.25, 1.5, 7)
    new = stp.step(stp.to_device(state))
    for nm in ("u_hat", "v_hat", "w_hat", "g_hat"):
        _close(getattr(new, nm).data, g[f"{k}_{tag}_{nm}"])
    for i in range(3):
        _close(new.h_curr[i].data, g[f"{k}_{tag}_hcur{i}"])
    want_beta = float(g[f"{k}_{tag}_beta"])
    assert abs(new.beta - want_beta) <= 1e-9 * max(1.0, abs(want_beta))
    assert (new.t, new.kappa) == (1.5 + 1e-3, 8)


def test_captured_step_matches_eager_steps(golden):
    """DeviceStepper.capture: three graph replays equal three eager steps."""
    import torch

    g = golden("rhs.npz")
    mesh = build_mesh(16, 8, 8, 2 * np.pi, np.pi, PointFamily.GAUSS)
    gd, gb = wavenumber_grid(mesh, Space.DIRICHLET), wavenumber_grid(mesh, Space.BIHARMONIC)
    stp = DeviceStepper(mesh, _Cfg("fixed-beta", beta=0.5))

    def fresh():
        def sf(x, grid):
            return SpectralField(x, grid, mesh)

        st = FlowState(sf(g["f0_u"], gb), sf(g["f0_v"], gd), sf(g["f0_w"], gd), sf(g["f0_g"], gd),
                       tuple(sf(g[f"f0_hc{i}"], gd) for i in range(3)), tuple(sf(g[f"f0_hp{i}"], gd) for i in range(3)),
                       0.25, 1.5, 7)
        return stp.to_device(st)

    eager = fresh()
    for _ in range(3):
        eager = stp.step(eager)
    state = fresh()
    replay = stp.capture(state)
    for _ in range(3):
        replay()
    torch.cuda.synchronize()
    for nm in ("u_hat", "v_hat", "w_hat", "g_hat"):
        assert torch.equal(getattr(state, nm).data, getattr(eager, nm).data), nm
    for i in range(3):
        assert torch.equal(state.h_curr[i].data, eager.h_curr[i].data)
        assert torch.equal(state.h_prev[i].data, eager.h_prev[i].data)
    assert state.kappa == eager.kappa == 10
