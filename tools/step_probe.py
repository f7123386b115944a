"""Per-step device times of DeviceStepper on the config-3 mesh from a random
spectral state, with the state's magnitude (does the evolving state slow the
step down?)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200.checkpoint import FlowState  # noqa: E402
from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid  # noqa: E402
from paper_1701_03787_b200.stepper import DeviceStepper  # noqa: E402
from paper_1701_03787_b200.transforms import SpectralField  # noqa: E402


class Cfg:
    nu, dt, forcing, beta, target_flux, dealias = 1 / 2000, 1e-4, "fixed-beta", 0.01, 0.0, True


mesh = build_mesh(256, 256, 256, 2 * np.pi, np.pi)
stp = DeviceStepper(mesh, Cfg)
gd, gb = wavenumber_grid(mesh, Space.DIRICHLET), wavenumber_grid(mesh, Space.BIHARMONIC)
gen = torch.Generator(device="cuda").manual_seed(7)
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0


def field(grid):
    shp = (grid.n_modes,) + mesh.spectral_shape_yz
    return SpectralField(scale * torch.randn(shp, dtype=torch.complex128, device="cuda", generator=gen), grid, mesh)


s = FlowState(field(gb), field(gd), field(gd), field(gd), tuple(field(gd) for _ in range(3)),
              tuple(field(gd) for _ in range(3)), 0.01, 0.0, 0)
for i in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s = stp.step(s)
    e1.record()
    torch.cuda.synchronize()
    u = s.u_hat.data
    print(i, round(e0.elapsed_time(e1), 2), "ms  max|u|", float(u.abs().max()), "finite", bool(torch.isfinite(u).all()))

# CUDA-graph replay of the same step (state advanced in place)
st = stp.to_device(s) if False else s
replay = stp.capture(st)
for _ in range(3):
    replay()
torch.cuda.synchronize()
for rep in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        replay()
    e1.record()
    torch.cuda.synchronize()
    print("graph", round(e0.elapsed_time(e1) / 10, 3), "ms/step", "finite", bool(torch.isfinite(st.u_hat.data).all()))
