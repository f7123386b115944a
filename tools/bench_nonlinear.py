"""Device-timed nonlinear term (nonlinear.py) at BASELINE config-3 size
(physical 257 x 256 x 256, n_x = 256) next to the oracle port (numpy/scipy,
reference arithmetic) of the same call on one core."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import shen_oracle as O  # noqa: E402
from paper_1701_03787_b200 import nonlinear as NL  # noqa: E402
from paper_1701_03787_b200.matrices import assemble  # noqa: E402
from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid  # noqa: E402

n_x, n_y, n_z = 256, 256, 256
mesh = build_mesh(n_x, n_y, n_z, 2 * np.pi, np.pi)
gd, gb = wavenumber_grid(mesh, Space.DIRICHLET), wavenumber_grid(mesh, Space.BIHARMONIC)
m, n = gd.m_scaled[:, None], gd.n_scaled[None, :]
mi = np.fft.fftfreq(n_y, 1.0 / n_y).astype(int)[:, None]
ni = np.arange(n_z // 2 + 1)[None, :]
mask = (np.abs(mi) != n_y // 2) & (ni != n_z // 2) & (np.abs(mi) < n_y // 3) & (ni < n_z // 3)
mats = assemble(n_x, 0)
rng = np.random.default_rng(0)


def c(grid):
    shp = (grid.n_modes,) + mesh.spectral_shape_yz
    return rng.standard_normal(shp) + 1j * rng.standard_normal(shp)


host = [c(gb), c(gd), c(gd), c(gd)]
dev = [torch.from_numpy(x).cuda() for x in host]
term = NL.NonlinearTerm(mats, mesh, m, n, mask)
for _ in range(3):
    term(*dev)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    term(*dev)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
t0 = time.perf_counter()
O.compute_nonlinear(mats, False, n_y, n_z, m, n, mask, *host)
cpu = time.perf_counter() - t0
# roofline: the call's compulsory HBM traffic is its 4 spectral inputs and 3
# spectral outputs (complex128); every transform stage in between is
# intermediate traffic the fused pipeline still pays
field = 16 * (n_x + 1) * n_y * (n_z // 2 + 1)
alg = 16 * sum(x.size for x in host) + 3 * 16 * gd.n_modes * n_y * (n_z // 2 + 1)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6548.2
print(json.dumps({"workload": "compute_nonlinear, config-3 mesh 257x256x256 (8 inverse + 3 forward transforms)",
                  "device_ms": ms, "cpu_oracle_s_1core": cpu, "speedup": cpu / (ms / 1e3),
                  "roofline": {"bound": "hbm", "algorithmic_bytes": alg, "achieved_GBps": alg / (ms * 1e6),
                               "peak_GBps": peak, "frac": alg / (ms * 1e6) / peak,
                               "note": "compulsory traffic only (4 fields in, 3 out)"}}))
