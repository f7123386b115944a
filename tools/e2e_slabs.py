"""e2e (host buffers, pipelined copies) at config-4 sample size for several
slab counts of the host pipeline (solvers._PIPE_MAX_SLABS)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import solvers as S  # noqa: E402
from paper_1701_03787_b200.matrices import assemble  # noqa: E402
from paper_1701_03787_b200.mesh import channel_z2  # noqa: E402

mats = assemble(1024, 0)
z2 = np.ascontiguousarray(channel_z2(2048, 2048)[:256])
hlu = S.build_helmholtz(mats, 1 / 2000, 1e-4, z2)
blu = S.build_biharmonic(mats, 1 / 2000, 1e-4, z2)


def pinned(shape):
    return torch.empty(shape, dtype=torch.complex128, pin_memory=True).numpy()


shp_h, shp_b = (mats.n_dir,) + z2.shape, (mats.n_bih,) + z2.shape
fh, fb, xh, xb = pinned(shp_h), pinned(shp_b), pinned(shp_h), pinned(shp_b)
fh[...] = 1.0
fb[...] = 1.0
jobs = [(hlu, fh, xh), (blu, fb, xb)]
unk = (mats.n_dir + mats.n_bih) * z2.size
for slabs in (8, 16, 24, 32, 48, 64):
    S._PIPE_MAX_SLABS = slabs
    for _ in range(2):
        S.solve_many(jobs)
    t0 = time.perf_counter()
    for _ in range(3):
        S.solve_many(jobs)
    dt = (time.perf_counter() - t0) / 3
    print(f"slabs {slabs:3d}: e2e {unk / dt:.3e} unknowns/s ({dt * 1e3:.1f} ms)", flush=True)
