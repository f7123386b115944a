"""Chunk-split Helmholtz on mirror pairs (SHEN_HELM_SPLIT=1) vs the streaming
kernel and the oracle: parity on channel grids (self-pairs, partial groups),
then config-4 timing of both kernels alternated in one process."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import shen_oracle as O  # noqa: E402
from paper_1701_03787_b200 import solvers as S  # noqa: E402
from paper_1701_03787_b200.matrices import assemble  # noqa: E402
from paper_1701_03787_b200.mesh import channel_z2  # noqa: E402

nu, dt = 1 / 2000, 1e-4
S.PAIRS_MIN = 1
for n_x, ny, nz in ((256, 16, 30), (512, 8, 62), (1024, 8, 64), (128, 40, 20), (64, 6, 10)):
    mats = assemble(n_x, 0)
    z2 = channel_z2(ny, nz)
    rng = np.random.default_rng(n_x)
    f = rng.standard_normal((mats.n_dir,) + z2.shape) + 1j * rng.standard_normal((mats.n_dir,) + z2.shape)
    lu = S.build_helmholtz(mats, nu, dt, z2)
    assert lu._pairs is not None
    S.HELM_SPLIT = 0
    xs = lu.solve(f)
    S.HELM_SPLIT = 1
    xp = lu.solve(f)
    want = O.helmholtz_solve(O.helmholtz_factor(mats, nu, dt, z2.reshape(-1)), f.reshape(mats.n_dir, -1))
    e_split = O.max_rel_per_system(xp.reshape(mats.n_dir, -1), want).max()
    e_stream = O.max_rel_per_system(xs.reshape(mats.n_dir, -1), want).max()
    zf = z2.reshape(-1)
    res = []
    for jj in np.linspace(0, zf.size - 1, 6).astype(int):
        m = O.dense_helmholtz(mats, nu, dt, zf[jj])
        res.append((float(O.residual_longdouble(m, xp.reshape(mats.n_dir, -1)[:, jj], f.reshape(mats.n_dir, -1)[:, jj])),
                    float(O.residual_longdouble(m, want[:, jj], f.reshape(mats.n_dir, -1)[:, jj]))))
    print(f"n_x={n_x}: split max rel {e_split:.2e} (stream {e_stream:.2e}); residual split/ref max "
          f"{max(r[0] for r in res):.2e}/{max(r[1] for r in res):.2e}", flush=True)

mats = assemble(1024, 0)
z2 = channel_z2(2048, 2048)
S.PAIRS_MIN = 8192
lu = S.build_helmholtz(mats, nu, dt, z2)
B = z2.size
g = torch.Generator(device="cuda").manual_seed(1)
rhs = torch.complex(torch.randn((mats.n_dir, B), generator=g, device="cuda", dtype=torch.float64),
                    torch.randn((mats.n_dir, B), generator=g, device="cuda", dtype=torch.float64))
out = torch.empty_like(rhs)
ref = torch.empty_like(rhs)
for flag in (0, 1, 0, 1):
    S.HELM_SPLIT = flag
    for _ in range(2):
        lu.solve_into(rhs, out if flag else ref, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        lu.solve_into(rhs, out if flag else ref, True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"config 4 helmholtz {'split ' if flag else 'stream'}: {ms:.3f} ms", flush=True)
d = max(float(((out[:, k:k + 65536] - ref[:, k:k + 65536]).abs().amax(dim=0) / ref[:, k:k + 65536].abs().amax(dim=0)).max())
        for k in range(0, B, 65536))
print(f"config 4 split vs stream: max rel per system {d:.2e}")
