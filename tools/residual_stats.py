"""Residual of the fast-mode streaming solves vs the reference's own, over
many config-4 systems (largest z^2 corner + random), 80-bit dense products."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import shen_oracle as O  # noqa: E402
from paper_1701_03787_b200 import solvers as S  # noqa: E402
from paper_1701_03787_b200.matrices import assemble  # noqa: E402
from paper_1701_03787_b200.mesh import channel_z2  # noqa: E402

nsys = int(sys.argv[1]) if len(sys.argv) > 1 else 48
mats = assemble(1024, 0)
full = channel_z2(2048, 2048).reshape(-1)
rng = np.random.default_rng(7)
idx = np.unique(np.concatenate([np.argsort(full)[-nsys // 2:], rng.choice(full.size, nsys // 2, replace=False)]))
z2 = full[idx]
nu, dt = 1 / 2000, 1e-4
for op in ("h", "b"):
    build = S.build_helmholtz if op == "h" else S.build_biharmonic
    nm = mats.n_dir if op == "h" else mats.n_bih
    f = rng.standard_normal((nm, z2.size)) + 1j * rng.standard_normal((nm, z2.size))
    x = build(mats, nu, dt, z2).solve(f)
    if op == "h":
        ref = O.helmholtz_solve(O.helmholtz_factor(mats, nu, dt, z2), f)
        dense = lambda z: O.dense_helmholtz(mats, nu, dt, z)  # noqa: E731
    else:
        ref = O.biharmonic_solve(O.biharmonic_factor(mats, nu, dt, z2), f)
        dense = lambda z: O.dense_biharmonic(mats, nu, dt, z)  # noqa: E731
    r_ours, r_ref = [], []
    for j in range(z2.size):
        M = dense(z2[j])
        r_ours.append(float(O.residual_longdouble(M, x[:, j], f[:, j])))
        r_ref.append(float(O.residual_longdouble(M, ref[:, j], f[:, j])))
    r_ours, r_ref = np.array(r_ours), np.array(r_ref)
    ratio = r_ours / r_ref
    print(op, "ours max %.2e  ref max %.2e  ratio median %.2f  max %.2f  >1e-12: ours %d ref %d" % (
        r_ours.max(), r_ref.max(), np.median(ratio), ratio.max(), (r_ours > 1e-12).sum(), (r_ref > 1e-12).sum()))
