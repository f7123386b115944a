"""Column-resident solves (csrc/shen_solve_cr.cu, method="cr"): parity with
the reference on its golden cases and with the oracle on awkward shapes
(batch not a multiple of the 8-system tile, scalar z2, real RHS, system
subranges as the host pipeline uses them)."""

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import solvers as S
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import channel_z2

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.mark.parametrize("case", range(8))
def test_cr_reference_cases(golden, golden_meta, case):
    g = golden("solvers.npz")
    meta = golden_meta["solver_cases"][case]
    mats = assemble(meta["n_x"], meta["family"])
    z2 = g[f"c{case}_z2"]
    lu = S.build_helmholtz(mats, meta["nu"], meta["dt"], z2, method="cr")
    for kind in ("cplx", "real"):
        x = lu.solve(g[f"c{case}_h_rhs_{kind}"])
        want = g[f"c{case}_h_x_{kind}"]
        assert x.dtype == want.dtype and x.shape == want.shape
        assert O.max_rel_per_system(x, want).max() <= TOL


@pytest.mark.parametrize("n_x,shape", [(16, (13,)), (64, ()), (255, (3, 7)), (1024, (9, 5)), (128, (512, 3))])
def test_cr_shapes(n_x, shape):
    mats = assemble(n_x, 0)
    rng = np.random.default_rng(n_x)
    z2 = rng.uniform(0, 5e5, shape)
    lu = S.build_helmholtz(mats, 1 / 2000, 1e-4, z2, method="cr")
    f = rng.standard_normal((mats.n_dir,) + shape) + 1j * rng.standard_normal((mats.n_dir,) + shape)
    x = lu.solve(f)
    ref = O.helmholtz_solve(O.helmholtz_factor(mats, 1 / 2000, 1e-4, np.atleast_1d(z2).reshape(-1)),
                            f.reshape(mats.n_dir, -1)).reshape(f.shape)
    assert O.max_rel_per_system(x, ref).max() <= TOL


def test_cr_subranges_equal_full():
    """Slabs [j0, j1) (the host pipeline's unit) give the same bits as one solve."""
    import torch

    mats = assemble(256, 0)
    z2 = channel_z2(64, 126)
    lu = S.build_helmholtz(mats, 1e-3, 1e-3, z2, method="cr")
    B = z2.size
    g = torch.Generator(device="cuda").manual_seed(3)
    f = torch.randn((mats.n_dir, B), dtype=torch.complex128, device="cuda", generator=g)
    full = torch.empty_like(f)
    lu.solve_into(f, full, True)
    part = torch.zeros_like(f)
    for a, b in ((0, 1001), (1001, 1005), (1005, B)):
        lu.solve_into(f, part, True, a, b)
    assert torch.equal(part, full)


def test_cr_host_pipeline():
    mats = assemble(64, 0)
    z2 = channel_z2(96, 190)
    lu = S.build_helmholtz(mats, 1e-3, 1e-3, z2, method="cr")
    rng = np.random.default_rng(1)
    f = rng.standard_normal((mats.n_dir,) + z2.shape) + 1j * rng.standard_normal((mats.n_dir,) + z2.shape)
    x = lu.solve(f)
    ref = O.helmholtz_solve(O.helmholtz_factor(mats, 1e-3, 1e-3, z2), f)
    assert O.max_rel_per_system(x, ref).max() <= TOL
