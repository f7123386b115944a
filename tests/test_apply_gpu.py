"""Device structured apply (operators.py / csrc/shen_apply.cu) against the
reference's matrices.py apply: bit-identical for every matrix of the set,
real and complex, 1-D and batched, both point families."""

import numpy as np
import pytest

from paper_1701_03787_b200 import operators as P
from paper_1701_03787_b200.matrices import assemble

pytestmark = pytest.mark.gpu

NAMES = ("mass_dir", "mass_bih", "mixed_mass", "stiff_dir", "stiff_bih", "fourth_bih", "deriv_dir_to_bih",
         "deriv_bih_to_dir", "deriv_dir_to_cheb")


@pytest.mark.parametrize("n_x", [8, 33, 256])
@pytest.mark.parametrize("fam", [0, 1])
def test_apply_bitwise(n_x, fam):
    mats = assemble(n_x, fam)
    rng = np.random.default_rng(n_x + fam)
    for name in NAMES:
        M = getattr(mats, name)
        nc = M.shape[1]
        for x in (rng.standard_normal((nc, 5, 3)) + 1j * rng.standard_normal((nc, 5, 3)),
                  rng.standard_normal((nc, 7)), rng.standard_normal(nc)):
            want = M.apply(x)
            got = P.apply(M, x)
            assert got.dtype == want.dtype and got.shape == want.shape, name
            assert np.array_equal(got, want), name


def test_apply_torch_and_errors():
    import torch

    mats = assemble(16, 0)
    x = torch.randn(mats.n_dir, 4, dtype=torch.complex128, device="cuda")
    y = P.apply(mats.stiff_dir, x)
    assert y.is_cuda and np.array_equal(y.cpu().numpy(), mats.stiff_dir.apply(x.cpu().numpy()))
    with pytest.raises(ValueError):
        P.apply(mats.mass_dir, np.zeros((mats.n_dir + 1, 2)))


@pytest.mark.parametrize("n_x", [16, 33])
@pytest.mark.parametrize("fam", [0, 1])
def test_apply_vs_reference_golden(golden, n_x, fam):
    """Pinned to the reference's own apply outputs (tests/golden/apply.npz)."""
    g = golden("apply.npz")
    mats = assemble(n_x, fam)
    for name in NAMES:
        x = g[f"nx{n_x}_f{fam}_{name}_x"]
        assert np.array_equal(P.apply(getattr(mats, name), x), g[f"nx{n_x}_f{fam}_{name}_y"]), name


@pytest.mark.parametrize("n_x,L", [(256, 1), (256, 9), (1024, 1), (1024, 3), (64, 4096), (256, 5000)])
def test_apply_bitwise_line_counts(n_x, L):
    """Both kernels: the staged one (few lines, x and tables in shared memory;
    lines per block shrink with n_x) and the per-line one (>= 4096 lines)."""
    mats = assemble(n_x, 0)
    rng = np.random.default_rng(L)
    for name in NAMES:
        M = getattr(mats, name)
        nc = M.shape[1]
        for x in (rng.standard_normal((nc, L)) + 1j * rng.standard_normal((nc, L)), rng.standard_normal((nc, L))):
            assert np.array_equal(P.apply(M, x), M.apply(x)), (name, x.dtype)
