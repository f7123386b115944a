"""Host-side checks of the wall-normal transform operators (no GPU):
the 80-bit-built matrices reproduce the reference's 1-D pipeline
(chebyshev_scalar -> shen_scalar -> mass_solve, shen_expand ->
chebyshev_evaluate; transforms.py:81-175) and are at least as accurate."""

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import transforms as T
from paper_1701_03787_b200.matrices import assemble


@pytest.mark.parametrize("n_x", [8, 16, 64])
@pytest.mark.parametrize("fam", [0, 1])
@pytest.mark.parametrize("sp", [0, 1, 2])
def test_operators_match_reference_pipeline(n_x, fam, sp):
    mats = assemble(n_x, fam)
    rng = np.random.default_rng(n_x + 3 * fam + sp)
    X = rng.standard_normal((n_x + 1, 7)) + 1j * rng.standard_normal((n_x + 1, 7))
    fsp = O.shen_scalar(X, fam == 1, sp)
    fwd = O.mass_solve(fsp, sp, mats) if sp else fsp
    for kind, want in (("fsp", fsp), ("fwd", fwd)):
        got = T._operator_host(kind, n_x, fam, sp) @ X
        assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max(), kind
    inv = O.chebyshev_evaluate(O.shen_expand(fwd, sp, n_x), fam == 1)
    got = T._operator_host("inv", n_x, fam, sp) @ fwd
    assert np.abs(got - inv).max() <= 1e-13 * np.abs(inv).max()


@pytest.mark.parametrize("fam", [0, 1])
def test_biharmonic_forward_operator_accuracy_n256(fam):
    """At config 3's n_x = 256 the biharmonic forward map is ill-conditioned:
    the reference's own result is ~2e-11 from an 80-bit evaluation, the
    operator ~2e-15.  Both stay inside BASELINE.json's 1e-10."""
    n_x = 256
    mats = assemble(n_x, fam)
    X = np.random.default_rng(1).standard_normal((n_x + 1, 16))
    N = n_x + 1
    exact = T._banded_solve_ld(mats.mass_bih.dense(), T._stencil_ld(2, N, fam) @ T._scalar_matrix_ld(N, fam))
    exact = exact @ X.astype(np.longdouble)
    scale = float(np.abs(exact).max())
    ref = O.mass_solve(O.shen_scalar(X, fam == 1, 2), 2, mats)
    mine = T._operator_host("fwd", n_x, fam, 2) @ X
    err_ref = float(np.abs(ref - exact).max()) / scale
    err_mine = float(np.abs(mine - exact).max()) / scale
    assert err_mine < 1e-14
    assert err_mine < err_ref
    assert np.abs(mine - ref).max() / np.abs(ref).max() < 1e-10
