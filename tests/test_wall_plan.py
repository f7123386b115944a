"""Host side of the fused wall-normal transform (paper_1701_03787_b200/wall.py):
the plan tables (digit reversal, Rader maps, convolution kernels, chirps)
drive a numpy model of the kernel's pass sequence that must reproduce the
oracle's transforms (reference transforms.py:81-205) -- no GPU needed."""

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200 import wall as W
from paper_1701_03787_b200.matrices import assemble


@pytest.mark.parametrize("M", [2, 4, 8, 16, 32, 64, 256, 512, 1024])
def test_dif_passes_digit_reversed(M):
    rad = W.stages_for(M)
    assert int(np.prod(rad)) == M and max(rad) <= 16
    x = np.random.default_rng(M).standard_normal((M, 3)) + 1j
    got = W.emulate_dft(x, rad)
    want = np.fft.fft(x, axis=0)[W.digit_reversal(rad)]
    assert np.allclose(got, want, rtol=0, atol=1e-12 * np.abs(want).max())


@pytest.mark.parametrize("n_x,kind", [(256, W.KIND_RADER), (16, W.KIND_RADER), (8, W.KIND_BLUESTEIN),
                                      (64, W.KIND_BLUESTEIN), (1024, W.KIND_BLUESTEIN)])
def test_gauss_kinds(n_x, kind):
    assert W.plan_tables(n_x, 0)["kind"] == kind
    assert W.plan_tables(n_x, 1)["kind"] == W.KIND_POW2 if n_x & (n_x - 1) == 0 else True


@pytest.mark.parametrize("n_x", [8, 16, 32, 64, 256, 12])
@pytest.mark.parametrize("fi", [0, 1])
@pytest.mark.parametrize("sc", [0, 1, 2])
def test_model_matches_oracle(n_x, fi, sc):
    rng = np.random.default_rng(n_x * 7 + fi)
    N = n_x + 1
    x = rng.standard_normal((N, 5)) + 1j * rng.standard_normal((N, 5))
    mats = assemble(n_x, fi)
    scale = np.pi / (2 * N) if fi == 0 else np.pi / (2 * n_x)
    got = W.emulate_wall(x, n_x, fi, sc, 0, True, scale)
    scal = O.shen_scalar(x, fi == 1, sc)
    want = O.mass_solve(scal, sc, mats) if sc else scal
    assert O.max_rel_per_system(got, want).max() < 1e-12
    got_s = W.emulate_wall(x, n_x, fi, sc, 0, False, scale)
    assert O.max_rel_per_system(got_s, scal).max() < 1e-12
    # inverse of the space's coefficients (no 1/(ny nz) here)
    c = want
    inv = W.emulate_wall(c, n_x, fi, sc, 1, False, 1.0)
    want_i = O.chebyshev_evaluate(O.shen_expand(c, sc, n_x), fi == 1)
    assert np.abs(inv - want_i).max() < 1e-12 * np.abs(want_i).max()
