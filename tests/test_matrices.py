"""Host setup tables: the product's assemble() must equal the reference's
MatrixSet bit for bit (golden tables from tests/golden/make_golden.py), and
the structured operators must agree with dense/quadrature forms (reference
tests/test_matrices.py strategy)."""

import numpy as np
import pytest

from paper_1701_03787_b200.matrices import assemble, dense_oracle, tail_factors
from paper_1701_03787_b200.mesh import PointFamily, Space


@pytest.mark.parametrize("n_x", [8, 16, 63, 64, 256])
@pytest.mark.parametrize("fi", [0, 1])
def test_assemble_bitwise_equals_reference(golden, n_x, fi):
    g = golden("matrices.npz")
    m = assemble(n_x, fi)
    key = f"nx{n_x}_f{fi}"
    assert np.array_equal(m.mass_cheb, g[key + "_mass_cheb"])
    for name in ("mass_dir", "mass_bih", "mixed_mass", "stiff_bih", "deriv_dir_to_bih", "deriv_bih_to_dir"):
        mat = getattr(m, name)
        for off, dg in zip(mat.offsets, mat.diagonals):
            assert np.array_equal(dg, g[f"{key}_{name}_{off}"]), (name, off)
    for name in ("stiff_dir", "deriv_dir_to_cheb"):
        mat = getattr(m, name)
        for off, dg in zip(mat.banded.offsets, mat.banded.diagonals):
            assert np.array_equal(dg, g[f"{key}_{name}_{off}"]), (name, off)
        assert np.array_equal(mat.tail, g[f"{key}_{name}_tail"])
    assert np.array_equal(m.fourth_bih.diag, g[key + "_fourth_bih_diag"])


def test_family_accepts_enum_and_code():
    assert assemble(16, PointFamily.GAUSS) is assemble(16, 0)
    assert assemble(16, PointFamily.GAUSS_LOBATTO) is assemble(16, 1)


def test_rank2_tail_identity():
    # reference known answer (SPEC: a_0 = p_0 = 0, r_0 = 48 pi)
    p, q, r, s = tail_factors(10)
    assert p[0] == 0.0
    assert np.isclose(r[0], 48 * np.pi)


@pytest.mark.parametrize("fam", [0, 1])
def test_structured_apply_matches_dense(fam):
    m = assemble(16, fam)
    rng = np.random.default_rng(5)
    for mat in (m.mass_dir, m.mass_bih, m.stiff_dir, m.stiff_bih, m.fourth_bih, m.deriv_dir_to_cheb):
        x = rng.standard_normal((mat.shape[1], 3))
        assert np.allclose(mat.apply(x), mat.dense() @ x, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("fam", [0, 1])
def test_closed_forms_vs_quadrature_oracle(fam):
    n_x = 16
    m = assemble(n_x, fam)
    cases = [(m.mass_dir, Space.DIRICHLET, Space.DIRICHLET, 0, 1),
             (m.mass_bih, Space.BIHARMONIC, Space.BIHARMONIC, 0, 1),
             (m.stiff_dir, Space.DIRICHLET, Space.DIRICHLET, 2, -1),
             (m.stiff_bih, Space.BIHARMONIC, Space.BIHARMONIC, 2, -1),
             (m.fourth_bih, Space.BIHARMONIC, Space.BIHARMONIC, 4, 1)]
    for mat, rs, cs, order, sign in cases:
        want = sign * dense_oracle(rs, cs, order, n_x, fam)
        scale = max(np.abs(want).max(), 1.0)
        assert np.abs(mat.dense() - want).max() / scale < 1e-11


def test_fourth_diag_positive():
    # the code's exact-quadrature Q~ diagonal is +8 pi (k+1)^2 (k+2)(k+4)
    m = assemble(32, 0)
    k = np.arange(m.n_bih)
    assert np.all(m.fourth_bih.diag > 0)
    assert np.allclose(m.fourth_bih.diag, 8 * np.pi * (k + 1) ** 2 * (k + 2) * (k + 4), rtol=1e-13)


def test_assemble_rejects_small():
    with pytest.raises(ValueError):
        assemble(7, 0)


@pytest.mark.parametrize("n_x", [16, 33])
@pytest.mark.parametrize("fam", [0, 1])
def test_host_apply_vs_reference_golden(golden, n_x, fam):
    """The host restatement of matrices.py apply (used by the oracle and the
    residual checks) is bit-identical to the reference's."""
    g = golden("apply.npz")
    mats = assemble(n_x, fam)
    for name in ("mass_dir", "mass_bih", "mixed_mass", "stiff_dir", "stiff_bih", "fourth_bih", "deriv_dir_to_bih",
                 "deriv_bih_to_dir", "deriv_dir_to_cheb"):
        x = g[f"nx{n_x}_f{fam}_{name}_x"]
        assert np.array_equal(getattr(mats, name).apply(x), g[f"nx{n_x}_f{fam}_{name}_y"]), name


@pytest.mark.parametrize("n_x", [1024, 2048])
@pytest.mark.parametrize("fi", [0, 1])
def test_assemble_headline_sizes_sha(n_x, fi):
    """assemble() at the headline sizes (config 4 n_x = 1024, config 5's
    largest N = 2049): every table equals the reference's byte for byte
    (sha256 pinned by tests/golden/make_golden.py big_fixture)."""
    import hashlib
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "big_tables.json")) as fh:
        want = json.load(fh)

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    m = assemble(n_x, fi)
    key = f"nx{n_x}_f{fi}"
    got = {key + "_mass_cheb": sha(m.mass_cheb), key + "_fourth_bih_diag": sha(m.fourth_bih.diag)}
    for name in ("mass_dir", "mass_bih", "mixed_mass", "stiff_bih", "deriv_dir_to_bih", "deriv_bih_to_dir"):
        mat = getattr(m, name)
        for off, dg in zip(mat.offsets, mat.diagonals):
            got[f"{key}_{name}_{off}"] = sha(dg)
    for name in ("stiff_dir", "deriv_dir_to_cheb"):
        mat = getattr(m, name)
        for off, dg in zip(mat.banded.offsets, mat.banded.diagonals):
            got[f"{key}_{name}_{off}"] = sha(dg)
        got[f"{key}_{name}_tail"] = sha(mat.tail)
    ref = {k: v for k, v in want.items() if k.startswith(key + "_")}
    assert got == ref
