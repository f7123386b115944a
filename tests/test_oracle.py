"""Pin the CPU oracle against the reference's own outputs (golden fixtures):
bit-for-bit for the solver recurrences and transforms it restates."""

import hashlib

import numpy as np
import pytest

from oracle import shen_oracle as O
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import build_mesh, channel_z2


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", range(8))
def test_oracle_solvers_bitwise(golden, golden_meta, case):
    g = golden("solvers.npz")
    meta = golden_meta["solver_cases"][case]
    mats = assemble(meta["n_x"], meta["family"])
    z2 = g[f"c{case}_z2"]
    fh = O.helmholtz_factor(mats, meta["nu"], meta["dt"], z2)
    fb = O.biharmonic_factor(mats, meta["nu"], meta["dt"], z2)
    for nm in ("low", "d", "e", "tail"):
        for p in (0, 1):
            assert np.array_equal(fh[nm][p], g[f"c{case}_h_{nm}{p}"]), (nm, p)
    for nm in ("low2", "low4", "d", "e", "f", "a", "b"):
        for p in (0, 1):
            assert np.array_equal(fb[nm][p], g[f"c{case}_b_{nm}{p}"]), (nm, p)
    for kind in ("real", "cplx"):
        assert np.array_equal(O.helmholtz_solve(fh, g[f"c{case}_h_rhs_{kind}"]), g[f"c{case}_h_x_{kind}"])
        assert np.array_equal(O.biharmonic_solve(fb, g[f"c{case}_b_rhs_{kind}"]), g[f"c{case}_b_x_{kind}"])


def test_oracle_baseline_configs_sha(golden_meta):
    """BASELINE configs 1 and 2: the oracle reproduces the reference's full
    solution arrays exactly (sha256 of the bytes)."""
    mats = assemble(63, 0)
    z2 = channel_z2(64, 64)
    meta = golden_meta["baseline"]
    for op in ("h", "b"):
        nm = mats.n_dir if op == "h" else mats.n_bih
        rng = np.random.default_rng(0)
        f = rng.standard_normal((nm,) + z2.shape) + 1j * rng.standard_normal((nm,) + z2.shape)
        assert _sha(f) == meta[op]["rhs_sha256"]
        if op == "h":
            x = O.helmholtz_solve(O.helmholtz_factor(mats, 1e-3, 1e-3, z2), f)
        else:
            x = O.biharmonic_solve(O.biharmonic_factor(mats, 1e-3, 1e-3, z2), f)
        assert _sha(x) == meta[op]["x_sha256"], op


@pytest.mark.parametrize("n_x", [8, 16, 32])
@pytest.mark.parametrize("fi", [0, 1])
def test_oracle_transforms_bitwise(golden, n_x, fi):
    g = golden("transforms.npz")
    mesh = build_mesh(n_x, 8, 4, 2 * np.pi, np.pi, fi)
    mats = assemble(n_x, fi)
    key = f"nx{n_x}_f{fi}"
    u = g[key + "_u"]
    for sc in (0, 1, 2):
        c = O.forward_transform(u, sc, fi == 1, mats)
        assert np.array_equal(c, g[f"{key}_s{sc}_fwd"]), sc
        assert np.array_equal(O.forward_scalar_product(u, sc, fi == 1), g[f"{key}_s{sc}_fsp"])
        back = O.inverse_transform(c, sc, fi == 1, n_x, mesh.n_y, mesh.n_z)
        assert np.array_equal(back, g[f"{key}_s{sc}_inv"]), sc


@pytest.mark.parametrize("fi", [0, 1])
def test_oracle_1d_blocks_bitwise(golden, fi):
    g = golden("transforms.npz")
    v = g[f"blk_f{fi}_v"]
    mats = assemble(12, fi)
    assert np.array_equal(O.chebyshev_scalar(v, fi == 1), g[f"blk_f{fi}_cheb_scalar"])
    assert np.array_equal(O.chebyshev_evaluate(v, fi == 1), g[f"blk_f{fi}_cheb_eval"])
    for sc, drop in ((1, 2), (2, 4)):
        assert np.array_equal(O.shen_scalar(v, fi == 1, sc), g[f"blk_f{fi}_s{sc}_shen_scalar"])
        w = v[:13 - drop]
        assert np.array_equal(O.shen_expand(w, sc, 12), g[f"blk_f{fi}_s{sc}_expand"])
        assert np.array_equal(O.mass_solve(w, sc, mats), g[f"blk_f{fi}_s{sc}_mass"])


def test_oracle_dense_recovery():
    """Known-answer style check (reference tests/test_solvers.py:30-59): the
    restated elimination matches a pivoted dense solve."""
    mats = assemble(32, 0)
    z2 = np.array([0.0, 100.0, 40000.0])
    nu, dt = 1 / 5200, 1e-5
    rng = np.random.default_rng(3)
    rhs = rng.standard_normal((mats.n_bih, 3))
    x = O.biharmonic_solve(O.biharmonic_factor(mats, nu, dt, z2), rhs)
    for i in range(3):
        want = np.linalg.solve(O.dense_biharmonic(mats, nu, dt, z2[i]), rhs[:, i])
        assert np.abs(x[:, i] - want).max() / np.abs(want).max() < 1e-10


def degenerate_mats(n_x, zero_rows):
    """MatrixSet whose Dirichlet mass diagonal vanishes on ``zero_rows``:
    with nu = 0 the Helmholtz pivot of those rows is exactly 0."""
    import dataclasses

    from paper_1701_03787_b200.matrices import BandedMatrix

    m = assemble(n_x, 0)
    d0 = m.mass_dir.diagonal(0).copy()
    d0[list(zero_rows)] = 0.0
    md = BandedMatrix(m.mass_dir.shape, m.mass_dir.offsets,
                      tuple(d0 if off == 0 else dg for off, dg in zip(m.mass_dir.offsets, m.mass_dir.diagonals)))
    return dataclasses.replace(m, mass_dir=md)


@pytest.mark.parametrize("rows,want", [([0], 0), ([1], 1), ([0, 1], 0)])
def test_oracle_pivot_error(rows, want):
    mats = degenerate_mats(16, rows)
    with pytest.raises(O.OraclePivotError, match=f"at row {want}$"):
        O.helmholtz_factor(mats, 0.0, 1.0, np.array([0.0, 1.0]))


@pytest.mark.parametrize("fi", [0, 1])
def test_oracle_rhs_assembly_bitwise(golden, fi):
    """stepper.py:189-219 restated: AB2 and both right-hand sides equal the
    reference's ChannelStepper outputs bit for bit."""
    g = golden("rhs.npz")
    k = f"f{fi}"
    mats = assemble(16, fi)
    hc = [g[f"{k}_hc{i}"] for i in range(3)]
    hp = [g[f"{k}_hp{i}"] for i in range(3)]
    hab = O.ab2(hc, hp)
    for i in range(3):
        assert np.array_equal(hab[i], g[f"{k}_hab{i}"])
    args = (mats, 1e-2, 1e-3, g[k + "_z2"], g[k + "_m"], g[k + "_n"])
    assert np.array_equal(O.assemble_rhs_u(*args, g[k + "_u"], hab), g[k + "_rhs_u"])
    assert np.array_equal(O.assemble_rhs_g(*args, g[k + "_g"], hab), g[k + "_rhs_g"])


@pytest.mark.parametrize("fi", [0, 1])
def test_oracle_nonlinear_and_recovery_bitwise(golden, fi):
    """stepper.py:148-185 (compute_nonlinear) and :296-303 (velocity
    recovery) restated: equal to the reference's outputs bit for bit."""
    g = golden("rhs.npz")
    k = f"f{fi}"
    mats = assemble(16, fi)
    nl = O.compute_nonlinear(mats, fi == 1, 8, 8, g[k + "_m"], g[k + "_n"], g[k + "_mask"], g[k + "_u"],
                             g[k + "_v"], g[k + "_w"], g[k + "_g"])
    for i in range(3):
        assert np.array_equal(nl[i], g[f"{k}_nl{i}"])
    v, w = O.recover_velocity(mats, g[k + "_z2"], g[k + "_m"], g[k + "_n"], g[k + "_u"], g[k + "_g"])
    assert np.array_equal(v, g[k + "_vrec"]) and np.array_equal(w, g[k + "_wrec"])


@pytest.mark.parametrize("n_x", [512, 1024])
@pytest.mark.parametrize("fi", [0, 1])
def test_oracle_big_transforms_bitwise(golden, n_x, fi):
    """The oracle's 3-D transforms at n_x = 512 / 1024 (where the biharmonic
    forward map is most ill-conditioned) reproduce the reference's bytes."""
    g = golden("big_transforms.npz")
    mats = assemble(n_x, fi)
    key = f"nx{n_x}_f{fi}"
    u = g[key + "_u"]
    for sc in (1, 2):
        c = O.forward_transform(u, sc, fi == 1, mats)
        assert np.array_equal(c, g[f"{key}_s{sc}_fwd"])
        assert np.array_equal(O.inverse_transform(c, sc, fi == 1, n_x, 4, 2), g[f"{key}_s{sc}_inv"])
