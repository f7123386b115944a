"""The drop-in accepts the reference's own ``MatrixSet``:
every host table the solvers, the structured apply and the RHS assembly read
from a matrix set must come out byte-identical whether the set is this
package's or ``chebchan.matrices.assemble``'s.  Needs the reference checkout
(/root/reference, this container only); the GPU box pins the same tables
through tests/golden (test_matrices.py)."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "chebchan")),
                                reason="reference checkout not present")

OPERATORS = ["stiff_dir", "mass_dir", "stiff_bih", "mass_bih", "fourth_bih"]


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import chebchan.matrices as rm
    import chebchan.mesh as rmesh
    return rm, rmesh


@pytest.mark.parametrize("n_x", [16, 63, 256])
@pytest.mark.parametrize("fam", ["gauss", "gauss_lobatto"])
def test_reference_matrixset_gives_the_same_tables(n_x, fam):
    rm, rmesh = _ref()
    from paper_1701_03787_b200 import matrices as M, mesh as me, operators as ops, solvers as S

    rfam = [f for f in rmesh.PointFamily if f.name.lower() == fam][0]
    ofam = [f for f in me.PointFamily if f.value == rfam.value][0]
    rmats, omats = rm.assemble(n_x, rfam), M.assemble(n_x, ofam)
    assert (rmats.n_x, rmats.n_dir, rmats.n_bih) == (omats.n_x, omats.n_dir, omats.n_bih)
    for a, b in zip(S._helm_tables(rmats), S._helm_tables(omats)):
        assert a.tobytes() == b.tobytes()
    for a, b in zip(S._bih_table(rmats), S._bih_table(omats)):
        assert np.asarray(a).tobytes() == np.asarray(b).tobytes()
    names = [n for n in dir(rmats) if not n.startswith("_") and hasattr(getattr(rmats, n), "shape")
             and hasattr(getattr(rmats, n), "apply")]
    assert set(OPERATORS) <= set(names)
    for name in names:
        kr, tr = ops.operator_tables(getattr(rmats, name))
        ko, to = ops.operator_tables(getattr(omats, name))
        assert kr == ko, name
        for a, b in zip(tr, to):
            if isinstance(a, np.ndarray):
                assert a.tobytes() == b.tobytes(), name
            else:
                assert a == b, name


def test_reference_matrixset_host_apply_matches():
    """The reference's structured apply and this package's agree bit for bit on
    the same input (the device kernel is pinned to the same goldens)."""
    rm, rmesh = _ref()
    from paper_1701_03787_b200 import matrices as M, mesh as me

    rng = np.random.default_rng(5)
    rfam = list(rmesh.PointFamily)[0]
    ofam = [f for f in me.PointFamily if f.value == rfam.value][0]
    rmats, omats = rm.assemble(48, rfam), M.assemble(48, ofam)
    for name in OPERATORS:
        r, o = getattr(rmats, name), getattr(omats, name)
        x = rng.standard_normal((r.shape[1], 3)) + 1j * rng.standard_normal((r.shape[1], 3))
        assert np.asarray(r.apply(x)).tobytes() == np.asarray(o.apply(x)).tobytes(), name
