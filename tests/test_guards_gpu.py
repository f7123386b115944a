"""Out-of-bounds and coverage checks of the device kernels (stand-in for
compute-sanitizer, which is closed on this GPU pool).

Every input and output array is placed inside a larger allocation whose
guard bands hold NaN (inputs) or a sentinel bit pattern (outputs):
* a write outside the output leaves a guard band changed;
* a read outside the input pulls a NaN into the results;
* an output element the kernel never writes keeps the NaN it was filled
  with.
Sizes are picked to leave partial warps, partial 32-item groups, partial
mirror-pair groups and partial line tiles, with both real and complex
right-hand sides."""

import numpy as np
import pytest
import torch

from oracle import shen_oracle as O
from paper_1701_03787_b200 import solvers as S, transforms as T
from paper_1701_03787_b200.matrices import assemble
from paper_1701_03787_b200.mesh import channel_z2

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements of guard band on each side
SENT = -7.7e300


def _guarded(shape, dtype, fill):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), fill, dtype=dtype, device="cuda")
    return buf, buf[GUARD:GUARD + n].view(shape)


def _guards_ok(buf, fill):
    a, b = buf[:GUARD], buf[-GUARD:]
    if buf.is_complex():
        return bool(((a == fill).all() and (b == fill).all()).item())
    return bool(((a == fill).all() and (b == fill).all()).item())


@pytest.mark.parametrize("op", ["h", "b"])
@pytest.mark.parametrize("cplx", [True, False])
@pytest.mark.parametrize("n_x,ny,nz,pairs", [(63, 16, 16, False), (40, 18, 58, True), (129, 34, 66, True),
                                             (20, 3, 14, False)])
def test_solve_guards(op, cplx, n_x, ny, nz, pairs):
    mats = assemble(n_x, 0)
    z2 = channel_z2(ny, nz)
    saved = S.PAIRS_MIN
    S.PAIRS_MIN = 1 if pairs else 10 ** 12
    try:
        lu = (S.build_helmholtz if op == "h" else S.build_biharmonic)(mats, 1 / 2000, 1e-4, z2)
    finally:
        S.PAIRS_MIN = saved
    if op == "b":
        assert (lu._pairs is not None) == pairs
    nm, B = lu.n_modes, z2.size
    dt = torch.complex128 if cplx else torch.float64
    rng = np.random.default_rng(n_x + ny)
    f = rng.standard_normal((nm, B)) + (1j * rng.standard_normal((nm, B)) if cplx else 0)
    ibuf, rhs = _guarded((nm, B), dt, float("nan"))
    rhs.copy_(torch.from_numpy(f))
    obuf, out = _guarded((nm, B), dt, SENT)
    out.fill_(float("nan"))
    lu.solve_into(rhs, out, cplx)
    torch.cuda.synchronize()
    assert _guards_ok(obuf, SENT), "write outside the output"
    x = out.cpu().numpy()
    assert np.isfinite(x).all(), "unwritten output or out-of-bounds read"
    fac, sol = ((O.helmholtz_factor, O.helmholtz_solve) if op == "h" else (O.biharmonic_factor, O.biharmonic_solve))
    assert O.max_rel_per_system(x, sol(fac(mats, 1 / 2000, 1e-4, z2.reshape(-1)), f)).max() <= 1e-10


def _wall(plan, L, xin, rows_out):
    import ctypes

    from paper_1701_03787_b200 import _lib
    from paper_1701_03787_b200._device import stream_handle

    obuf, out = _guarded((rows_out, L), torch.complex128, complex(SENT, SENT))
    out.fill_(complex(float("nan"), float("nan")))
    _lib.check(_lib.lib().shen_wall_transform(ctypes.byref(plan.struct), L, xin.data_ptr(), out.data_ptr(),
                                              stream_handle()), "shen_wall_transform")
    torch.cuda.synchronize()
    assert _guards_ok(obuf, complex(SENT, SENT)), "write outside the output"
    bad = ~torch.isfinite(torch.view_as_real(out)).all(dim=-1)
    if bad.any():
        r, c = torch.nonzero(bad, as_tuple=True)
        raise AssertionError(f"unwritten output or out-of-bounds read: {int(bad.sum())} values, rows "
                             f"{sorted(set(r.tolist()))[:8]}, lines {sorted(set(c.tolist()))[:8]}")
    return out


@pytest.mark.parametrize("fi", [0, 1])
@pytest.mark.parametrize("sp", [0, 1, 2])
@pytest.mark.parametrize("n_x,L", [(16, 37), (256, 1000), (24, 3), (63, 17), (100, 50), (127, 40), (300, 33)])
def test_wall_transform_guards(fi, sp, n_x, L):
    """The fused wall-normal kernels (TMA boxes clipped at the array edges,
    partial line tiles) forward with the mass solve and inverse."""
    from paper_1701_03787_b200.transforms import _cheb_scale
    from paper_1701_03787_b200.wall import wall_plan

    N = n_x + 1
    n = {0: N, 1: n_x - 1, 2: n_x - 3}[sp]
    rng = np.random.default_rng(n_x + L)
    x = rng.standard_normal((N, L)) + 1j * rng.standard_normal((N, L))
    nanc = complex(float("nan"), float("nan"))
    _, xin = _guarded((N, L), torch.complex128, nanc)
    xin.copy_(torch.from_numpy(x))
    fwd = wall_plan(n_x, fi, sp, 0, True, _cheb_scale(N, fi))
    assert fwd is not None
    c = _wall(fwd, L, xin, n).cpu().numpy()
    mats = assemble(n_x, fi)
    want = O.mass_solve(O.shen_scalar(x, fi == 1, sp), sp, mats) if sp else O.shen_scalar(x, fi == 1, 0)
    assert np.abs(c - want).max() <= 1e-10 * np.abs(want).max()
    _, cin = _guarded((n, L), torch.complex128, nanc)
    cin.copy_(torch.from_numpy(want))
    inv = wall_plan(n_x, fi, sp, 1, False, 1.0)
    back = _wall(inv, L, cin, N).cpu().numpy()
    wantb = O.chebyshev_evaluate(O.shen_expand(want, sp, n_x), fi == 1)
    assert np.abs(back - wantb).max() <= 1e-12 * np.abs(wantb).max()
