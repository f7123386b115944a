"""Drop-in for ``chebchan.transforms`` (reference ``transforms.py``) on B200.

Same names, signatures, shapes and dtypes as the reference:

* ``chebyshev_scalar(values, family)``          transforms.py:81-86
* ``shen_scalar(values, family, space)``         transforms.py:89-110
* ``shen_expand(coeffs, space, n_x)``            transforms.py:113-126
* ``chebyshev_evaluate(coeffs, family)``         transforms.py:129-137
* ``mass_solve(scalar, space, n_x, family)``     transforms.py:163-175
* ``forward_transform(field, space)``            transforms.py:181-188
* ``forward_scalar_product(field, space)``       transforms.py:191-196
* ``inverse_transform(coeffs)``                  transforms.py:199-205
* ``PhysicalField`` / ``SpectralField``          transforms.py:40-75

Device pipeline.  Everything runs on the GPU with axis 0
(the wall-normal direction) as the row index and the Fourier lines as the
contiguous lane index:

* periodic y/z: ``torch.fft.rfft2`` / ``irfft2`` (cuFFT, library);
* wall-normal DCT: our ``shen_xform_extend`` / ``shen_xform_inv_pre`` kernels
  build the extended sequence, cuFFT does one FFT along the rows, our
  ``shen_xform_fwd_post`` / ``shen_xform_inv_post`` kernels apply the twiddle,
  the Chebyshev scaling and the Shen stencil in the same pass;
* mass solve: our ``shen_xform_mass_solve`` kernel, one thread per
  (line, parity), with the host's LAPACK banded Cholesky factors of the 1-D
  mass matrix (the very factors the reference computes,
  transforms.py:143-160).

numpy inputs are copied to the device and the result copied back (numpy out);
torch CUDA tensors stay on the device (torch out).  There is no CPU fallback:
without the library or a GPU every call raises ``ShenBackendError``.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from ._device import device, is_torch, stream_handle
from .matrices import assemble
from .mesh import Mesh, WavenumberGrid, as_family, as_space, family_code, space_code, wavenumber_grid

__all__ = [
    "PhysicalField",
    "SpectralField",
    "chebyshev_scalar",
    "shen_scalar",
    "shen_expand",
    "chebyshev_evaluate",
    "mass_solve",
    "mass_cholesky",
    "forward_transform",
    "forward_scalar_product",
    "inverse_transform",
    "wall_forward",
    "wall_inverse",
]

_RAW = 3  # fwd_post "space" code for the plain chebyshev_scalar products


# ---------------------------------------------------------------- containers

@dataclass
class PhysicalField:
    """Real samples of a scalar on the collocation mesh (transforms.py:40-49).
    ``data`` is a numpy array or a torch tensor (CUDA tensors stay on device)."""

    data: object
    mesh: Mesh

    def __post_init__(self):
        if tuple(self.data.shape) != tuple(self.mesh.shape):
            raise ValueError(
                f"field shape {tuple(self.data.shape)} does not match mesh {tuple(self.mesh.shape)}")


@dataclass
class SpectralField:
    """Complex expansion coefficients on a wavenumber grid (transforms.py:52-75)."""

    data: object
    grid: WavenumberGrid
    mesh: Mesh

    def __post_init__(self):
        expected = (self.grid.n_modes,) + tuple(self.mesh.spectral_shape_yz)
        if tuple(self.data.shape) != expected:
            raise ValueError(f"coefficient shape {tuple(self.data.shape)}, expected {expected}")

    def copy(self) -> "SpectralField":
        d = self.data.clone() if is_torch(self.data) else self.data.copy()
        return SpectralField(d, self.grid, self.mesh)

    def zeros_like(self) -> "SpectralField":
        if is_torch(self.data):
            import torch

            return SpectralField(torch.zeros_like(self.data), self.grid, self.mesh)
        return SpectralField(np.zeros_like(self.data), self.grid, self.mesh)


# ---------------------------------------------------------------- plumbing

class _Lines:
    """An axis-0 array as a contiguous complex128 (rows, L) device tensor,
    remembering how to hand the result back in the caller's type."""

    def __init__(self, values):
        import torch

        self.from_numpy = not is_torch(values)
        if self.from_numpy:
            a = np.asarray(values)
            self.is_complex = np.iscomplexobj(a)
            self.trailing = a.shape[1:]
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128 if self.is_complex else np.float64))
            if t.numel() > 0:
                t = t.pin_memory()
            t = t.to(device(), non_blocking=True)
        else:
            self.is_complex = values.is_complex()
            self.trailing = tuple(values.shape[1:])
            t = values.to(device=device(), dtype=torch.complex128 if self.is_complex else torch.float64)
        if t.dim() == 0:
            raise ValueError("expected at least one axis (axis 0 = wall-normal)")
        if not self.is_complex:
            t = t.to(torch.complex128)
        self.rows = t.shape[0]
        self.L = int(np.prod(self.trailing, dtype=np.int64)) if self.trailing else 1
        self.t = t.contiguous().reshape(self.rows, self.L)

    def give_back(self, out, keep_complex=None):
        """out: (rows', L) complex128 device tensor -> caller's type/shape."""
        cplx = self.is_complex if keep_complex is None else keep_complex
        res = out.reshape((out.shape[0],) + tuple(self.trailing))
        if not cplx:
            res = res.real.contiguous()
        if self.from_numpy:
            return res.cpu().numpy()
        return res


@lru_cache(maxsize=32)
def _twiddles_cached(N: int, dev_index: int):
    import torch

    k = np.arange(N, dtype=np.float64)
    ang = -np.pi * k / (2 * N)
    tw = np.cos(ang) + 1j * np.sin(ang)
    return torch.from_numpy(tw.astype(np.complex128)).to(torch.device("cuda", dev_index))


def _twiddles(N):
    return _twiddles_cached(int(N), device().index)


def _fam(family) -> int:
    return family_code(family)  # 0 = Gauss, 1 = Gauss-Lobatto


def _wall_run(plan, x, rows_out):
    """shen_wall_transform of (rows_in, L) complex128 lines -> (rows_out, L)."""
    import ctypes

    import torch

    L = x.shape[1]
    out = torch.empty((rows_out, L), dtype=torch.complex128, device=x.device)
    _lib.check(_lib.lib().shen_wall_transform(ctypes.byref(plan.struct), L, x.data_ptr(), out.data_ptr(),
                                              stream_handle()), "shen_wall_transform")
    return out


def _cheb_scale(N: int, fam: int) -> float:
    return np.pi / (2 * N) if fam == 0 else np.pi / (2 * (N - 1))  # transforms.py:84-86


def _chebyshev_pass(x, fam: int, space: int):
    """x: (N, L) complex128 device -> fwd_post output (n_modes(space), L)."""
    import torch

    N, L = x.shape
    if N < 2:
        raise ValueError("need at least 2 points along axis 0")
    if XFORM_METHOD == "wall" and N >= 3:
        from .wall import wall_plan

        plan = wall_plan(N - 1, fam, space, 0, False, _cheb_scale(N, fam))
        if plan is not None:
            return _wall_run(plan, x.contiguous(), plan.struct.n_out)
    M = 2 * N if fam == 0 else 2 * N - 2
    e = torch.empty((M, L), dtype=torch.complex128, device=x.device)
    lib = _lib.lib()
    st = stream_handle()
    _lib.check(lib.shen_xform_extend(fam, N, L, x.data_ptr(), e.data_ptr(), st), "shen_xform_extend")
    Y = torch.fft.fft(e, dim=0).contiguous()  # cuFFT may hand back permuted strides
    del e
    n_x = N - 1
    rows = {0: N, 1: n_x - 1, 2: n_x - 3, _RAW: N}[space]
    out = torch.empty((rows, L), dtype=torch.complex128, device=x.device)
    scale = np.pi / (2 * N) if fam == 0 else np.pi / (2 * (N - 1))
    tw = _twiddles(N)
    _lib.check(lib.shen_xform_fwd_post(fam, space, N, L, float(scale), tw.data_ptr(), Y.data_ptr(),
                                       out.data_ptr(), st), "shen_xform_fwd_post")
    return out


def _expand_pass(c, space: int, n_x: int, fam: int):
    """c: (n, L) coefficients of `space` -> fam 0/1: point values (n_x+1, L);
    fam 2: expanded Chebyshev coefficients (n_x+1, L)."""
    import torch

    n, L = c.shape
    N = n_x + 1
    if fam != 2 and XFORM_METHOD == "wall" and N >= 3:
        from .wall import wall_plan

        plan = wall_plan(n_x, fam, space, 1, False, 1.0)
        if plan is not None and plan.struct.n_in == n:
            return _wall_run(plan, c.contiguous(), N)
    lib = _lib.lib()
    st = stream_handle()
    tw = _twiddles(N)
    if fam == 2:
        out = torch.empty((N, L), dtype=torch.complex128, device=c.device)
        _lib.check(lib.shen_xform_inv_pre(2, space, n, N, L, tw.data_ptr(), c.data_ptr(), out.data_ptr(), None, st),
                   "shen_xform_inv_pre")
        return out
    M = 2 * N if fam == 0 else 2 * N - 2
    Z = torch.empty((M, L), dtype=torch.complex128, device=c.device)
    ends = torch.empty((2, L), dtype=torch.complex128, device=c.device)
    _lib.check(lib.shen_xform_inv_pre(fam, space, n, N, L, tw.data_ptr(), c.data_ptr(), Z.data_ptr(),
                                      ends.data_ptr(), st), "shen_xform_inv_pre")
    F = (torch.fft.ifft(Z, dim=0, norm="forward") if fam == 0 else torch.fft.fft(Z, dim=0)).contiguous()
    del Z
    out = torch.empty((N, L), dtype=torch.complex128, device=c.device)
    _lib.check(lib.shen_xform_inv_post(fam, N, L, F.data_ptr(), ends.data_ptr(), out.data_ptr(), st),
               "shen_xform_inv_post")
    return out


def _check_expand_rows(n, space, n_x):
    extra = {0: 0, 1: 2, 2: 4}[space]
    if n + extra > n_x + 1 or n < 1:
        raise ValueError(f"{n} coefficients of space {as_space(space).name} do not fit n_x = {n_x}")


# ---------------------------------------------------------------- 1-D blocks

def chebyshev_scalar(values, family):
    """Weighted scalar products (f, T_k), k = 0..n_x (transforms.py:81-86)."""
    ln = _Lines(values)
    return ln.give_back(_chebyshev_pass(ln.t, _fam(family), _RAW))


def shen_scalar(values, family, space):
    """Scalar products against the basis of ``space`` (transforms.py:89-110);
    for the Chebyshev space the interpolation coefficients."""
    sp = space_code(space)
    ln = _Lines(values)
    n_x = ln.rows - 1
    if (sp == 1 and n_x < 2) or (sp == 2 and n_x < 4):
        raise ValueError(f"n_x = {n_x} too small for space {as_space(sp).name}")
    return ln.give_back(_chebyshev_pass(ln.t, _fam(family), sp))


def shen_expand(coeffs, space, n_x: int):
    """Basis coefficients of ``space`` -> plain Chebyshev ones (transforms.py:113-126)."""
    sp = space_code(space)
    ln = _Lines(coeffs)
    _check_expand_rows(ln.rows, sp, int(n_x))
    return ln.give_back(_expand_pass(ln.t, sp, int(n_x), 2))


def chebyshev_evaluate(coeffs, family):
    """Evaluate a Chebyshev series on the collocation points (transforms.py:129-137)."""
    ln = _Lines(coeffs)
    n_x = ln.rows - 1
    if n_x < 1:
        raise ValueError("need at least 2 Chebyshev coefficients")
    return ln.give_back(_expand_pass(ln.t, 0, n_x, _fam(family)))


@lru_cache(maxsize=16)
def _mass_factors_host(n_x: int, fam: int, sp: int):
    """Per-parity upper banded Cholesky factors (transforms.py:143-160), packed
    as [2][nband+1][mmax] float64 (LAPACK upper band storage, zero padded)."""
    from scipy.linalg import cholesky_banded

    mats = assemble(n_x, as_family(fam))
    full, nband = (mats.mass_dir, 1) if sp == 1 else (mats.mass_bih, 2)
    dense = full.dense()
    n = dense.shape[0]
    mmax = (n + 1) // 2
    packed = np.zeros((2, nband + 1, mmax))
    facs = []
    for par in (0, 1):
        sub = dense[par::2, par::2]
        m = sub.shape[0]
        ab = np.zeros((nband + 1, m))
        for b in range(nband + 1):
            ab[nband - b, b:] = np.diag(sub, b)
        f = cholesky_banded(ab, lower=False)
        facs.append(f)
        packed[par, :, :m] = f
    return packed, nband, n, mmax, tuple(facs)


def mass_cholesky(n_x: int, family, space):
    """The per-parity factors as the reference's ``_mass_cholesky`` returns them."""
    sp = space_code(space)
    if sp == 0:
        raise ValueError("Chebyshev mass solve is a rescale; see shen_scalar")
    return _mass_factors_host(int(n_x), _fam(family), sp)[4]


@lru_cache(maxsize=16)
def _mass_factors_dev(n_x: int, fam: int, sp: int, dev_index: int):
    import torch

    packed, nband, n, mmax, _ = _mass_factors_host(n_x, fam, sp)
    return torch.from_numpy(np.ascontiguousarray(packed)).to(torch.device("cuda", dev_index)), nband, n, mmax


def _mass_pass(s, sp: int, n_x: int, fam: int, out=None):
    fac, nband, n, mmax = _mass_factors_dev(n_x, fam, sp, device().index)
    if s.shape[0] != n:
        raise ValueError(f"mass_solve: {s.shape[0]} rows, expected {n} for space {as_space(sp).name}, n_x = {n_x}")
    x = s if out is None else out
    _lib.check(_lib.lib().shen_xform_mass_solve(nband, n, mmax, s.shape[1], fac.data_ptr(), s.data_ptr(),
                                                x.data_ptr(), stream_handle()), "shen_xform_mass_solve")
    return x


def mass_solve(scalar, space, n_x: int, family):
    """Solve B y = scalar products along axis 0 (transforms.py:163-175)."""
    sp = space_code(space)
    if sp == 0:
        raise ValueError("Chebyshev mass solve is a rescale; see shen_scalar")
    ln = _Lines(scalar)
    import torch

    out = torch.empty_like(ln.t)
    return ln.give_back(_mass_pass(ln.t, sp, int(n_x), _fam(family), out=out))


# ---------------------------------------------------------------- wall-normal operators
#
# For the 3-D transforms the whole wall-normal map is one linear operator per
# (n_x, family, space): forward = B^-1 S W (Chebyshev scalar products W, Shen
# stencil S, mass solve B^-1), scalar product = S W, inverse = C X (Shen ->
# Chebyshev expansion X, evaluation at the points C).  At N = 257 (config 3)
# the FFT route needs a Bluestein FFT (N prime) and several HBM passes; one
# fp64 GEMM over all Fourier lines (cuBLAS) is about 4x faster, reads the
# spectrum once and writes the result once.  The operators are built once in
# 80-bit arithmetic and rounded to float64.  SHEN_XFORM=fft selects the
# kernel/cuFFT pipeline above instead (used by the 1-D building blocks).

XFORM_METHOD = __import__("os").environ.get("SHEN_XFORM", "wall")


def _ld_pi():
    return np.arccos(np.longdouble(-1))


def _scalar_matrix_ld(N: int, fam: int):
    """W (N x N): chebyshev_scalar as a matrix (transforms.py:81-86)."""
    pi = _ld_pi()
    k = np.arange(N, dtype=np.longdouble)[:, None]
    n = np.arange(N, dtype=np.longdouble)[None, :]
    if fam == 0:
        return (pi / N) * np.cos(pi * k * (2 * n + 1) / (2 * N))
    nx = N - 1
    W = (pi / nx) * np.cos(pi * k * n / nx)
    W[:, 0] *= 0.5
    W[:, nx] *= 0.5
    return W


def _stencil_ld(sp: int, N: int, fam: int):
    """S (n x N): shen_scalar applied to the Chebyshev scalar products (transforms.py:89-110)."""
    n_x = N - 1
    if sp == 0:
        S = np.eye(N, dtype=np.longdouble) * (2 / _ld_pi())
        S[0, 0] /= 2
        if fam == 1:
            S[n_x, n_x] /= 2
        return S
    if sp == 1:
        n = n_x - 1
        S = np.zeros((n, N), dtype=np.longdouble)
        r = np.arange(n)
        S[r, r] = 1
        S[r, r + 2] = -1
        return S
    n = n_x - 3
    S = np.zeros((n, N), dtype=np.longdouble)
    r = np.arange(n)
    k = r.astype(np.longdouble)
    S[r, r] = 1
    S[r, r + 2] = -2 * (k + 2) / (k + 3)
    S[r, r + 4] = (k + 1) / (k + 3)
    return S


def _banded_solve_ld(Bd, R):
    """Solve B Y = R in long double (B banded SPD, no pivoting needed)."""
    A = Bd.astype(np.longdouble).copy()
    Y = R.copy()
    n = A.shape[0]
    bw = 4
    for i in range(n):
        hi = min(n, i + bw + 1)
        for r in range(i + 1, hi):
            if A[r, i] != 0:
                f = A[r, i] / A[i, i]
                A[r, i:hi] -= f * A[i, i:hi]
                Y[r] -= f * Y[i]
    for i in range(n - 1, -1, -1):
        hi = min(n, i + bw + 1)
        Y[i] = (Y[i] - A[i, i + 1:hi] @ Y[i + 1:hi]) / A[i, i]
    return Y


@lru_cache(maxsize=16)
def _operator_host(kind: str, n_x: int, fam: int, sp: int):
    N = n_x + 1
    if kind in ("fwd", "fsp"):
        M = _stencil_ld(sp, N, fam) @ _scalar_matrix_ld(N, fam)
        if kind == "fwd" and sp != 0:
            mats = assemble(n_x, as_family(fam))
            Bd = (mats.mass_dir if sp == 1 else mats.mass_bih).dense()
            M = _banded_solve_ld(Bd, M)
        return np.ascontiguousarray(M.astype(np.float64))
    # inverse: C (N x N) evaluation at the points times the expansion X (N x n)
    pi = _ld_pi()
    j = np.arange(N, dtype=np.longdouble)[:, None]
    m = np.arange(N, dtype=np.longdouble)[None, :]
    theta = pi * (2 * j + 1) / (2 * N) if fam == 0 else pi * j / n_x
    C = np.cos(m * theta)
    n = N - (0, 2, 4)[sp]
    X = np.zeros((N, n), dtype=np.longdouble)
    c = np.arange(n)
    k = c.astype(np.longdouble)
    X[c, c] = 1
    if sp == 1:
        X[c + 2, c] = -1
    elif sp == 2:
        X[c + 2, c] = -2 * (k + 2) / (k + 3)
        X[c + 4, c] = (k + 1) / (k + 3)
    return np.ascontiguousarray((C @ X).astype(np.float64))


@lru_cache(maxsize=16)
def _operator_dev(kind: str, n_x: int, fam: int, sp: int, dev_index: int, scale: float = 1.0):
    """Device copy; ``scale`` folds a constant factor into the operator (the
    inverse folds irfft2's 1/(n_y n_z) so no separate scaling pass runs)."""
    import torch

    M = _operator_host(kind, n_x, fam, sp)
    if scale != 1.0:
        M = M * scale
    return torch.from_numpy(np.ascontiguousarray(M)).to(torch.device("cuda", dev_index))


def _apply_operator(M, lines):
    """(n x N) float64 operator applied to (N, L) complex128 lines -> (n, L)."""
    import torch

    N, L = lines.shape
    xr = torch.view_as_real(lines).reshape(N, 2 * L)
    out = torch.matmul(M, xr)
    return torch.view_as_complex(out.view(M.shape[0], L, 2))


@lru_cache(maxsize=16)
def _paired_dev(kind: str, n_x: int, fam: int, sp: int, dev_index: int, scale: float = 1.0):
    """Mirror-paired blocks of an operator, or None if it has no mirror parity.

    x_{N-1-j} = -x_j and every basis function has the parity of its mode, so
    the inverse E (N x n) satisfies E[N-1-j, k] = (-1)^k E[j, k] and the
    forward F (n x N) F[k, N-1-j] = (-1)^k F[k, j]: even modes couple only
    to pair sums (plus the centre point), odd modes only to pair differences.
    Two GEMMs with the blocks do half the flops of the full operator
    (nonlinear.py uses the same split)."""
    import torch

    M = _operator_host(kind, n_x, fam, sp)
    if scale != 1.0:
        M = M * scale
    N = n_x + 1
    P, Q = (N + 1) // 2, N // 2
    tol = 1e-12 * np.abs(M).max()
    if kind == "inv":
        sign = np.where(np.arange(M.shape[1]) % 2 == 0, 1.0, -1.0)
        if not np.allclose(M[::-1], M * sign, rtol=0, atol=tol):
            return None
        S, A = M[:P, 0::2], M[:Q, 1::2]
    else:
        sign = np.where(np.arange(M.shape[0]) % 2 == 0, 1.0, -1.0)[:, None]
        if not np.allclose(M[:, ::-1], M * sign, rtol=0, atol=tol):
            return None
        S, A = M[0::2, :P], M[1::2, :Q]
    dev = torch.device("cuda", dev_index)
    return (torch.from_numpy(np.ascontiguousarray(S)).to(dev), torch.from_numpy(np.ascontiguousarray(A)).to(dev),
            P, Q)


PAIRED_MIN_LINES = 512  # below this one full GEMM beats split + two GEMMs + pass


def _forward_paired(blocks, lines):
    """(N, L) lines -> (n, L) coefficients: pair split pass, then the even /
    odd mode blocks write the interleaved output rows directly (cuBLAS ldc)."""
    import torch

    S, A, P, Q = blocks
    N, L = lines.shape
    y = torch.empty((N, L), dtype=torch.complex128, device=lines.device)
    _lib.check(_lib.lib().shen_pair_split(P, Q, 2 * L, lines.data_ptr(), y.data_ptr(), stream_handle()),
               "shen_pair_split")
    n = S.shape[0] + A.shape[0]
    out = torch.empty((n, L), dtype=torch.complex128, device=lines.device)
    outr, yr = torch.view_as_real(out).reshape(n, 2 * L), torch.view_as_real(y).reshape(N, 2 * L)
    torch.matmul(S, yr[:P], out=outr[0::2])
    torch.matmul(A, yr[P:], out=outr[1::2])
    return out


def _inverse_paired(blocks, coef):
    """(n, L) coefficients -> (N, L) lines: the even / odd mode blocks read
    strided coefficient rows (cuBLAS ldb) into e, o; one merge pass."""
    import torch

    S, A, P, Q = blocks
    n, L = coef.shape
    N = P + Q
    y = torch.empty((N, L), dtype=torch.complex128, device=coef.device)
    cr, yr = torch.view_as_real(coef).reshape(n, 2 * L), torch.view_as_real(y).reshape(N, 2 * L)
    torch.matmul(S, cr[0::2], out=yr[:P])
    torch.matmul(A, cr[1::2], out=yr[P:])
    lines = torch.empty((N, L), dtype=torch.complex128, device=coef.device)
    _lib.check(_lib.lib().shen_pair_merge(P, Q, 2 * L, y.data_ptr(), lines.data_ptr(), stream_handle()),
               "shen_pair_merge")
    return lines


# ---------------------------------------------------------------- wall-normal stage on lines

def wall_forward(lines, n_x: int, fam: int, sp: int, solve_mass: bool = True):
    """(N, L) complex128 Fourier lines on the device -> (n_modes, L) Shen
    coefficients (scalar products if ``solve_mass`` is False)."""
    if XFORM_METHOD == "wall" and n_x >= 2:
        from .wall import wall_plan

        plan = wall_plan(n_x, fam, sp, 0, solve_mass, _cheb_scale(n_x + 1, fam))
        if plan is not None:
            return _wall_run(plan, lines.contiguous(), plan.struct.n_out)
    if XFORM_METHOD == "matrix":
        kind = "fwd" if solve_mass else "fsp"
        if lines.shape[1] >= PAIRED_MIN_LINES:
            blocks = _paired_dev(kind, n_x, fam, sp, device().index)
            if blocks is not None:
                return _forward_paired(blocks, lines.contiguous())
        return _apply_operator(_operator_dev(kind, n_x, fam, sp, device().index), lines)
    scal = _chebyshev_pass(lines, fam, sp)
    if solve_mass and sp != 0:
        scal = _mass_pass(scal, sp, n_x, fam)
    return scal


def wall_inverse(coef, n_x: int, fam: int, sp: int, yz_points: int = 1):
    """(n, L) coefficients -> (N, L) values on the Chebyshev points, and the
    ``norm`` for the following ``irfft2`` (the matrix route folds the
    1/(n_y n_z) of the inverse FFT into its operator)."""
    if XFORM_METHOD == "wall" and n_x >= 2:
        from .wall import wall_plan

        plan = wall_plan(n_x, fam, sp, 1, False, 1.0 / yz_points)
        if plan is not None and plan.struct.n_in == coef.shape[0]:
            return _wall_run(plan, coef.contiguous(), n_x + 1), "forward"
    if XFORM_METHOD == "matrix":
        if coef.shape[1] >= PAIRED_MIN_LINES:
            blocks = _paired_dev("inv", n_x, fam, sp, device().index, 1.0 / yz_points)
            if blocks is not None:
                return _inverse_paired(blocks, coef.contiguous()), "forward"
        op = _operator_dev("inv", n_x, fam, sp, device().index, 1.0 / yz_points)
        return _apply_operator(op, coef), "forward"
    return _expand_pass(coef, sp, n_x, fam), "backward"


# ---------------------------------------------------------------- 3-D transforms

def _physical_to_device(field: PhysicalField):
    import torch

    d = field.data
    if is_torch(d):
        return d.to(device=device(), dtype=torch.float64).contiguous(), False
    t = torch.from_numpy(np.ascontiguousarray(d, dtype=np.float64))
    if t.numel() > 0:
        t = t.pin_memory()
    return t.to(device(), non_blocking=True), True


def _forward(field: PhysicalField, space, solve_mass: bool):
    import torch

    mesh = field.mesh
    sp = space_code(space)
    fam = _fam(mesh.family)
    u, from_numpy = _physical_to_device(field)
    fourier = torch.fft.rfft2(u, dim=(1, 2)).contiguous()
    del u
    N = fourier.shape[0]
    yz = tuple(fourier.shape[1:])
    lines = fourier.view(N, -1)
    scal = wall_forward(lines, mesh.n_x, fam, sp, solve_mass)
    del fourier, lines
    data = scal.reshape((scal.shape[0],) + yz)
    if from_numpy:
        data = data.cpu().numpy()
    return SpectralField(data, wavenumber_grid(mesh, as_space(sp)), mesh)


def forward_transform(field: PhysicalField, space) -> SpectralField:
    """Physical samples -> expansion coefficients in ``space`` (transforms.py:181-188)."""
    return _forward(field, space, True)


def forward_scalar_product(field: PhysicalField, space) -> SpectralField:
    """Like ``forward_transform`` but stops before the mass solve (transforms.py:191-196)."""
    return _forward(field, space, False)


def inverse_transform(coeffs: SpectralField) -> PhysicalField:
    """Expansion coefficients -> physical samples (transforms.py:199-205)."""
    import torch

    mesh = coeffs.mesh
    sp = space_code(coeffs.grid.space)
    fam = _fam(mesh.family)
    d = coeffs.data
    from_numpy = not is_torch(d)
    if from_numpy:
        t = torch.from_numpy(np.ascontiguousarray(d, dtype=np.complex128))
        if t.numel() > 0:
            t = t.pin_memory()
        t = t.to(device(), non_blocking=True)
    else:
        t = d.to(device=device(), dtype=torch.complex128).contiguous()
    n = t.shape[0]
    yz = tuple(t.shape[1:])
    _check_expand_rows(n, sp, mesh.n_x)
    lines, norm = wall_inverse(t.reshape(n, -1), mesh.n_x, fam, sp, mesh.n_y * mesh.n_z)
    del t
    data = torch.fft.irfft2(lines.reshape((mesh.n_x + 1,) + yz), s=(mesh.n_y, mesh.n_z), dim=(1, 2), norm=norm)
    if from_numpy:
        data = data.cpu().numpy()
    return PhysicalField(data, mesh)
