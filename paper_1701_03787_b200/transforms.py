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
* wall-normal stage (default): one fused kernel per direction
  (``shen_wall_transform``, csrc/shen_wall.cu) on tiles of Fourier lines in
  shared memory -- the DCT as an on-chip FFT (power-of-two, Rader or
  Bluestein), the Chebyshev scaling, the Shen stencil and the per-parity
  banded Cholesky mass solve with the reference's own LAPACK factors
  (transforms.py:143-160), one HBM read and one write per line;
* alternative route (``SHEN_XFORM=fft``, and the 1-D blocks below N = 3):
  our ``shen_xform_extend`` / ``shen_xform_inv_pre`` kernels build the
  extended sequence, cuFFT does one FFT along the rows, our post kernels
  apply twiddle, scaling and stencil, ``shen_xform_mass_solve`` the mass
  solve.

numpy inputs are copied to the device and the result copied back (numpy out);
torch CUDA tensors stay on the device (torch out).  There is no CPU fallback:
without the library or a GPU every call raises ``ShenBackendError``.
"""

from __future__ import annotations

import ctypes
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


def _wall_run(plan, x, rows_out, out=None):
    """shen_wall_transform of (rows_in, L) complex128 lines -> (rows_out, L)
    (into ``out`` when given: a contiguous complex128 device buffer of that shape)."""
    import torch

    L = x.shape[1]
    if out is None:
        out = torch.empty((rows_out, L), dtype=torch.complex128, device=x.device)
    elif not (out.is_cuda and out.dtype == torch.complex128 and out.is_contiguous() and out.numel() == rows_out * L):
        raise ValueError("out must be a contiguous complex128 device buffer of rows_out x L elements")
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
        if plan is not None and not (fam == 0 and plan.struct.log2_lines == 0):  # (route choice: wall_forward)
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
        if plan is not None and plan.struct.n_in == n and not (fam == 0 and plan.struct.log2_lines == 0):
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


# ---------------------------------------------------------------- wall-normal route
#
# Default (SHEN_XFORM=wall): the fused wall-normal kernel (csrc/shen_wall.cu,
# plans built in wall.py) does the whole axis-0 stage of a transform in one
# pass over the lines.  SHEN_XFORM=fft selects the extension / cuFFT / post
# pipeline above instead (also the route of the 1-D blocks when N < 3).

XFORM_METHOD = __import__("os").environ.get("SHEN_XFORM", "wall")


# ---------------------------------------------------------------- wall-normal stage on lines

# Route choice for large n_x (tools/wall_split_mass.py, 8192 and 33,024 lines):
# the fused kernel's mass solve runs 2 TL serial chains per CTA, so with few
# lines per tile the fused scalar product followed by the standalone
# mass-solve kernel (one thread per (line, parity) over all lines) is faster:
# TL <= 2 always (n_x = 1024 Lobatto, 33k lines: 4.59 -> 1.58 ms), TL = 4
# once there are enough lines to fill the GPU with chains (n_x = 512
# Lobatto: 0.76 -> 0.66 ms at 33k lines, but 0.20 -> 0.32 ms at 8192).  With
# one line per tile (Gauss n_x >= 1024, Bluestein over M = 4096) the cuFFT
# route is faster in both directions (3.5 vs 4.5 ms forward, 0.72 vs 0.98 ms
# inverse at 8192 lines).


def _split_mass(log2_lines: int, n_lines: int) -> bool:
    return log2_lines <= 1 or (log2_lines == 2 and n_lines >= 16384)


def wall_forward(lines, n_x: int, fam: int, sp: int, solve_mass: bool = True):
    """(N, L) complex128 Fourier lines on the device -> (n_modes, L) Shen
    coefficients (scalar products if ``solve_mass`` is False)."""
    if XFORM_METHOD == "wall" and n_x >= 2:
        from .wall import wall_plan

        plan = wall_plan(n_x, fam, sp, 0, solve_mass, _cheb_scale(n_x + 1, fam))
        tls = plan.struct.log2_lines if plan is not None else -1
        if plan is not None and not (fam == 0 and tls == 0):
            if solve_mass and sp != 0 and _split_mass(tls, lines.shape[1]):
                fsp = wall_plan(n_x, fam, sp, 0, False, _cheb_scale(n_x + 1, fam))
                scal = _wall_run(fsp, lines.contiguous(), fsp.struct.n_out)
                return _mass_pass(scal, sp, n_x, fam)
            return _wall_run(plan, lines.contiguous(), plan.struct.n_out)
    scal = _chebyshev_pass(lines, fam, sp)
    if solve_mass and sp != 0:
        scal = _mass_pass(scal, sp, n_x, fam)
    return scal


def wall_inverse(coef, n_x: int, fam: int, sp: int, yz_points: int = 1, out=None):
    """(n, L) coefficients -> (N, L) values on the Chebyshev points, and the
    ``norm`` for the following ``irfft2`` (the wall kernel folds the
    1/(n_y n_z) of the inverse FFT into its output scale).  ``out``: write the
    values into this (N, L) complex128 device buffer (the slab transforms'
    exchange buffer)."""
    if XFORM_METHOD == "wall" and n_x >= 2:
        from .wall import wall_plan

        plan = wall_plan(n_x, fam, sp, 1, False, 1.0 / yz_points)
        if plan is not None and plan.struct.n_in == coef.shape[0] and not (fam == 0 and plan.struct.log2_lines == 0):
            return _wall_run(plan, coef.contiguous(), n_x + 1, out), "forward"
    vals = _expand_pass(coef, sp, n_x, fam)
    if out is not None:
        out.view(vals.shape).copy_(vals)
        vals = out.view(vals.shape)
    return vals, "backward"


# ---------------------------------------------------------------- 3-D transforms

def plane_rfft2(u, fac=None):
    """numpy ``rfft2`` over the last two axes of a contiguous float64 CUDA
    tensor (..., n_y, n_z).  256 x 256 planes run on the cluster kernel of
    ``csrc/shen_plane_fft.cu`` (one HBM pass); other sizes on cuFFT.
    ``fac``: a real float64 device tensor of n_y (n_z/2+1) elements that
    multiplies every plane's spectrum (applied at the kernel's store)."""
    import torch

    n_y, n_z = u.shape[-2], u.shape[-1]
    if not _lib.lib().shen_plane_fft_supported(n_y, n_z):
        X = torch.fft.rfft2(u, dim=(-2, -1))
        if fac is not None:
            X = X * fac.view(n_y, n_z // 2 + 1)
        return X.contiguous()
    u = u.contiguous()
    out = torch.empty(u.shape[:-1] + (n_z // 2 + 1,), dtype=torch.complex128, device=u.device)
    planes = u.numel() // (n_y * n_z)
    if fac is None:
        _lib.check(_lib.lib().shen_plane_rfft2(planes, n_y, n_z, u.data_ptr(), out.data_ptr(), stream_handle()),
                   "shen_plane_rfft2")
    else:
        _check_fac(fac, n_y, n_z, u.device)
        _lib.check(_lib.lib().shen_plane_rfft2_fac(planes, n_y, n_z, u.data_ptr(), out.data_ptr(), fac.data_ptr(),
                                                   stream_handle()), "shen_plane_rfft2_fac")
    return out


def _check_fac(f, n_y, n_z, dev):
    import torch

    if not (is_torch(f) and f.device == dev and f.dtype == torch.float64 and f.is_contiguous()
            and f.numel() == n_y * (n_z // 2 + 1)):
        raise ValueError("line factors must be contiguous float64 device tensors of n_y (n_z/2+1) elements")


def plane_irfft2(X, n_y: int, n_z: int, norm: str = "backward", fac=None, out=None):
    """numpy ``irfft2(X, s=(n_y, n_z), norm=norm)`` over the last two axes of
    a contiguous complex128 CUDA tensor (..., n_y, n_z/2 + 1); cluster kernel
    for 256 x 256 planes, cuFFT otherwise.  ``fac = (re, im)``: float64 device
    tensors of n_y (n_z/2+1) elements; every plane's spectrum is multiplied by
    re + i im first (at the kernel's load).  ``out``: a contiguous float64
    device tensor of the result's shape to write into."""
    import torch

    shape = X.shape[:-2] + (n_y, n_z)
    if out is not None and not (out.is_cuda and out.dtype == torch.float64 and out.is_contiguous()
                                and tuple(out.shape) == tuple(shape)):
        raise ValueError(f"out must be a contiguous float64 device tensor of shape {tuple(shape)}")
    if not _lib.lib().shen_plane_fft_supported(n_y, n_z) or X.shape[-1] != n_z // 2 + 1 or X.shape[-2] != n_y:
        if fac is not None:
            X = X * torch.complex(fac[0], fac[1]).view(n_y, n_z // 2 + 1)
        r = torch.fft.irfft2(X, s=(n_y, n_z), dim=(-2, -1), norm=norm)
        if out is None:
            return r
        out.copy_(r)
        return out
    X = X.contiguous()
    if out is None:
        out = torch.empty(shape, dtype=torch.float64, device=X.device)
    planes = X.numel() // (n_y * (n_z // 2 + 1))
    scale = {"backward": 1.0 / (n_y * n_z), "forward": 1.0, "ortho": 1.0 / np.sqrt(n_y * n_z)}[norm]
    if fac is None:
        _lib.check(_lib.lib().shen_plane_irfft2(planes, n_y, n_z, X.data_ptr(), out.data_ptr(), ctypes.c_double(scale),
                                                stream_handle()), "shen_plane_irfft2")
    else:
        _check_fac(fac[0], n_y, n_z, X.device)
        _check_fac(fac[1], n_y, n_z, X.device)
        _lib.check(_lib.lib().shen_plane_irfft2_fac(planes, n_y, n_z, X.data_ptr(), out.data_ptr(),
                                                    ctypes.c_double(scale), fac[0].data_ptr(), fac[1].data_ptr(),
                                                    stream_handle()), "shen_plane_irfft2_fac")
    return out


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
    fourier = plane_rfft2(u)
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
    data = plane_irfft2(lines.reshape((mesh.n_x + 1,) + yz), mesh.n_y, mesh.n_z, norm)
    if from_numpy:
        data = data.cpu().numpy()
    return PhysicalField(data, mesh)
