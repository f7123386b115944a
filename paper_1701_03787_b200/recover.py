"""Divergence variable and horizontal-velocity recovery on the device
(reference ``stepper.py:296-303``):

    f_scal = deriv_bih_to_dir.apply(u_new)
    f_hat  = mass_solve(f_scal, DIRICHLET, n_x, family)
    v_new  = (1j m f_hat + 1j n g_new) / safe_z2
    w_new  = (1j n f_hat - 1j m g_new) / safe_z2

fused into one kernel (``csrc/shen_recover.cu``).  The mean mode
(m = n = 0, where safe_z2 = 1) is overwritten by the stepper's mean-flow
solve (``stepper.py:305-333``), which callers do with a one-system
``build_helmholtz(mats, nu, dt, 0)``.  The mass solve follows LAPACK's
banded Cholesky with the same factors, so results agree with the reference
to rounding (tests gate 1e-12), not bitwise.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._device import device, is_torch, stream_handle
from .mesh import family_code
from .rhs import _band

__all__ = ["VelocityRecovery", "recover_velocity"]


class VelocityRecovery:
    """Device velocity recovery for one (mats, wavenumber plane)."""

    def __init__(self, mats, z2, m, n):
        import torch

        from .transforms import _mass_factors_dev

        dev = device()
        self.dev = dev
        self.n_dir, self.n_bih = mats.n_dir, mats.n_bih
        z2 = np.asarray(z2, dtype=float)
        self.plane = np.broadcast_shapes(z2.shape, np.shape(m), np.shape(n))
        self.L = int(np.prod(self.plane, dtype=np.int64))
        keep = []

        def up(a):
            t = torch.from_numpy(np.array(np.broadcast_to(a, self.plane), dtype=np.float64).reshape(-1)).to(dev)
            keep.append(t)
            return t.data_ptr()

        im_m, im_n = 1j * np.asarray(m, dtype=float), 1j * np.asarray(n, dtype=float)
        fac, nband, nrows, mmax = _mass_factors_dev(mats.n_x, family_code(mats.family), 1, dev.index)
        a = _lib.ShenRecoverArgs()
        a.n_dir = mats.n_dir
        a.deriv, t = _band(mats.deriv_bih_to_dir, dev)
        keep += [t, fac]
        a.fac, a.mmax = fac.data_ptr(), mmax
        a.im_m_re, a.im_m_im = up(np.real(im_m)), up(np.imag(im_m))
        a.im_n_re, a.im_n_im = up(np.real(im_n)), up(np.imag(im_n))
        a.safe_z2 = up(np.where(z2 > 0, z2, 1.0))
        self._a, self._keep = a, keep

    def __call__(self, u_new, g_new):
        """(v_new, w_new), (n_dir, n_y, n_z/2+1) complex128 each."""
        import torch

        from_numpy = not is_torch(u_new)

        def dev(x, rows, what):
            t = (x.to(device=self.dev, dtype=torch.complex128).contiguous() if is_torch(x)
                 else torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(self.dev))
            if tuple(t.shape) != (rows,) + tuple(self.plane):
                raise ValueError(f"{what}: shape {tuple(t.shape)}, expected {(rows,) + tuple(self.plane)}")
            return t

        ud, gd = dev(u_new, self.n_bih, "u_new"), dev(g_new, self.n_dir, "g_new")
        v = torch.empty_like(gd)
        w = torch.empty_like(gd)
        a = self._a
        a.L = self.L
        a.u, a.g, a.v, a.w = ud.data_ptr(), gd.data_ptr(), v.data_ptr(), w.data_ptr()
        _lib.check(_lib.lib().shen_recover_velocity(ctypes.byref(a), stream_handle()), "shen_recover_velocity")
        if from_numpy:
            return v.cpu().numpy(), w.cpu().numpy()
        return v, w


def recover_velocity(mats, z2, m, n, u_new, g_new):
    """Functional form of stepper.py:296-303 (mean mode left to the caller)."""
    return VelocityRecovery(mats, z2, m, n)(u_new, g_new)
