"""The stepper's nonlinear term on the device (
reference ``stepper.py:148-185``, ``ChannelStepper.compute_nonlinear``).

H = u x omega from the spectral state (u in the biharmonic space, v, w and
g = omega_x in the Dirichlet space):

* wall-normal stage: every inverse transform the reference performs
  (u, v, w, om_x, dv/dx, dw/dx) is one operator per input in 80-bit-built
  fp64 (transforms.py section "wall-normal operators"); dv/dx and dw/dx use
  C diag(1/mass_cheb) D (D = deriv_dir_to_cheb), v and dv/dx come out of ONE
  GEMM with the operators stacked (same for w);
* du/dy, du/dz: the 1j m / 1j n factors are applied to u's lines after its
  wall-normal GEMM (the operators are linear and act per line), by
  ``shen_scale_lines``;
* one batched cuFFT irfft2 for the 8 fields, ``shen_cross`` for
  om_y, om_z and the three components of H (one HBM pass), one batched rfft2,
  the forward Dirichlet operator, and the dealiasing mask (``shen_scale_lines``).

Rounding differs from the reference's pocketfft/LAPACK chain at the 1e-15
level (tests/test_nonlinear_gpu.py gates 1e-12 of the field maximum).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from . import _lib
from ._device import device, is_torch, stream_handle
from .mesh import family_code

__all__ = ["NonlinearTerm", "compute_nonlinear"]


@lru_cache(maxsize=8)
def _ddx_operator_host(n_x: int, fam: int):
    """C diag(1/mass_cheb) D: Dirichlet coefficients -> point values of d/dx
    (stepper.py:156-163 then transforms.py:199-205 in the Chebyshev space)."""
    from .matrices import assemble
    from .transforms import _ld_pi

    mats = assemble(n_x, fam)
    N = n_x + 1
    pi = _ld_pi()
    j = np.arange(N, dtype=np.longdouble)[:, None]
    mm = np.arange(N, dtype=np.longdouble)[None, :]
    theta = pi * (2 * j + 1) / (2 * N) if fam == 0 else pi * j / n_x
    C = np.cos(mm * theta)
    D = mats.deriv_dir_to_cheb.dense().astype(np.longdouble)
    minv = 1 / mats.mass_cheb.astype(np.longdouble)
    return np.ascontiguousarray((C @ (minv[:, None] * D)).astype(np.float64))


class NonlinearTerm:
    """Device ``compute_nonlinear`` for one mesh (operators uploaded once).

    ``m``, ``n``, ``mask`` as the stepper holds them (``grid.m_scaled[:, None]``,
    ``grid.n_scaled[None, :]``, ``_spectral_mask()``)."""

    def __init__(self, mats, mesh, m, n, mask):
        import torch

        from .transforms import _operator_host

        dev = device()
        self.dev = dev
        self.mesh = mesh
        self.n_x, self.n_y, self.n_z = mesh.n_x, mesh.n_y, mesh.n_z
        fam = family_code(mesh.family)
        self.nzh = self.n_z // 2 + 1
        plane = (self.n_y, self.nzh)
        self.L = self.n_y * self.nzh
        scale = 1.0 / (self.n_y * self.n_z)  # irfft2 normalisation folded into the operators
        e_dir = _operator_host("inv", self.n_x, fam, 1) * scale
        e_ddx = _ddx_operator_host(self.n_x, fam) * scale
        self.E_vd = torch.from_numpy(np.ascontiguousarray(np.vstack([e_dir, e_ddx]))).to(dev)  # (2N, n_dir)
        self.E_dir = torch.from_numpy(np.ascontiguousarray(e_dir)).to(dev)
        self.E_bih = torch.from_numpy(np.ascontiguousarray(_operator_host("inv", self.n_x, fam, 2) * scale)).to(dev)
        self.F_dir = torch.from_numpy(_operator_host("fwd", self.n_x, fam, 1)).to(dev)

        def line(a):
            return torch.from_numpy(np.array(np.broadcast_to(a, plane), dtype=np.float64).reshape(-1)).to(dev)

        im_m, im_n = 1j * np.asarray(m, dtype=float), 1j * np.asarray(n, dtype=float)
        self._cm = (line(np.real(im_m)), line(np.imag(im_m)))
        self._cn = (line(np.real(im_n)), line(np.imag(im_n)))
        self._mask = (line(np.asarray(mask, dtype=float)), line(np.zeros(plane)))

    def _gemm(self, E, c, out):
        """out (rows, L) complex view <- E (rows x n) @ c (n, L) complex."""
        import torch

        n = c.shape[0]
        xr = torch.view_as_real(c.reshape(n, self.L)).reshape(n, 2 * self.L)
        torch.matmul(E, xr, out=torch.view_as_real(out).reshape(E.shape[0], 2 * self.L))

    def _scale(self, x, c, y):
        _lib.check(_lib.lib().shen_scale_lines(x.shape[0], self.L, x.data_ptr(), c[0].data_ptr(), c[1].data_ptr(),
                                               y.data_ptr(), stream_handle()), "shen_scale_lines")

    def __call__(self, u_hat, v_hat, w_hat, g_hat):
        """Three (n_dir, n_y, n_z/2+1) complex128 arrays: masked Dirichlet
        coefficients of H = u x omega (numpy in -> numpy out)."""
        import torch

        from_numpy = not is_torch(u_hat)

        def dev(x):
            if is_torch(x):
                return x.to(device=self.dev, dtype=torch.complex128).contiguous()
            return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(self.dev)

        u_hat, v_hat, w_hat, g_hat = (dev(x) for x in (u_hat, v_hat, w_hat, g_hat))
        N, L = self.n_x + 1, self.L
        # spectral lines of the 8 fields, in shen_cross order
        spec = torch.empty((8, N, L), dtype=torch.complex128, device=self.dev)
        self._gemm(self.E_bih, u_hat, spec[0])
        vd = torch.empty((2 * N, L), dtype=torch.complex128, device=self.dev)
        self._gemm(self.E_vd, v_hat, vd)
        spec[1].copy_(vd[:N])
        spec[4].copy_(vd[N:])
        self._gemm(self.E_vd, w_hat, vd)
        spec[2].copy_(vd[:N])
        spec[5].copy_(vd[N:])
        del vd
        self._gemm(self.E_dir, g_hat, spec[3])
        self._scale(spec[0], self._cm, spec[6])   # du/dy lines
        self._scale(spec[0], self._cn, spec[7])   # du/dz lines
        phys = torch.fft.irfft2(spec.view(8, N, self.n_y, self.nzh), s=(self.n_y, self.n_z), dim=(2, 3),
                                norm="forward").contiguous()
        del spec
        h = torch.empty((3, N, self.n_y, self.n_z), dtype=torch.float64, device=self.dev)
        _lib.check(_lib.lib().shen_cross(N * self.n_y * self.n_z, phys.data_ptr(), h.data_ptr(), stream_handle()),
                   "shen_cross")
        del phys
        hf = torch.fft.rfft2(h, dim=(2, 3)).contiguous()
        del h
        out = []
        for i in range(3):
            o = torch.empty((self.F_dir.shape[0], L), dtype=torch.complex128, device=self.dev)
            self._gemm(self.F_dir, hf[i], o)
            self._scale(o, self._mask, o)
            o = o.view(self.F_dir.shape[0], self.n_y, self.nzh)
            out.append(o.cpu().numpy() if from_numpy else o)
        return tuple(out)


def compute_nonlinear(mats, mesh, m, n, mask, u_hat, v_hat, w_hat, g_hat):
    """Functional ``ChannelStepper.compute_nonlinear`` (stepper.py:148-185)."""
    return NonlinearTerm(mats, mesh, m, n, mask)(u_hat, v_hat, w_hat, g_hat)
