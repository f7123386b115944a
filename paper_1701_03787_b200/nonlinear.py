"""The stepper's nonlinear term on the device (
reference ``stepper.py:148-185``, ``ChannelStepper.compute_nonlinear``).

H = u x omega from the spectral state (u in the biharmonic space, v, w and
g = omega_x in the Dirichlet space), every wall-normal stage on the fused
transform kernel (``csrc/shen_wall.cu``, the same kernel as the 3-D
transforms):

* u, v, w, om_x: ``shen_wall_transform`` inverse plans of their spaces, the
  1/(n_y n_z) of the inverse periodic FFT folded into the kernel;
* dv/dx, dw/dx: ``deriv_dir_to_cheb.apply`` (``csrc/shen_apply.cu``, the
  reference's structured apply) gives the Chebyshev coefficients, the inverse
  Chebyshev-space plan scales them by 1/mass_cheb in its gather (the
  reference's ``c *= mass_inv``, same product) and evaluates them;
* du/dy, du/dz: the 1j m / 1j n factors act per Fourier line, so the plane
  irfft2 kernel applies them to u's evaluated lines while it loads them
  (``shen_plane_irfft2_fac``): no pass or array of their own;
* the periodic irfft2 of the 8 fields (``csrc/shen_plane_fft.cu`` for 256 x
  256 planes), ``shen_cross`` for om_y, om_z and the three components of H
  (one pass), one batched rfft2 with the dealiasing mask applied at its store
  (``shen_plane_rfft2_fac``; the 0 / 1 factor per line commutes with the
  per-line stage that follows), three forward Dirichlet plans (DCT + stencil
  + mass solve).

No GEMM: the wall-normal work is the O(N log N) on-chip DCTs.  Rounding
differs from the reference's pocketfft/LAPACK chain at the 1e-15 level
(tests/test_nonlinear_gpu.py gates 1e-12 of each field's maximum).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import device, is_torch, stream_handle
from .mesh import family_code
from .transforms import plane_irfft2, plane_rfft2

__all__ = ["NonlinearTerm", "compute_nonlinear"]


class NonlinearTerm:
    """Device ``compute_nonlinear`` for one mesh (plans and tables uploaded once).

    ``m``, ``n``, ``mask`` as the stepper holds them (``grid.m_scaled[:, None]``,
    ``grid.n_scaled[None, :]``, ``_spectral_mask()``)."""

    def __init__(self, mats, mesh, m, n, mask):
        import torch

        from .operators import DeviceOperator
        from .transforms import _cheb_scale
        from .wall import wall_plan

        dev = device()
        self.dev = dev
        self.mesh = mesh
        self.n_x, self.n_y, self.n_z = mesh.n_x, mesh.n_y, mesh.n_z
        fam = family_code(mesh.family)
        self.nzh = self.n_z // 2 + 1
        plane = (self.n_y, self.nzh)
        self.L = self.n_y * self.nzh
        N = self.n_x + 1
        yz = 1.0 / (self.n_y * self.n_z)
        self._inv = {sp: wall_plan(self.n_x, fam, sp, 1, False, yz) for sp in (1, 2)}
        self._inv_ddx = wall_plan(self.n_x, fam, 0, 1, False, yz, rowscale=1.0 / mats.mass_cheb,
                                  rowscale_key=("inv_mass_cheb", id(mats)))
        self._fwd = wall_plan(self.n_x, fam, 1, 0, True, _cheb_scale(N, fam))
        if any(pl is None for pl in (*self._inv.values(), self._inv_ddx, self._fwd)):
            raise _lib.ShenBackendError(f"n_x = {self.n_x} does not fit the wall-normal transform kernel")
        self._keep_mats = mats  # the rowscale plan is cached under id(mats)
        self._deriv = DeviceOperator(mats.deriv_dir_to_cheb)

        def line(a):
            return torch.from_numpy(np.array(np.broadcast_to(a, plane), dtype=np.float64).reshape(-1)).to(dev)

        im_m, im_n = 1j * np.asarray(m, dtype=float), 1j * np.asarray(n, dtype=float)
        self._cm = (line(np.real(im_m)), line(np.imag(im_m)))
        self._cn = (line(np.real(im_n)), line(np.imag(im_n)))
        self._mask = (line(np.asarray(mask, dtype=float)), line(np.zeros(plane)))

    def _wall(self, plan, x, out):
        import ctypes

        _lib.check(_lib.lib().shen_wall_transform(ctypes.byref(plan.struct), self.L, x.data_ptr(), out.data_ptr(),
                                                  stream_handle()), "shen_wall_transform")

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
        L, N = self.L, self.n_x + 1
        # point values (wall-normal) of the 8 fields on the Fourier lines, in shen_cross order:
        # u, v, w, om_x, dv/dx, dw/dx, du/dy, du/dz (stepper.py:165-174)
        # The y / z derivatives of u (fields 6, 7) are its lines times i m / i n: the plane kernel
        # applies the factor while it loads the lines, so they need no pass (or array) of their own.
        spec = torch.empty((6, N, L), dtype=torch.complex128, device=self.dev)
        self._wall(self._inv[2], u_hat, spec[0])
        self._wall(self._inv[1], v_hat, spec[1])
        self._wall(self._inv[1], w_hat, spec[2])
        self._wall(self._inv[1], g_hat, spec[3])
        self._wall(self._inv_ddx, self._deriv(v_hat.view(v_hat.shape[0], L)), spec[4])
        self._wall(self._inv_ddx, self._deriv(w_hat.view(w_hat.shape[0], L)), spec[5])
        phys = torch.empty((8, N, self.n_y, self.n_z), dtype=torch.float64, device=self.dev)
        plane_irfft2(spec.view(6, N, self.n_y, self.nzh), self.n_y, self.n_z, "forward", out=phys[:6])
        u_lines = spec[0].view(N, self.n_y, self.nzh)
        plane_irfft2(u_lines, self.n_y, self.n_z, "forward", fac=self._cm, out=phys[6])  # du/dy
        plane_irfft2(u_lines, self.n_y, self.n_z, "forward", fac=self._cn, out=phys[7])  # du/dz
        del spec
        npt = N * self.n_y * self.n_z
        h = torch.empty((3, N, self.n_y, self.n_z), dtype=torch.float64, device=self.dev)
        _lib.check(_lib.lib().shen_cross(npt, phys.data_ptr(), h.data_ptr(), stream_handle()), "shen_cross")
        del phys
        # dealiasing mask (apply_mask, stepper.py:142-144) at the plane kernel's store: a 0 / 1 factor
        # per Fourier line commutes with the per-line wall-normal transform that follows
        hf = plane_rfft2(h, fac=self._mask[0]).view(3, N, L)
        del h
        n_dir = self.n_x - 1
        out = []
        for i in range(3):
            o = torch.empty((n_dir, L), dtype=torch.complex128, device=self.dev)
            self._wall(self._fwd, hf[i], o)
            o = o.view(n_dir, self.n_y, self.nzh)
            out.append(o.cpu().numpy() if from_numpy else o)
        return tuple(out)


def compute_nonlinear(mats, mesh, m, n, mask, u_hat, v_hat, w_hat, g_hat):
    """Functional ``ChannelStepper.compute_nonlinear`` (stepper.py:148-185)."""
    return NonlinearTerm(mats, mesh, m, n, mask)(u_hat, v_hat, w_hat, g_hat)
