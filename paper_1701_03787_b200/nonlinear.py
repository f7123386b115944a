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
* mirror pairing: the points x_j and x_{N-1-j} = -x_j are mirror images and
  every basis function has a parity (phi_k(-x) = (-1)^k phi_k(x); d/dx flips
  it), so each wall-normal operator splits into a symmetric block (even
  modes -> e_j = half-sum of the pair's values) and an antisymmetric block
  (odd modes -> o_j): two GEMMs of a quarter of the size each, half the flops.
  The fields stay in that e/o form through the FFTs (linear per wall-normal
  row), ``shen_cross_paired`` forms the values at both points of each pair,
  computes H there and writes H's pair sums and differences, which the
  forward operator's even / odd mode blocks consume; ``shen_scale_rows``
  interleaves the two coefficient blocks while applying the mask.  No pass is
  added.

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

        # mirror-paired blocks (module docstring): P = ceil(N/2) symmetric
        # rows (pairs + centre), Q = floor(N/2) antisymmetric rows
        N = self.n_x + 1
        self.P, self.Q = (N + 1) // 2, N // 2
        self._inv_bih = self._pair_inverse(_operator_host("inv", self.n_x, fam, 2) * scale, 0)
        self._inv_dir = self._pair_inverse(e_dir, 0)
        self._inv_ddx = self._pair_inverse(e_ddx, 1)
        self._fwd = self._pair_forward(_operator_host("fwd", self.n_x, fam, 1))

        def line(a):
            return torch.from_numpy(np.array(np.broadcast_to(a, plane), dtype=np.float64).reshape(-1)).to(dev)

        im_m, im_n = 1j * np.asarray(m, dtype=float), 1j * np.asarray(n, dtype=float)
        self._cm = (line(np.real(im_m)), line(np.imag(im_m)))
        self._cn = (line(np.real(im_n)), line(np.imag(im_n)))
        self._mask = (line(np.asarray(mask, dtype=float)), line(np.zeros(plane)))

    def _pair_inverse(self, E, s0):
        """(N x n) evaluation operator -> device blocks (E[:P, s0::2], E[:Q, 1-s0::2]);
        s0 = first mode of the symmetric block (0 for values, 1 for d/dx)."""
        import torch

        N, P, Q = E.shape[0], self.P, self.Q
        sign = np.where((np.arange(E.shape[1]) + s0) % 2 == 0, 1.0, -1.0)
        assert np.allclose(E[::-1], E * sign, rtol=0, atol=1e-12 * np.abs(E).max()), "operator has no mirror parity"
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(self.dev)  # noqa: E731
        return dev(E[:P, s0::2]), dev(E[:Q, 1 - s0::2]), s0

    def _pair_forward(self, F):
        """(n x N) forward operator -> (F[0::2, :P], F[1::2, :Q]) acting on the
        pair sums (centre point included) and differences."""
        import torch

        sign = np.where(np.arange(F.shape[0]) % 2 == 0, 1.0, -1.0)[:, None]
        assert np.allclose(F[:, ::-1], F * sign, rtol=0, atol=1e-12 * np.abs(F).max()), "operator has no mirror parity"
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(self.dev)  # noqa: E731
        return dev(F[0::2, :self.P]), dev(F[1::2, :self.Q])

    def _gemm_rows(self, E, c, first, out):
        """out (rows, L) complex view <- E @ (rows first, first+2, ... of c)."""
        import torch

        n = c.shape[0]
        xr = torch.view_as_real(c.reshape(n, self.L)).reshape(n, 2 * self.L)[first::2]
        torch.matmul(E, xr, out=torch.view_as_real(out).reshape(E.shape[0], 2 * self.L))

    def _inverse_paired(self, blocks, c, out):
        """out (P + Q, L): e rows then o rows of the field with coefficients c."""
        Es, Ea, s0 = blocks
        self._gemm_rows(Es, c, s0, out[:self.P])
        self._gemm_rows(Ea, c, 1 - s0, out[self.P:])

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
        L, P, Q = self.L, self.P, self.Q
        R = P + Q
        # spectral lines of the 8 fields (mirror-paired rows), in shen_cross order
        spec = torch.empty((8, R, L), dtype=torch.complex128, device=self.dev)
        self._inverse_paired(self._inv_bih, u_hat, spec[0])
        self._inverse_paired(self._inv_dir, v_hat, spec[1])
        self._inverse_paired(self._inv_dir, w_hat, spec[2])
        self._inverse_paired(self._inv_dir, g_hat, spec[3])
        self._inverse_paired(self._inv_ddx, v_hat, spec[4])
        self._inverse_paired(self._inv_ddx, w_hat, spec[5])
        self._scale(spec[0], self._cm, spec[6])   # du/dy lines
        self._scale(spec[0], self._cn, spec[7])   # du/dz lines
        phys = torch.fft.irfft2(spec.view(8, R, self.n_y, self.nzh), s=(self.n_y, self.n_z), dim=(2, 3),
                                norm="forward").contiguous()
        del spec
        h = torch.empty((3, R, self.n_y, self.n_z), dtype=torch.float64, device=self.dev)
        _lib.check(_lib.lib().shen_cross_paired(P, Q, self.n_y * self.n_z, phys.data_ptr(), h.data_ptr(),
                                                stream_handle()), "shen_cross_paired")
        del phys
        hf = torch.fft.rfft2(h, dim=(2, 3)).contiguous().view(3, R, L)
        del h
        Fs, Fa = self._fwd
        n_dir = Fs.shape[0] + Fa.shape[0]
        out = []
        tmp_s = torch.empty((Fs.shape[0], L), dtype=torch.complex128, device=self.dev)
        tmp_a = torch.empty((Fa.shape[0], L), dtype=torch.complex128, device=self.dev)
        lib, st = _lib.lib(), stream_handle()
        for i in range(3):
            self._gemm(Fs, hf[i, :P], tmp_s)
            self._gemm(Fa, hf[i, P:], tmp_a)
            o = torch.empty((n_dir, L), dtype=torch.complex128, device=self.dev)
            # even / odd coefficient rows interleaved while the mask is applied
            _lib.check(lib.shen_scale_rows(Fs.shape[0], L, tmp_s.data_ptr(), L, self._mask[0].data_ptr(),
                                           self._mask[1].data_ptr(), o.data_ptr(), 2 * L, st), "shen_scale_rows")
            _lib.check(lib.shen_scale_rows(Fa.shape[0], L, tmp_a.data_ptr(), L, self._mask[0].data_ptr(),
                                           self._mask[1].data_ptr(), o[1:].data_ptr(), 2 * L, st), "shen_scale_rows")
            o = o.view(n_dir, self.n_y, self.nzh)
            out.append(o.cpu().numpy() if from_numpy else o)
        return tuple(out)


def compute_nonlinear(mats, mesh, m, n, mask, u_hat, v_hat, w_hat, g_hat):
    """Functional ``ChannelStepper.compute_nonlinear`` (stepper.py:148-185)."""
    return NonlinearTerm(mats, mesh, m, n, mask)(u_hat, v_hat, w_hat, g_hat)
