"""Right-hand sides of the implicit updates on the device (SURVEY.md 8(f)
rank 1; reference ``stepper.py:189-219``).

The reference's stepper forms, every time step,

* ``_ab2``: ``h_ab = 1.5 h_curr - 0.5 h_prev`` for the three nonlinear
  components (``stepper.py:189-191``);
* ``assemble_rhs_g`` (``:209-219``): the explicit side of the Helmholtz
  update of the wall-normal vorticity g;
* ``assemble_rhs_u`` (``:193-207``): the explicit side of the biharmonic
  update of the wall-normal velocity u;

through a dozen numpy temporaries.  Here each is ONE pass of
``csrc/shen_rhs.cu`` over the Fourier lines (AB2 folded in), bit-identical to
the reference.  The outputs are exactly the right-hand sides
``HelmholtzLU.solve`` / ``BiharmonicLU.solve`` take.

``RhsAssembler(mats, nu, dt, grid)`` uploads the matrix tables and per-line
coefficients once (like the stepper's constructor); ``rhs_g`` / ``rhs_u``
take device tensors (zero copy) or numpy arrays.  The functional forms
``assemble_rhs_g`` / ``assemble_rhs_u`` mirror the stepper methods with the
state passed explicitly.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._device import device, is_torch, stream_handle

__all__ = ["RhsAssembler", "assemble_rhs_g", "assemble_rhs_u", "ab2"]


def ab2(h_curr, h_prev):
    """``_ab2`` (stepper.py:189-191) -- host/torch elementwise form, for callers
    that want h_ab itself (the device assemblers fold it in)."""
    return tuple(1.5 * c - 0.5 * p for c, p in zip(h_curr, h_prev))


def _band(M, dev):
    import torch

    nr, nc = M.shape
    offs = tuple(int(d) for d in M.offsets)
    tab = np.zeros((max(len(offs), 1), nr))
    for i, (d, diag) in enumerate(zip(offs, M.diagonals)):
        a, b = max(0, -d), min(nr, nc - d)
        tab[i, a:b] = diag
    t = torch.from_numpy(tab).to(dev)
    b = _lib.ShenBand()
    b.nr, b.nc, b.n_off = nr, nc, len(offs)
    for i, d in enumerate(offs):
        b.off[i] = d
    b.diag = t.data_ptr()
    return b, t


class RhsAssembler:
    """Device right-hand-side assembly for one (mats, nu, dt, wavenumber grid).

    ``m`` and ``n`` are the scaled wavenumbers as the stepper holds them
    (``grid.m_scaled[:, None]``, ``grid.n_scaled[None, :]``) and ``z2`` their
    squared sum (``grid.z2()``); any shapes broadcasting to the (n_y, n_z/2+1)
    plane are accepted."""

    def __init__(self, mats, nu: float, dt: float, z2, m, n):
        import torch

        dev = device()
        self.dev = dev
        self.n_dir, self.n_bih = mats.n_dir, mats.n_bih
        z2 = np.asarray(z2, dtype=float)
        m = np.asarray(m, dtype=float)
        n = np.asarray(n, dtype=float)
        self.plane = np.broadcast_shapes(z2.shape, m.shape, n.shape)
        keep = []

        def up(a, dtype=np.float64):
            t = torch.from_numpy(np.array(np.broadcast_to(a, self.plane), dtype=dtype).reshape(-1)).to(dev)
            keep.append(t)
            return t.data_ptr()

        # per-line coefficients: the reference's own numpy expressions
        cg = 1 - nu * dt * z2 / 2                      # stepper.py:214
        im_m, im_n = 1j * m, 1j * n                    # stepper.py:217
        cs_u = 1 - nu * dt * z2                        # stepper.py:200
        cm_u = -z2 + nu * dt * z2 ** 2 / 2             # stepper.py:201
        cx_u = dt * z2                                 # stepper.py:204
        cy_u, cz_u = dt * 1j * m, dt * 1j * n          # stepper.py:205-206
        g = _lib.ShenRhsGArgs()
        g.n_dir = mats.n_dir
        g.stiff, t1 = _band(mats.stiff_dir.banded, dev)
        g.mass, t2 = _band(mats.mass_dir, dev)
        keep += [t1, t2]
        tail = torch.from_numpy(np.ascontiguousarray(mats.stiff_dir.tail, dtype=np.float64)).to(dev)
        keep.append(tail)
        g.tail, g.tail_start = tail.data_ptr(), int(mats.stiff_dir.tail_start)
        g.c_stiff, g.dt = -(nu * dt / 2), dt
        g.cg = up(cg)
        g.im_m_re, g.im_m_im = up(np.real(im_m)), up(np.imag(im_m))
        g.im_n_re, g.im_n_im = up(np.real(im_n)), up(np.imag(im_n))
        u = _lib.ShenRhsUArgs()
        u.n_bih = mats.n_bih
        fb = mats.fourth_bih
        vecs = [torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(dev) for v in (fb.diag, fb.p, fb.q,
                                                                                            fb.r, fb.s)]
        keep += vecs
        u.d, u.p, u.q, u.r, u.s = (v.data_ptr() for v in vecs)
        u.c_fourth = nu * dt / 2
        for name, M in (("stiff", mats.stiff_bih), ("mass", mats.mass_bih), ("mixed", mats.mixed_mass),
                        ("deriv", mats.deriv_dir_to_bih)):
            b, t = _band(M, dev)
            keep.append(t)
            setattr(u, name, b)
        u.c_stiff, u.c_mass, u.c_mixed = up(cs_u), up(cm_u), up(cx_u)
        u.c_dy_re, u.c_dy_im = up(np.real(cy_u)), up(np.imag(cy_u))
        u.c_dz_re, u.c_dz_im = up(np.real(cz_u)), up(np.imag(cz_u))
        self._g, self._u, self._keep = g, u, keep
        self.L = int(np.prod(self.plane, dtype=np.int64))

    def _dev(self, x, rows, what):
        import torch

        if is_torch(x):
            t = x.to(device=self.dev, dtype=torch.complex128).contiguous()
        else:
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(self.dev)
        if tuple(t.shape) != (rows,) + tuple(self.plane):
            raise ValueError(f"{what}: shape {tuple(t.shape)}, expected {(rows,) + tuple(self.plane)}")
        return t

    def rhs_g(self, g, h_curr, h_prev):
        """``assemble_rhs_g(state, _ab2(state))`` (stepper.py:209-219)."""
        import torch

        from_numpy = not is_torch(g)
        gd = self._dev(g, self.n_dir, "g")
        hs = [self._dev(h, self.n_dir, "h") for h in (h_curr[1], h_prev[1], h_curr[2], h_prev[2])]
        out = torch.empty_like(gd)
        a = self._g
        a.L = self.L
        a.g, a.hcy, a.hpy, a.hcz, a.hpz = gd.data_ptr(), *(h.data_ptr() for h in hs)
        a.out = out.data_ptr()
        _lib.check(_lib.lib().shen_rhs_g(ctypes.byref(a), stream_handle()), "shen_rhs_g")
        return out.cpu().numpy() if from_numpy else out

    def rhs_u(self, u, h_curr, h_prev):
        """``assemble_rhs_u(state, _ab2(state))`` (stepper.py:193-207)."""
        import torch

        from_numpy = not is_torch(u)
        ud = self._dev(u, self.n_bih, "u")
        hs = [self._dev(h, self.n_dir, "h") for h in (h_curr[0], h_prev[0], h_curr[1], h_prev[1], h_curr[2],
                                                       h_prev[2])]
        out = torch.empty_like(ud)
        a = self._u
        a.L = self.L
        a.u = ud.data_ptr()
        a.hcx, a.hpx, a.hcy, a.hpy, a.hcz, a.hpz = (h.data_ptr() for h in hs)
        a.out = out.data_ptr()
        _lib.check(_lib.lib().shen_rhs_u(ctypes.byref(a), stream_handle()), "shen_rhs_u")
        return out.cpu().numpy() if from_numpy else out


def assemble_rhs_g(mats, nu, dt, z2, m, n, g, h_curr, h_prev):
    """Functional ``ChannelStepper.assemble_rhs_g`` (stepper.py:209-219)."""
    return RhsAssembler(mats, nu, dt, z2, m, n).rhs_g(g, h_curr, h_prev)


def assemble_rhs_u(mats, nu, dt, z2, m, n, u, h_curr, h_prev):
    """Functional ``ChannelStepper.assemble_rhs_u`` (stepper.py:193-207)."""
    return RhsAssembler(mats, nu, dt, z2, m, n).rhs_u(u, h_curr, h_prev)
