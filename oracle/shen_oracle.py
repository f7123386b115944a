"""CPU oracle for the B200 hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the reference algorithms of the
path being accelerated (``/root/reference/pkg/src/chebchan``):

* O(N) Helmholtz factor/solve        -> ``solvers.py:67-126,201-241``
* O(N) biharmonic factor/solve       -> ``solvers.py:72-75,162-198,244-355``
* Shen scalar products / transforms  -> ``transforms.py:81-205``

Every operation keeps the reference's evaluation order (numpy ufunc by ufunc,
no fused multiply-add), so on the same inputs the oracle reproduces the
reference bit for bit; ``tests/test_oracle.py`` pins that against the golden
vectors in ``tests/golden`` (generated from the reference by
``tests/golden/make_golden.py``).  The transforms call scipy.fft / LAPACK
exactly as the reference does (third-party numerics: scipy 1.18.1, pocketfft
and LAPACK ``?pbtrf/?pbtrs``).

Who may import this: ``tests/``, ``__graft_entry__.smoke()`` (as the checker)
and ``bench.py`` (``cpu_baseline`` leg and ``--impl reference``).  The
product package ``paper_1701_03787_b200`` never imports it.

The 1-D row tables (``MatrixSet``) are setup inputs and come from the
product's ``matrices.assemble``, itself pinned bitwise against the reference
by ``tests/test_matrices.py``.
"""

from __future__ import annotations

import numpy as np
from scipy import fft as sfft
from scipy.linalg import cho_solve_banded, cholesky_banded

PIVOT_FLOOR = 1e-300  # solvers.py:54


class OraclePivotError(ArithmeticError):
    pass


# ---------------------------------------------------------------- coefficients

def helmholtz_coefficients(nu, dt, z2):
    """solvers.py:67-69"""
    return nu * dt / 2, 1 + nu * dt * np.asarray(z2, dtype=float) / 2


def biharmonic_coefficients(nu, dt, z2):
    """solvers.py:72-75"""
    z2 = np.asarray(z2, dtype=float)
    return -nu * dt / 2, 1 + nu * dt * z2, -(2 * z2 + nu * dt * z2 ** 2) / 2


def _check(d, what, row):
    if np.any(np.abs(d) < PIVOT_FLOOR):
        raise OraclePivotError(f"{what} factorization hit a near-zero pivot at row {row}")


# ---------------------------------------------------------------- Helmholtz

def helmholtz_factor(mats, nu, dt, z2):
    """Per-parity compressed LU (low, d, e, tail); solvers.py:201-241.
    Returns dict with lists indexed by parity, arrays (rows, batch)."""
    z2 = np.asarray(z2, dtype=float)
    ca, cb = helmholtz_coefficients(nu, dt, z2)
    cbf = np.atleast_1d(cb).reshape(-1)
    nd = mats.n_dir
    sdiag = mats.stiff_dir.banded.diagonal(0)
    stail = mats.stiff_dir.tail
    mdiag = mats.mass_dir.diagonal(0)
    off = -np.pi / 2
    res = {"low": [], "d": [], "e": [], "tail": [], "z2_shape": np.shape(z2)}
    for par in (0, 1):
        k = np.arange(par, nd, 2)
        n = k.size
        hdiag = ca * sdiag[k][:, None] + cbf * mdiag[k][:, None]
        htail = ca * stail[k][:, None] + np.zeros_like(cbf)
        hsup = htail.copy()
        nsup = len(range(par, nd - 2, 2))
        hsup[:nsup] += cbf * off
        hsub = np.broadcast_to(cbf * off, (max(n - 1, 0), cbf.size))
        d = np.empty_like(hdiag)
        e = np.empty_like(hdiag)
        t = np.empty_like(hdiag)
        low = np.empty_like(hsub)
        d[0], e[0], t[0] = hdiag[0], hsup[0], htail[0]
        _check(d[0], "Helmholtz", par)
        for i in range(1, n):
            low[i - 1] = hsub[i - 1] / d[i - 1]
            d[i] = hdiag[i] - low[i - 1] * e[i - 1]
            e[i] = hsup[i] - low[i - 1] * t[i - 1]
            t[i] = htail[i] - low[i - 1] * t[i - 1]
            _check(d[i], "Helmholtz", 2 * i + par)
        for key, val in (("low", low), ("d", d), ("e", e), ("tail", t)):
            res[key].append(val)
    return res


def helmholtz_solve(fac, rhs):
    """solvers.py:100-126 (forward bidiagonal, back-substitution with one
    running tail sum)."""
    n_modes = len(fac["d"][0]) + len(fac["d"][1])
    if rhs.shape != (n_modes,) + tuple(fac["z2_shape"]):
        raise ValueError(f"rhs shape {rhs.shape} does not match "
                         f"{(n_modes,) + tuple(fac['z2_shape'])}")
    flat = rhs.reshape(n_modes, -1)
    out = np.empty_like(flat, dtype=np.result_type(flat, float))
    for par in (0, 1):
        low, d, e, tail = (fac[k][par] for k in ("low", "d", "e", "tail"))
        b = flat[par::2]
        n = b.shape[0]
        y = np.empty_like(b, dtype=np.result_type(b, float))
        y[0] = b[0]
        for i in range(1, n):
            y[i] = b[i] - low[i - 1] * y[i - 1]
        x = np.empty_like(y)
        x[n - 1] = y[n - 1] / d[n - 1]
        if n > 1:
            x[n - 2] = (y[n - 2] - e[n - 2] * x[n - 1]) / d[n - 2]
        run = np.zeros_like(x[0])
        for i in range(n - 3, -1, -1):
            run = run + x[i + 2]
            x[i] = (y[i] - e[i] * x[i + 1] - tail[i] * run) / d[i]
        out[par::2] = x
    return out.reshape(rhs.shape)


# ---------------------------------------------------------------- biharmonic

def biharmonic_bands(mats, xi0, xi1, xi2):
    """Banded entries of the operator; solvers.py:244-268."""
    nb = mats.n_bih
    p, q, r, s = _tail_factors(nb)
    q0 = mats.fourth_bih.diag
    ar_m2 = -mats.stiff_bih.diagonal(-2)
    ar_0 = -mats.stiff_bih.diagonal(0)
    ar_2 = -mats.stiff_bih.diagonal(2)
    bb0 = mats.mass_bih.diagonal(0)
    bb2 = mats.mass_bih.diagonal(2)
    bb4 = mats.mass_bih.diagonal(4)
    h = {"m4": xi2 * bb4[:, None],
         "m2": xi1 * ar_m2[:, None] + xi2 * bb2[:, None],
         "d0": xi0 * q0[:, None] + xi1 * ar_0[:, None] + xi2 * bb0[:, None]}
    tail2 = p[:nb - 2] * q[2:] + r[:nb - 2] * s[2:]
    h["p2"] = xi0 * tail2[:, None] + np.zeros((nb - 2, np.size(xi1)))
    h["p2"][:len(ar_2)] += xi1 * ar_2[:, None]
    h["p2"][:len(bb2)] += xi2 * bb2[:, None]
    tail4 = p[:nb - 4] * q[4:] + r[:nb - 4] * s[4:]
    h["p4"] = xi0 * tail4[:, None] + np.zeros((nb - 4, np.size(xi1)))
    h["p4"][:len(bb4)] += xi2 * bb4[:, None]
    return h, p, q, r, s


def _tail_factors(n):
    """matrices.py:163-170"""
    k = np.arange(n, dtype=float)
    return (8 * k * (k + 1) * (k + 2) * (k + 4) * np.pi, 1.0 / (k + 3),
            24 * (k + 1) * (k + 2) * np.pi, (k + 2) ** 2 / (k + 3))


def biharmonic_factor(mats, nu, dt, z2):
    """Alg. 2+3 fused elimination; solvers.py:271-355."""
    z2 = np.asarray(z2, dtype=float)
    xi0, xi1, xi2 = biharmonic_coefficients(nu, dt, z2)
    x1 = np.atleast_1d(xi1).reshape(-1)
    x2 = np.atleast_1d(xi2).reshape(-1)
    nb = mats.n_bih
    h, p, q, r, s = biharmonic_bands(mats, xi0, x1, x2)
    batch = x1.size
    res = {k: [] for k in ("low2", "low4", "d", "e", "f", "a", "b")}
    res.update(xi0=float(xi0), q=q, s=s, z2_shape=np.shape(z2))
    for par in (0, 1):
        k = np.arange(par, nb, 2)
        n = k.size

        def band(name, off):
            out = np.zeros((n, batch))
            if off >= 0:
                rows = k[k + 2 * off <= nb - 1]
                idx = rows
            else:
                rows = k[k + 2 * off >= 0]
                idx = rows + 2 * off
            out[(rows - par) // 2] = h[name][idx]
            return out

        hd, hp2, hp4, hm2, hm4 = (band("d0", 0), band("p2", 1), band("p4", 2),
                                  band("m2", -1), band("m4", -2))
        d = np.empty((n, batch))
        e = np.zeros((n, batch))
        f = np.zeros((n, batch))
        av = np.empty((n, batch))
        bv = np.empty((n, batch))
        low2 = np.zeros((max(n - 1, 0), batch))
        low4 = np.zeros((max(n - 2, 0), batch))
        for i in range(n):
            kk = k[i]
            in2 = kk + 2 <= nb - 1
            in4 = kk + 4 <= nb - 1
            if i >= 2:
                l4 = hm4[i] / d[i - 2]
                tmp = hm2[i] - l4 * e[i - 2]
                l2 = tmp / d[i - 1]
                low4[i - 2] = l4
                low2[i - 1] = l2
                u42 = xi0 * (av[i - 2] * q[kk + 2] + bv[i - 2] * s[kk + 2]) if in2 else 0.0
                u44 = xi0 * (av[i - 2] * q[kk + 4] + bv[i - 2] * s[kk + 4]) if in4 else 0.0
                u24 = xi0 * (av[i - 1] * q[kk + 4] + bv[i - 1] * s[kk + 4]) if in4 else 0.0
                d[i] = hd[i] - l4 * f[i - 2] - l2 * e[i - 1]
                e[i] = hp2[i] - l4 * u42 - l2 * f[i - 1]
                f[i] = hp4[i] - l4 * u44 - l2 * u24
                av[i] = p[kk] - l2 * av[i - 1] - l4 * av[i - 2]
                bv[i] = r[kk] - l2 * bv[i - 1] - l4 * bv[i - 2]
            elif i == 1:
                l2 = hm2[i] / d[i - 1]
                low2[i - 1] = l2
                u24 = xi0 * (av[i - 1] * q[kk + 4] + bv[i - 1] * s[kk + 4]) if in4 else 0.0
                d[i] = hd[i] - l2 * e[i - 1]
                e[i] = hp2[i] - l2 * f[i - 1]
                f[i] = hp4[i] - l2 * u24
                av[i] = p[kk] - l2 * av[i - 1]
                bv[i] = r[kk] - l2 * bv[i - 1]
            else:
                d[i], e[i], f[i] = hd[i], hp2[i], hp4[i]
                av[i], bv[i] = p[kk], r[kk]
            _check(d[i], "biharmonic", kk)
        for key, val in (("low2", low2), ("low4", low4), ("d", d), ("e", e),
                         ("f", f), ("a", av), ("b", bv)):
            res[key].append(val)
    return res


def biharmonic_solve(fac, rhs):
    """Alg. 4; solvers.py:162-198."""
    n_modes = len(fac["d"][0]) + len(fac["d"][1])
    if rhs.shape != (n_modes,) + tuple(fac["z2_shape"]):
        raise ValueError(f"rhs shape {rhs.shape} does not match "
                         f"{(n_modes,) + tuple(fac['z2_shape'])}")
    flat = rhs.reshape(n_modes, -1)
    out = np.empty_like(flat, dtype=np.result_type(flat, float))
    xi0 = fac["xi0"]
    for par in (0, 1):
        low2, low4, d, e, f, a, b = (fac[k][par] for k in
                                     ("low2", "low4", "d", "e", "f", "a", "b"))
        q, s = fac["q"][par::2], fac["s"][par::2]
        rr = flat[par::2]
        n = rr.shape[0]
        y = np.empty_like(rr, dtype=np.result_type(rr, float))
        y[0] = rr[0]
        if n > 1:
            y[1] = rr[1] - low2[0] * y[0]
        for i in range(2, n):
            y[i] = rr[i] - low2[i - 1] * y[i - 1] - low4[i - 2] * y[i - 2]
        x = np.empty_like(y)
        sq = np.zeros_like(y[0])
        ss = np.zeros_like(y[0])
        for i in range(n - 1, -1, -1):
            acc = y[i]
            if i + 1 < n:
                acc = acc - e[i] * x[i + 1]
            if i + 2 < n:
                acc = acc - f[i] * x[i + 2]
            if i + 3 < n:
                sq = sq + q[i + 3] * x[i + 3]
                ss = ss + s[i + 3] * x[i + 3]
                acc = acc - xi0 * (a[i] * sq + b[i] * ss)
            x[i] = acc / d[i]
        out[par::2] = x
    return out.reshape(rhs.shape)


# ---------------------------------------------------------------- dense checks

def dense_helmholtz(mats, nu, dt, z2):
    """solvers.py:361-363"""
    ca, cb = helmholtz_coefficients(nu, dt, float(z2))
    return ca * mats.stiff_dir.dense() + cb * mats.mass_dir.dense()


def dense_biharmonic(mats, nu, dt, z2):
    """solvers.py:366-369"""
    xi0, xi1, xi2 = biharmonic_coefficients(nu, dt, float(z2))
    return xi0 * mats.fourth_bih.dense() - xi1 * mats.stiff_bih.dense() + xi2 * mats.mass_bih.dense()


def residual_longdouble(dense, x, f):
    """||M x - f||_2 / ||f||_2 with the product evaluated in 80-bit long
    double (the fp64 structured apply alone sits at 1.4e-12
    for the biharmonic at cfg4 extremes)."""
    m = np.asarray(dense, dtype=np.longdouble)
    if np.iscomplexobj(x):
        xr = np.asarray(x.real, dtype=np.longdouble)
        xi = np.asarray(x.imag, dtype=np.longdouble)
        rr = m @ xr - np.asarray(f.real, dtype=np.longdouble)
        ri = m @ xi - np.asarray(f.imag, dtype=np.longdouble)
        num = np.sqrt(np.sum(rr * rr + ri * ri, axis=0))
        den = np.sqrt(np.sum(np.asarray(np.abs(f), dtype=np.longdouble) ** 2, axis=0))
    else:
        r = m @ np.asarray(x, dtype=np.longdouble) - np.asarray(f, dtype=np.longdouble)
        num = np.sqrt(np.sum(r * r, axis=0))
        den = np.sqrt(np.sum(np.asarray(f, dtype=np.longdouble) ** 2, axis=0))
    return np.asarray(num / den, dtype=float)


def max_rel_per_system(got, want):
    """Per-system max|got-want| / max|want| (tests/test_solvers.py:41-43
    idiom), systems along every axis but the first."""
    g = got.reshape(got.shape[0], -1)
    w = want.reshape(want.shape[0], -1)
    return np.abs(g - w).max(axis=0) / np.maximum(np.abs(w).max(axis=0), np.finfo(float).tiny)


# ---------------------------------------------------------------- transforms

def chebyshev_scalar(values, family_gl):
    """transforms.py:81-86"""
    n_pts = values.shape[0]
    if not family_gl:
        return sfft.dct(values, type=2, axis=0) * (np.pi / (2 * n_pts))
    return sfft.dct(values, type=1, axis=0) * (np.pi / (2 * (n_pts - 1)))


def shen_scalar(values, family_gl, space):
    """transforms.py:89-110; space 0 = Chebyshev, 1 = Dirichlet, 2 = biharmonic."""
    w = chebyshev_scalar(values, family_gl)
    n_x = values.shape[0] - 1
    if space == 0:
        y = w * (2.0 / np.pi)
        y[0] /= 2
        if family_gl:
            y[n_x] /= 2
        return y
    if space == 1:
        return w[:n_x - 1] - w[2:n_x + 1]
    k = np.arange(n_x - 3, dtype=float)
    sh = (-1,) + (1,) * (w.ndim - 1)
    c2 = (2 * (k + 2) / (k + 3)).reshape(sh)
    c4 = ((k + 1) / (k + 3)).reshape(sh)
    return w[:n_x - 3] - c2 * w[2:n_x - 1] + c4 * w[4:n_x + 1]


def shen_expand(coeffs, space, n_x):
    """transforms.py:113-126"""
    out = np.zeros((n_x + 1,) + coeffs.shape[1:], dtype=coeffs.dtype)
    n = coeffs.shape[0]
    out[:n] = coeffs
    if space == 1:
        out[2:n + 2] -= coeffs
    elif space == 2:
        k = np.arange(n, dtype=float)
        sh = (-1,) + (1,) * (coeffs.ndim - 1)
        out[2:n + 2] -= (2 * (k + 2) / (k + 3)).reshape(sh) * coeffs
        out[4:n + 4] += ((k + 1) / (k + 3)).reshape(sh) * coeffs
    return out


def chebyshev_evaluate(coeffs, family_gl):
    """transforms.py:129-137"""
    if not family_gl:
        return sfft.dct(coeffs, type=3, axis=0) / 2 + coeffs[0] / 2
    n_x = coeffs.shape[0] - 1
    y = sfft.dct(coeffs, type=1, axis=0) / 2 + coeffs[0] / 2
    sg = ((-1.0) ** np.arange(n_x + 1)).reshape((-1,) + (1,) * (coeffs.ndim - 1))
    return y + sg * coeffs[n_x] / 2


def mass_cholesky(mats, space):
    """Per-parity upper banded Cholesky factors of the mass matrix
    (transforms.py:143-160; LAPACK dpbtrf via scipy)."""
    full, nband = (mats.mass_dir, 1) if space == 1 else (mats.mass_bih, 2)
    dense = full.dense()
    out = []
    for par in (0, 1):
        sub = dense[par::2, par::2]
        m = sub.shape[0]
        ab = np.zeros((nband + 1, m))
        for b in range(nband + 1):
            ab[nband - b, b:] = np.diag(sub, b)
        out.append(cholesky_banded(ab, lower=False))
    return tuple(out)


def mass_solve(scalar, space, mats):
    """transforms.py:163-175 (per-parity cho_solve_banded)."""
    if space == 0:
        raise ValueError("Chebyshev mass solve is a rescale; see shen_scalar")
    fac = mass_cholesky(mats, space)
    out = np.empty_like(scalar, dtype=np.result_type(scalar, float))
    for par in (0, 1):
        rhs = scalar[par::2]
        flat = rhs.reshape(rhs.shape[0], -1)
        out[par::2] = cho_solve_banded((fac[par], False), flat).reshape(rhs.shape)
    return out


def forward_transform(data, space, family_gl, mats):
    """transforms.py:181-188: physical (n_x+1, n_y, n_z) -> coefficients."""
    fourier = sfft.rfftn(data, axes=(1, 2))
    scal = shen_scalar(fourier, family_gl, space)
    if space != 0:
        scal = mass_solve(scal, space, mats)
    return scal


def forward_scalar_product(data, space, family_gl):
    """transforms.py:191-196"""
    return shen_scalar(sfft.rfftn(data, axes=(1, 2)), family_gl, space)


def inverse_transform(coeffs, space, family_gl, n_x, n_y, n_z):
    """transforms.py:199-205"""
    cheb = shen_expand(coeffs, space, n_x)
    lines = chebyshev_evaluate(cheb, family_gl)
    return sfft.irfftn(lines, s=(n_y, n_z), axes=(1, 2))


# ---------------------------------------------------------------- stepper right-hand sides

def ab2(h_curr, h_prev):
    """stepper.py:189-191"""
    return tuple(1.5 * c - 0.5 * p for c, p in zip(h_curr, h_prev))


def assemble_rhs_u(mats, nu, dt, z2, m, n, u, h_ab):
    """stepper.py:193-207 (m, n, z2 as the stepper holds them)."""
    rhs = (nu * dt / 2) * mats.fourth_bih.apply(u)
    rhs -= (1 - nu * dt * z2) * mats.stiff_bih.apply(u)
    rhs += (-z2 + nu * dt * z2 ** 2 / 2) * mats.mass_bih.apply(u)
    h_x, h_y, h_z = h_ab
    rhs -= dt * z2 * mats.mixed_mass.apply(h_x)
    rhs -= dt * 1j * m * mats.deriv_dir_to_bih.apply(h_y)
    rhs -= dt * 1j * n * mats.deriv_dir_to_bih.apply(h_z)
    return rhs


def assemble_rhs_g(mats, nu, dt, z2, m, n, g, h_ab):
    """stepper.py:209-219"""
    rhs = -(nu * dt / 2) * mats.stiff_dir.apply(g)
    rhs += (1 - nu * dt * z2 / 2) * mats.mass_dir.apply(g)
    _, h_y, h_z = h_ab
    src = 1j * m * h_z - 1j * n * h_y
    rhs += dt * mats.mass_dir.apply(src)
    return rhs


def compute_nonlinear(mats, family_gl, n_y, n_z, m, n, mask, u_hat, v_hat, w_hat, g_hat):
    """stepper.py:148-185: Dirichlet coefficients of H = u x omega, masked.
    m, n, mask as the stepper holds them ((n_y, 1), (1, n_z//2+1), plane)."""
    n_x = mats.n_x
    mass_inv = 1.0 / mats.mass_cheb

    def ddx(d):
        c = mats.deriv_dir_to_cheb.apply(d)
        c *= mass_inv.reshape(-1, 1, 1)
        return c

    def inv(c, sp):
        return inverse_transform(c, sp, family_gl, n_x, n_y, n_z)

    u = inv(u_hat, 2)
    v = inv(v_hat, 1)
    w = inv(w_hat, 1)
    om_x = inv(g_hat, 1)
    dv_dx = inv(ddx(v_hat), 0)
    dw_dx = inv(ddx(w_hat), 0)
    du_dy = inv(1j * m * u_hat, 2)
    du_dz = inv(1j * n * u_hat, 2)
    om_y = du_dz - dw_dx
    om_z = dv_dx - du_dy
    h_x = v * om_z - w * om_y
    h_y = w * om_x - u * om_z
    h_z = u * om_y - v * om_x
    out = []
    for h in (h_x, h_y, h_z):
        c = forward_transform(h, 1, family_gl, mats)
        c *= mask
        out.append(c)
    return tuple(out)


def recover_velocity(mats, z2, m, n, u_new, g_new):
    """stepper.py:296-303: divergence variable f = mass_solve(D u) and the
    horizontal velocities (the mean mode (m = n = 0) is overwritten by the
    stepper's mean-flow solve afterwards)."""
    f_scal = mats.deriv_bih_to_dir.apply(u_new)
    f_hat = mass_solve(f_scal, 1, mats)
    safe_z2 = np.where(z2 > 0, z2, 1.0)
    v_new = (1j * m * f_hat + 1j * n * g_new) / safe_z2
    w_new = (1j * n * f_hat - 1j * m * g_new) / safe_z2
    return v_new, w_new
