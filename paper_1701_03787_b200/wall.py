"""Plans for the fused wall-normal transform kernel (csrc/shen_wall.cu).

The kernel does the whole axis-0 stage of the reference's 3-D transforms
(transforms.py:81-205) for a tile of Fourier lines in shared memory.  Its
DCTs are complex DFTs of one sequence per line:

* Gauss points (``dct`` type 2 / 3): Makhoul's reordering, DFT length N;
* Gauss-Lobatto points (``dct`` type 1): the even extension, DFT length 2 n_x.

A DFT of length Ld runs as one of

* ``KIND_POW2``  -- Ld a power of two: the FFT itself;
* ``KIND_RADER`` -- Ld prime with Ld - 1 a power of two (N = 257 at BASELINE
  config 3): Rader's cyclic convolution of length Ld - 1;
* ``KIND_BLUESTEIN`` -- otherwise: Bluestein's chirp convolution on the
  smallest power of two >= 2 Ld - 1.

The FFT is a sequence of decimation-in-frequency passes of radix 16/8/4/2
that leaves the spectrum in digit-reversed order (``digit_reversal``);
convolution kernels are stored in that order and scaled by 1/M, and the
mirrored decimation-in-time passes bring the convolution back to natural
order.  ``emulate`` is a numpy model of exactly that pass sequence, used by
the CPU tests to pin every table before the device runs it.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

__all__ = ["plan_tables", "WallPlan", "wall_plan", "emulate_dft", "digit_reversal", "stages_for", "KIND_POW2",
           "KIND_RADER", "KIND_BLUESTEIN"]

KIND_POW2, KIND_RADER, KIND_BLUESTEIN = 0, 1, 2
THREADS = 256          # kernel block size (csrc/shen_wall.cu kWallThreads)
ITEMS_MAX = 24         # register-staged rows per thread (launch_wall)
SMEM_MAX = 200 * 1024  # shared-memory budget per CTA for the plan's tile


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    f = 2
    while f * f <= n:
        if n % f == 0:
            return False
        f += 1
    return True


def primitive_root(p: int) -> int:
    """Smallest generator of the multiplicative group mod the prime p."""
    if p == 2:
        return 1
    phi = p - 1
    fac = []
    n, f = phi, 2
    while f * f <= n:
        if n % f == 0:
            fac.append(f)
            while n % f == 0:
                n //= f
        f += 1
    if n > 1:
        fac.append(n)
    for g in range(2, p):
        if all(pow(g, phi // q, p) != 1 for q in fac):
            return g
    raise ValueError(p)


def stages_for(M: int) -> list:
    """Radix of each pass: radix 16 first (the first and last passes bound
    the lines a CTA can take: M / R1 butterflies per line), the remaining
    bits in balanced passes of at most 4 bits."""
    m = M.bit_length() - 1
    if m == 0:
        return [1]
    first = min(4, m)
    rest = m - first
    if rest == 0:
        return [2 ** first]
    nst = -(-rest // 4)
    base, extra = divmod(rest, nst)
    return [2 ** first] + [2 ** (base + 1)] * extra + [2 ** base] * (nst - extra)


def digit_reversal(radices) -> np.ndarray:
    """rho[p] = frequency held at position p after the DIF passes."""
    M = int(np.prod(radices))
    if len(radices) == 0 or M == 1:
        return np.zeros(1, dtype=np.int64)
    R = radices[0]
    q = M // R
    sub = digit_reversal(radices[1:]) if len(radices) > 1 else np.zeros(1, dtype=np.int64)
    p = np.arange(M)
    k2, pp = p // q, p % q
    return k2 + R * sub[pp]


def _twiddles(M: int) -> np.ndarray:
    k = np.arange(M, dtype=np.longdouble)
    ang = -2 * np.arccos(np.longdouble(-1)) * k / M
    return (np.cos(ang).astype(np.float64) + 1j * np.sin(ang).astype(np.float64)).astype(np.complex128)


def _expi_ld(num: np.ndarray, den: int) -> np.ndarray:
    """exp(-i pi num / den) evaluated in long double, rounded to complex128."""
    ang = -np.arccos(np.longdouble(-1)) * np.asarray(num, dtype=np.longdouble) / den
    return (np.cos(ang).astype(np.float64) + 1j * np.sin(ang).astype(np.float64)).astype(np.complex128)


def emulate_dft(a: np.ndarray, radices) -> np.ndarray:
    """numpy model of the kernel's DIF pass sequence: natural-order input
    (M, ...) -> spectrum in digit-reversed order (pass_dif, shen_wall.cu)."""
    M = a.shape[0]
    tw = _twiddles(M)
    T = a.astype(np.complex128).copy()
    Ls = M
    for R in radices:
        q = Ls // R
        out = T.copy()
        for blk in range(M // Ls):
            for n1 in range(q):
                base = blk * Ls + n1
                idx = base + q * np.arange(R)
                v = np.fft.fft(T[idx], axis=0)
                if q > 1:
                    k = np.arange(R)
                    v = v * tw[(n1 * k * (M // Ls)) % M].reshape((-1,) + (1,) * (T.ndim - 1))
                out[idx] = v
        T = out
        Ls = q
    return T


def _sigma(N: int) -> np.ndarray:
    """Makhoul's reordering for the Gauss DCT: v_i = x_sigma(i)."""
    i = np.arange(N)
    h = (N + 1) // 2
    return np.where(i < h, 2 * i, 2 * (N - 1 - i) + 1)


@lru_cache(maxsize=64)
def plan_tables(n_x: int, fam: int):
    """Host tables shared by every (space, direction) of one (n_x, family)."""
    N = n_x + 1
    Ld = N if fam == 0 else 2 * n_x
    if fam == 1 and _is_pow2(Ld):
        kind, M = KIND_POW2, Ld
    elif fam == 0 and _is_prime(N) and _is_pow2(N - 1) and N > 2:
        kind, M = KIND_RADER, N - 1
    else:
        kind = KIND_BLUESTEIN
        M = 1
        while M < 2 * Ld - 1:
            M *= 2
    radices = stages_for(M)
    rho = digit_reversal(radices)
    t = {"N": N, "Ld": Ld, "kind": kind, "M": M, "radices": radices, "tw": _twiddles(M)}
    if kind == KIND_POW2:
        pinv = np.empty(M, dtype=np.int32)
        pinv[rho] = np.arange(M, dtype=np.int32)
        t["pinv"] = pinv
    elif kind == KIND_RADER:
        g = primitive_root(N)
        p = np.arange(M)
        gp = np.array([pow(g, int(i), N) for i in p], dtype=np.int64)
        gneg = np.array([pow(g, (-int(i)) % (N - 1), N) for i in p], dtype=np.int64)
        t["gin_f"] = _sigma(N)[gp].astype(np.int32)
        t["gin_i"] = gp.astype(np.int32)
        t["gout"] = gneg.astype(np.int32)
        # b_m = W_N^{g^{-m}} (forward), conjugate for the inverse DFT
        b = _expi_ld(2 * gneg, N)
        t["ker_f"] = (np.fft.fft(b) / M)[rho]
        t["ker_i"] = (np.fft.fft(np.conj(b)) / M)[rho]
    else:
        n = np.arange(Ld, dtype=np.int64)
        c = _expi_ld((n * n) % (2 * Ld), Ld)  # exp(-i pi n^2 / Ld)
        h = np.zeros(M, dtype=np.complex128)
        h[:Ld] = np.conj(c)
        h[M - Ld + 1:] = np.conj(c[1:])[::-1]
        t["chirp_f"], t["chirp_i"] = c, np.conj(c)
        t["ker_f"] = (np.fft.fft(h) / M)[rho]
        t["ker_i"] = (np.fft.fft(np.conj(h)) / M)[rho]
    if fam == 0:
        t["mk"] = _expi_ld(np.arange(N), 2 * N)  # exp(-i pi k / 2N)
    def boxed(r):  # rows covered by the fewest TMA boxes of <= 256 rows, 8-row multiples (launch_wall)
        nb = -(-r // 256)
        return nb * ((-(-r // nb) + 7) // 8 * 8)

    rows = max(N + 2, M, boxed(N), boxed(max(n_x - 3, 1)), boxed(max(n_x - 1, 1)))
    R1 = radices[0]
    TLs = 4
    while TLs > 0 and ((M // R1) << TLs > THREADS or (rows + 2) * (16 << TLs) > SMEM_MAX
                       or -(-(N << TLs) // THREADS) > ITEMS_MAX or (TLs > 3 and (rows + 2) * (16 << TLs) > 110 * 1024)):
        TLs -= 1
    t["log2_lines"] = TLs
    t["rows_smem"] = rows
    t["fits"] = ((M // R1) << TLs) <= THREADS and (rows + 2) * (16 << TLs) <= 227 * 1024 and \
        -(-(N << TLs) // THREADS) <= ITEMS_MAX
    return t


def stencil_tables(n_x: int):
    """Biharmonic stencil c2, c4 as the reference evaluates them (transforms.py:104-106)."""
    k = np.arange(max(n_x - 3, 0), dtype=float)
    return 2 * (k + 2) / (k + 3), (k + 1) / (k + 3)


def mass_tables(packed: np.ndarray, nband: int, space: int, n_x: int) -> np.ndarray:
    """Per parity and row i of the mass solve, [2][mmax + 1][8]:
    a0 = 1/U_ii, a2 = c2_k/U_ii, a4 = c4_k/U_ii (the Shen stencil of row k =
    par + 2 i folded in; Dirichlet: c2 = 1, c4 = 0), f1 = U_{i-1,i}/U_ii,
    f2 = U_{i-2,i}/U_ii (forward sweep U^T y = s), g1 = U_{i,i+1}/U_ii,
    g2 = U_{i,i+2}/U_ii (backward U x = y), 0; from the LAPACK upper band
    storage of the reference's factors.  One zero row past the end (the
    kernel loads one row ahead)."""
    mmax = packed.shape[2]
    out = np.zeros((2, mmax + 1, 8))
    if space == 2:
        c2, c4 = stencil_tables(n_x)
    n = n_x - 1 if space == 1 else n_x - 3
    for par in (0, 1):
        ab = packed[par]
        m = (n - par + 1) // 2
        diag = ab[nband, :m]
        r = 1.0 / diag
        u1 = ab[nband - 1, :m]                   # U_{i-1,i} at column i
        u2 = ab[0, :m] if nband == 2 else np.zeros(m)
        k = par + 2 * np.arange(m)
        out[par, :m, 0] = r
        out[par, :m, 1] = (c2[k] if space == 2 else 1.0) * r
        out[par, :m, 2] = (c4[k] if space == 2 else 0.0) * r
        out[par, :m, 3] = u1 * r
        out[par, :m, 4] = u2 * r
        out[par, :m - 1, 5] = u1[1:] * r[:-1]
        if nband == 2:
            out[par, :m - 2, 6] = u2[2:] * r[:-2]
    return out


class WallPlan:
    """A device-resident plan: the ctypes struct plus the tensors it points to."""

    def __init__(self, struct, keep):
        self.struct = struct
        self._keep = keep


_DEV_PLANS = {}


def wall_plan(n_x: int, fam: int, space: int, direction: int, mass: bool, scale: float, rowscale=None,
              rowscale_key=None):
    """Device plan for ``shen_wall_transform``.  Returns None if the size does
    not fit the kernel's shared-memory tile (the caller falls back).
    ``rowscale`` (inverse, Chebyshev space): per-coefficient factors applied
    first, cached under ``rowscale_key`` (e.g. 1/mass_cheb for d/dx)."""
    import torch

    from . import _lib
    from ._device import device

    dev = device()
    key = (n_x, fam, space, direction, bool(mass), float(scale), rowscale_key, dev.index)
    pl = _DEV_PLANS.get(key)
    if pl is not None:
        return pl
    t = plan_tables(n_x, fam)
    if not t["fits"]:
        return None
    N = t["N"]
    keep = []

    def dptr(a, dtype):
        if a is None:
            return None
        ten = torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(dev)
        keep.append(ten)
        return ten.data_ptr()

    s = _lib.ShenWallPlan()
    s.direction, s.family, s.space = direction, fam, space
    s.mass = int(bool(mass) and direction == 0 and space in (1, 2))
    s.N = N
    n_modes = {0: N, 1: n_x - 1, 2: n_x - 3, 3: N}[space]
    s.n_out = n_modes if direction == 0 else N
    s.n_in = N if direction == 0 else n_modes
    s.kind, s.Ld, s.M = t["kind"], t["Ld"], t["M"]
    s.nstage = len(t["radices"])
    for i, r in enumerate(t["radices"]):
        s.radix[i] = r
    s.log2_lines, s.rows_smem = t["log2_lines"], t["rows_smem"]
    s.scale = float(scale)
    s.tw = dptr(t["tw"], np.complex128)
    s.ker_f = dptr(t.get("ker_f"), np.complex128)
    s.ker_i = dptr(t.get("ker_i"), np.complex128)
    s.chirp_f = dptr(t.get("chirp_f"), np.complex128)
    s.chirp_i = dptr(t.get("chirp_i"), np.complex128)
    s.gin_f = dptr(t.get("gin_f"), np.int32)
    s.gin_i = dptr(t.get("gin_i"), np.int32)
    s.gout = dptr(t.get("gout"), np.int32)
    s.pinv = dptr(t.get("pinv"), np.int32)
    s.mk = dptr(t.get("mk"), np.complex128)
    if space == 2:
        c2, c4 = stencil_tables(n_x)
        s.c2, s.c4 = dptr(c2, np.float64), dptr(c4, np.float64)
    s.nband, s.mmax = 0, 0
    if direction == 0 and mass and space in (1, 2):
        from .transforms import _mass_factors_host

        packed, nband, n, mmax, _ = _mass_factors_host(n_x, fam, space)
        s.nband, s.mmax = nband, mmax
        s.mfac = dptr(mass_tables(packed, nband, space, n_x), np.float64)
    if rowscale is not None:
        if direction != 1 or space != 0:
            raise ValueError("rowscale applies to inverse Chebyshev-space plans")
        s.rowscale = dptr(np.asarray(rowscale, dtype=np.float64).reshape(N), np.float64)
    pl = WallPlan(s, keep)
    _DEV_PLANS[key] = pl
    return pl


# ---------------------------------------------------------------- numpy model of the kernel

def _model_dft(x, t, inverse: bool):
    """Length-Ld DFT (inverse: sign +, unnormalised) of the gathered rows x
    (Ld, L) the way the kernel computes it, from the plan tables."""
    M, Ld, kind, rad = t["M"], t["Ld"], t["kind"], t["radices"]
    rho = digit_reversal(rad)

    def conv(a, ker):  # G(F(a) * ker): ker in digit-reversed order, / M
        P = emulate_dft(a, rad) * ker[:, None]
        nat = np.empty_like(P)
        nat[rho] = P
        return np.fft.ifft(nat, axis=0) * M

    if kind == KIND_POW2:
        a = np.conj(x) if inverse else x
        X = emulate_dft(a, rad)[t["pinv"]]
        return np.conj(X) if inverse else X
    if kind == KIND_RADER:
        a = x[t["gin_i"]]
        c = conv(a, t["ker_i"] if inverse else t["ker_f"])
        X = np.empty_like(x)
        X[t["gout"]] = x[0] + c
        X[0] = x[0] + a.sum(axis=0)
        return X
    chirp = t["chirp_i"] if inverse else t["chirp_f"]
    a = np.zeros((M,) + x.shape[1:], dtype=np.complex128)
    a[:Ld] = x * chirp[:, None]
    c = conv(a, t["ker_i"] if inverse else t["ker_f"])
    return c[:Ld] * chirp[:, None]


def emulate_wall(lines, n_x: int, fam: int, space: int, direction: int, mass: bool, scale: float):
    """numpy model of wall_forward_kernel / wall_inverse_kernel on (rows, L)
    complex lines (CPU tests pin the plan tables with it)."""
    t = plan_tables(n_x, fam)
    N = n_x + 1
    x = np.asarray(lines, dtype=np.complex128)
    if direction == 0:
        if fam == 0:
            V = _model_dft(x[_sigma(N)], t, False)
            Vn = np.conj(np.concatenate([V[:1], V[1:][::-1]]))
            mk = t["mk"][:, None]
            w = (mk * (V + Vn)).real + 1j * (mk * (V - Vn)).imag
        else:
            z = np.concatenate([x, x[1:-1][::-1]])
            w = _model_dft(z, t, False)[:N]
        w = w * scale
        if space == 1:
            s = w[:n_x - 1] - w[2:n_x + 1]
        elif space == 2:
            c2, c4 = stencil_tables(n_x)
            s = w[:n_x - 3] - c2[:, None] * w[2:n_x - 1] + c4[:, None] * w[4:n_x + 1]
        elif space == 0:
            s = w * (2.0 / np.pi)
            s[0] /= 2
            if fam == 1:
                s[n_x] /= 2
        else:
            s = w
        if mass and space in (1, 2):
            from scipy.linalg import cho_solve_banded

            from .transforms import _mass_factors_host

            facs = _mass_factors_host(n_x, fam, space)[4]
            out = np.empty_like(s)
            for par in (0, 1):
                out[par::2] = cho_solve_banded((facs[par], False), s[par::2])
            s = out
        return s
    n = x.shape[0]
    c = np.zeros((N,) + x.shape[1:], dtype=np.complex128)
    c[:n] = x
    if space == 1:
        c[2:n + 2] -= x
    elif space == 2:
        c2, c4 = stencil_tables(n_x)
        c[2:n + 2] -= c2[:n, None] * x
        c[4:n + 4] += c4[:n, None] * x
    if fam == 0:
        y = c.copy()
        y[0] *= 2
        yn = np.concatenate([np.zeros_like(y[:1]), y[1:][::-1]])
        V = np.conj(t["mk"])[:, None] * (y - 1j * yn) / 2
        X = _model_dft(V, t, True)
        f = np.empty_like(X)
        f[_sigma(N)] = X
        return f * scale
    e = c.copy()
    e[0] *= 2
    e[n_x] *= 2
    z = np.concatenate([e, e[1:-1][::-1]])
    return _model_dft(z, t, True)[:N] * (0.5 * scale)
