"""Drop-in replacement for ``chebchan.solvers`` running on a B200.

Same public surface as the reference module (``solvers.py:43-52``):
``helmholtz_coefficients``, ``biharmonic_coefficients``, ``build_helmholtz``,
``build_biharmonic``, ``HelmholtzLU``/``BiharmonicLU`` with ``.solve``,
``n_modes``, ``storage_vectors()`` and the per-parity factor attributes,
``ZeroPivotError``, ``solve_field`` and the dense test helpers.

What changes is where and how the work happens:

* ``build_*`` uploads z^2-derived coefficients and the 1-D row constants
  once, runs the factor recurrence on the device (one thread per
  wavenumber system and parity) and keeps only *chunk checkpoints* -- the
  factor state entering every chunk of R rows -- instead of the reference's
  4 (Helmholtz) or 7 (biharmonic) full factor vectors per system;
* ``solve`` (default ``method="stream"``) is the streaming fused
  factor+solve kernel (``csrc/shen_solve_stream.cu``): one thread per
  (system, parity), coalesced row pieces, the factors recomputed from the
  checkpoints in both sweeps (the biharmonic on mirror pairs of systems);
* the full factors ``low``/``d``/``e``/``tail`` (and ``low2`` ... ``b``) are
  materialised lazily, bit-identical to the reference, only when accessed;
* ``method="stored"`` keeps full reference-exact factors on the device and
  solves with the reference's operation order (bit-identical solutions).

Inputs are numpy arrays (copied to the device and back, result is numpy) or
torch CUDA tensors (zero-copy, result is a torch tensor).  There is no CPU
fallback: without the CUDA library or a device every call raises.
"""

from __future__ import annotations

import numpy as np

from . import _device as dv
from ._lib import check, lib, ptr_array
from .matrices import MatrixSet, tail_factors

__all__ = [
    "HelmholtzLU",
    "BiharmonicLU",
    "ZeroPivotError",
    "build_helmholtz",
    "build_biharmonic",
    "helmholtz_coefficients",
    "biharmonic_coefficients",
    "dense_helmholtz",
    "dense_biharmonic",
    "lu_nopivot",
    "solve_field",
    "solve_many",
    "chunk_rows_for",
]

PIVOT_FLOOR = 1e-300  # reference solvers.py:54
_INT_MAX = 2**31 - 1
_METHODS = ("stream", "stored")


def _env_int(name, default):
    import os

    return int(os.environ.get(name, default))


STREAM_ROWS_H = 8  # checkpoint spacing (rows) the streaming solve kernels are built for
STREAM_ROWS_B = 8


def stream_warps() -> int:
    """CTA size of the streaming solve in warps per SM (8 or 12; 0 = the
    per-operator default measured best at BASELINE config 4)."""
    import os

    return int(os.environ.get("SHEN_STREAM_WARPS", "0"))


# ------------------------------------------------------------------ host <-> device

def _solve_api(lu, rhs, out):
    import torch

    _check_rhs_shape(rhs, lu.n_modes, lu.z2_shape)
    if dv.is_torch(rhs) and rhs.is_cuda:
        r, cplx, _ = dv.as_rhs(rhs)
        flat = r.reshape(lu.n_modes, -1)
        if out is not None:
            # the kernels write n_modes x batch elements of r's dtype into out's storage
            if not (dv.is_torch(out) and out.is_cuda and out.device == r.device and out.dtype == r.dtype
                    and tuple(out.shape) == tuple(rhs.shape) and out.is_contiguous()):
                raise ValueError(f"out must be a contiguous CUDA tensor on {r.device} of dtype {r.dtype} "
                                 f"and shape {tuple(rhs.shape)}")
        res = torch.empty_like(flat) if out is None else out.view(lu.n_modes, -1)
        lu.solve_into(flat, res, cplx)
        return res.reshape(tuple(rhs.shape))
    a = rhs.numpy() if dv.is_torch(rhs) else np.asarray(rhs)
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    if out is None:
        out = np.empty(a.shape, dtype=a.dtype)
    elif out.shape != a.shape or out.dtype != a.dtype or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous {a.dtype} array of shape {a.shape}")
    if lu.batch == 0:
        return out
    _host_pipeline(lu, a.reshape(lu.n_modes, -1), out.reshape(lu.n_modes, -1), cplx)
    return out


_PIPE_MIN_SLAB = 4096
_PIPE_MAX_SLABS = _env_int("SHEN_PIPE_SLABS", 16)  # fewer slabs = longer first-copy-in / last-copy-out bubbles


def _host_pipeline(lu, h_rhs, h_out, cplx):
    _host_pipeline_many([(lu, h_rhs, h_out, cplx)])


_STREAMS = {}


def _pipe_streams(dev):
    import torch

    st = _STREAMS.get(dev)
    if st is None:
        st = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
        _STREAMS[dev] = st
    return st


def _host_pipeline_many(jobs):
    """Column-slab pipeline over one or several solves: the H2D copy of slab
    k+1 and the D2H copy of slab k-1 run on their own streams while slab k is
    solved (stream method; the stored method solves each batch after one copy).
    Consecutive jobs share the pipeline, so the next operator's first copy-in
    overlaps the previous one's last copy-out.  Page-locked host arrays make
    the copies asynchronous; pageable ones still work (staged)."""
    import torch

    dev = dv.device()
    s_in, s_out = _pipe_streams(dev)
    comp = torch.cuda.current_stream(dev)
    h = lib()
    s_in.wait_stream(comp)
    for lu, h_rhs, h_out, cplx in jobs:
        n, B = h_rhs.shape
        es = h_rhs.itemsize
        dtype = torch.complex128 if cplx else torch.float64
        cache = getattr(lu, "_pipe", None)
        if cache is None or cache[0].shape != (n, B) or cache[0].dtype != dtype:
            cache = (torch.empty((n, B), dtype=dtype, device=dev), torch.empty((n, B), dtype=dtype, device=dev))
            lu._pipe = cache
        d_rhs, d_out = cache
        if lu.method != "stream" or B < 2 * _PIPE_MIN_SLAB:
            bounds = [(0, B)]
        else:
            nslab = min(_PIPE_MAX_SLABS, B // _PIPE_MIN_SLAB)
            step = -(-B // nslab)
            step = -(-step // 128) * 128
            bounds = [(a, min(a + step, B)) for a in range(0, B, step)]
        pitch = B * es
        for a, b in bounds:
            ev_in = torch.cuda.Event()
            with torch.cuda.stream(s_in):
                check(h.shen_memcpy2d_async(d_rhs.data_ptr() + a * es, pitch, h_rhs.ctypes.data + a * es, pitch,
                                            (b - a) * es, n, 0, s_in.cuda_stream), "H2D slab")
                ev_in.record(s_in)
            comp.wait_event(ev_in)
            if len(bounds) == 1:
                lu.solve_into(d_rhs, d_out, cplx)
            else:
                lu.solve_into(d_rhs, d_out, cplx, a, b)
            ev_c = torch.cuda.Event()
            ev_c.record(comp)
            s_out.wait_event(ev_c)
            with torch.cuda.stream(s_out):
                check(h.shen_memcpy2d_async(h_out.ctypes.data + a * es, pitch, d_out.data_ptr() + a * es, pitch,
                                            (b - a) * es, n, 1, s_out.cuda_stream), "D2H slab")
    s_out.synchronize()


def solve_many(jobs):
    """Solve several (lu, rhs[, out]) at once -- e.g. the Helmholtz and the
    biharmonic right-hand sides of a time step.  Same results as calling
    ``lu.solve(rhs, out)`` for each; with host arrays the solves share one
    copy/compute pipeline (no drain between operators).  Returns the outputs."""
    host, outs = [], []
    for job in jobs:
        lu, rhs = job[0], job[1]
        out = job[2] if len(job) > 2 else None
        if dv.is_torch(rhs) and rhs.is_cuda:
            outs.append(_solve_api(lu, rhs, out))
            continue
        _check_rhs_shape(rhs, lu.n_modes, lu.z2_shape)
        a = rhs.numpy() if dv.is_torch(rhs) else np.asarray(rhs)
        cplx = np.iscomplexobj(a)
        a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
        if out is None:
            out = np.empty(a.shape, dtype=a.dtype)
        elif out.shape != a.shape or out.dtype != a.dtype or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous {a.dtype} array of shape {a.shape}")
        outs.append(out)
        if lu.batch > 0:
            host.append((lu, a.reshape(lu.n_modes, -1), out.reshape(lu.n_modes, -1), cplx))
    if host:
        _host_pipeline_many(host)
    return outs


MIRROR_PAIRS = _env_int("SHEN_PAIRS", 1)  # solve mirror-paired systems together (biharmonic stream)
PAIRS_MIN = _env_int("SHEN_PAIRS_MIN", 8192)  # below: one system per thread (c1: 40 vs 33 us; c3 pairs: 0.097 vs 0.120 ms)

def mirror_pairs(z2):
    """Pairs of systems with bitwise-identical z2 rows (the channel grid's
    (m, n) / (-m, n) wavenumbers), as an int64 (2, P) array over the
    flattened z2, or None.  Rows of a 2-D z2 that are byte-identical are
    paired up; unpaired rows become self-pairs.  Items of one row pair are
    consecutive, so a warp's 32 lanes read coalesced row pieces of both
    systems."""
    z2 = np.asarray(z2, dtype=float)
    if z2.ndim != 2 or z2.shape[0] < 2 or z2.shape[1] < 1:
        return None
    rows, cols = z2.shape
    groups = {}
    for r in range(rows):
        groups.setdefault(z2[r].tobytes(), []).append(r)
    pairs_r = []
    for members in groups.values():
        for k in range(0, len(members) - 1, 2):
            pairs_r.append((members[k], members[k + 1]))
        if len(members) % 2:
            pairs_r.append((members[-1], members[-1]))
    if sum(a != b for a, b in pairs_r) * 2 < rows // 2:  # too few pairs to pay
        return None
    pairs_r.sort()
    n = np.arange(cols, dtype=np.int64)
    a = np.concatenate([r0 * cols + n for r0, _ in pairs_r])
    b = np.concatenate([r1 * cols + n for _, r1 in pairs_r])
    return np.stack([a, b])


def _solve_real_via_complex(lu, rhs_dev, out_dev, j0=0, j1=-1):
    """Real RHS with an odd batch or misaligned storage: the streaming kernels
    move 16-B row pieces, so solve the complex system with zero
    imaginary part -- every coefficient is real, so the real part is the same
    arithmetic as the real solve."""
    import torch

    if rhs_dev.is_complex():
        z = rhs_dev.clone()
    else:
        z = torch.complex(rhs_dev, torch.zeros_like(rhs_dev)).contiguous()
    xz = torch.empty_like(z)
    lu.solve_into(z, xz, True, j0, j1)
    hi = xz.shape[1] if j1 < 0 else j1
    src = xz[:, j0:hi]
    out_dev[:, j0:hi].copy_(src if out_dev.is_complex() else src.real)
    return out_dev


def _scratch(lu, op, n_modes, batch, is_complex, device):
    """Per-LU cached device scratch of the streaming solve (y checkpoints)."""
    import torch

    nbytes = int(lib().shen_stream_scratch_bytes(op, n_modes, lu.chunk_rows, batch, int(is_complex)))
    buf = getattr(lu, "_scratch_buf", None)
    if buf is None or buf.numel() < nbytes or buf.device != device:
        buf = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
        lu._scratch_buf = buf
    return buf.data_ptr()


class ZeroPivotError(ArithmeticError):
    """Unpivoted elimination met a vanishing pivot (reference solvers.py:57-58)."""


def helmholtz_coefficients(nu: float, dt: float, z2):
    """(ca, cb) = (nu*dt/2, 1 + nu*dt*z2/2)  (reference solvers.py:67-69)."""
    return nu * dt / 2, 1 + nu * dt * np.asarray(z2, dtype=float) / 2


def biharmonic_coefficients(nu: float, dt: float, z2):
    """(xi0, xi1, xi2) (reference solvers.py:72-75)."""
    z2 = np.asarray(z2, dtype=float)
    return -nu * dt / 2, 1 + nu * dt * z2, -(2 * z2 + nu * dt * z2 ** 2) / 2


def chunk_rows_for(n_modes: int) -> int:
    """Rows per lane (a power of two, compile-time in the kernels) so that 32
    lanes cover the larger parity."""
    rows0 = (n_modes + 1) // 2
    need = max(1, -(-rows0 // 32))
    R = 1
    while R < need:
        R *= 2
    if R > 32:
        raise ValueError(f"n_modes = {n_modes} exceeds the supported 2048 rows per parity")
    return R


def _n_chunks(n_modes: int, R: int) -> int:
    return -(-((n_modes + 1) // 2) // R)


def _raise_pivot(piv, what: str):
    if piv[0] != _INT_MAX:
        row = 2 * int(piv[0])
    elif piv[1] != _INT_MAX:
        row = 2 * int(piv[1]) + 1
    else:
        return
    raise ZeroPivotError(f"{what} factorization hit a near-zero pivot at row {row}")


def _check_rhs_shape(rhs, n_modes, z2_shape):
    shape = tuple(rhs.shape)
    want = (n_modes,) + tuple(z2_shape)
    if shape != want:
        raise ValueError(f"rhs shape {shape} does not match {want}")


# ------------------------------------------------------------------ Helmholtz

def _helm_tables(mats):
    nd = mats.n_dir
    sd = np.ascontiguousarray(mats.stiff_dir.banded.diagonal(0), dtype=np.float64)
    st = np.ascontiguousarray(mats.stiff_dir.tail, dtype=np.float64)
    md = np.ascontiguousarray(mats.mass_dir.diagonal(0), dtype=np.float64)
    assert sd.size == nd and st.size == nd and md.size == nd
    return sd, st, md


class HelmholtzLU:
    """Device-resident Helmholtz factorisation, batched over z^2 (reference
    ``HelmholtzLU``, solvers.py:78-126)."""

    def __init__(self, n_x, family, z2_shape, ca, cb_dev, tables_dev, chunk_rows, ckpt, method, stored=None):
        self.n_x = int(n_x)
        self.family = family
        self.z2_shape = tuple(z2_shape)
        self.ca = float(ca)
        self._cb = cb_dev
        self._tab = tables_dev
        self.chunk_rows = int(chunk_rows)
        self._ckpt = ckpt
        self.method = method
        self._stored = stored  # list of 8 device tensors (exact factors) or None
        self._host = None

    @property
    def n_modes(self) -> int:
        return self.n_x - 1

    @property
    def batch(self) -> int:
        return int(self._cb.numel())

    # lazily materialised reference-exact factors --------------------------
    def _factors_dev(self):
        import torch

        if self._stored is not None:
            return self._stored
        nd, B = self.n_modes, self.batch
        dev = self._cb.device
        rows = [(nd + 1) // 2, nd // 2]
        bufs = []
        for name in ("low", "d", "e", "tail"):
            for p in (0, 1):
                n = rows[p] - 1 if name == "low" else rows[p]
                bufs.append(torch.empty((max(n, 0), B), dtype=torch.float64, device=dev))
        ptrs, keep = ptr_array([b.data_ptr() for b in bufs])
        sd, st, md = self._tab
        check(lib().shen_helm_factor(nd, self.ca, self._cb.data_ptr(), B, sd.data_ptr(), st.data_ptr(),
                                     md.data_ptr(), 0, None, ptrs, 1, None, dv.stream_handle()),
              "shen_helm_factor(exact)")
        del keep
        return bufs

    def _host_factors(self):
        if self._host is None:
            bufs = [b.cpu().numpy() for b in self._factors_dev()]
            self._host = {"low": bufs[0:2], "d": bufs[2:4], "e": bufs[4:6], "tail": bufs[6:8]}
        return self._host

    @property
    def low(self):
        return self._host_factors()["low"]

    @property
    def d(self):
        return self._host_factors()["d"]

    @property
    def e(self):
        return self._host_factors()["e"]

    @property
    def tail(self):
        return self._host_factors()["tail"]

    def storage_bytes(self) -> int:
        n = sum(int(t.numel()) for t in (self._stored or []))
        return 8 * (n + (int(self._ckpt.numel()) if self._ckpt is not None else 0) + self.batch)

    def solve(self, rhs, out=None):
        """Solve H x = rhs; rhs shape (n_modes, *z2_shape); numpy in -> numpy
        out, torch CUDA in -> torch out (reference solvers.py:100-109).
        ``out`` (optional, numpy) receives the result; with page-locked host
        buffers the copies overlap the solve slab by slab."""
        return _solve_api(self, rhs, out)

    def solve_into(self, rhs_dev, out_dev, is_complex, j0=0, j1=-1, max_ctas=0):
        """Device-to-device solve on (n_modes, batch) contiguous tensors
        (systems [j0, j1) only with the stream method)."""
        nd, B = self.n_modes, self.batch
        if B == 0:
            return out_dev
        if self.method == "stream" and not is_complex and (B % 2 or rhs_dev.data_ptr() % 16):
            return _solve_real_via_complex(self, rhs_dev, out_dev)
        h = lib()
        sh = dv.stream_handle()
        if self.method == "stored":
            ptrs, keep = ptr_array([b.data_ptr() for b in self._stored])
            check(h.shen_helm_solve_stored(nd, B, ptrs, rhs_dev.data_ptr(), out_dev.data_ptr(),
                                           int(is_complex), sh), "shen_helm_solve_stored")
            del keep
        else:
            sd, st, md = self._tab
            ck = self._ckpt.data_ptr() if self._ckpt is not None else None
            scratch = _scratch(self, 0, nd, B, is_complex, out_dev.device)
            check(h.shen_helm_solve_stream(nd, self.ca, self._cb.data_ptr(), B, sd.data_ptr(), st.data_ptr(),
                                           md.data_ptr(), self.chunk_rows, ck, rhs_dev.data_ptr(),
                                           out_dev.data_ptr(), scratch, int(is_complex), stream_warps(), max_ctas,
                                           j0, j1, sh),
                  "shen_helm_solve_stream")
        return out_dev


def build_helmholtz(mats: MatrixSet, nu: float, dt: float, z2, method: str = "stream") -> HelmholtzLU:
    """Factor the Helmholtz operator for every z^2 (reference solvers.py:201-241).

    ``method="stream"`` (default): checkpoints every 8 rows for the streaming
    fused solve (one thread per system, coalesced rows).
    ``method="stored"``: full reference-exact factors kept on the device.
    Raises ``ZeroPivotError`` exactly like the reference."""
    import torch

    if method not in _METHODS:
        raise ValueError(f"unknown method {method!r}")
    if dv.is_torch(z2):
        z2 = z2.detach().cpu().numpy()
    z2 = np.asarray(z2, dtype=float)
    ca, cb = helmholtz_coefficients(nu, dt, z2)
    cb_flat = np.atleast_1d(cb).reshape(-1)
    nd = mats.n_dir
    dev = dv.device()
    tabs = tuple(torch.from_numpy(t).to(dev) for t in _helm_tables(mats))
    cb_dev = torch.from_numpy(np.ascontiguousarray(cb_flat)).to(dev)
    B = cb_flat.size
    R = STREAM_ROWS_H
    h = lib()
    sh = dv.stream_handle()
    pivot = torch.empty(2, dtype=torch.int32, device=dev)
    check(h.shen_pivot_reset(pivot.data_ptr(), sh), "shen_pivot_reset")
    ckpt = None
    stored = None
    if method == "stream":
        C = _n_chunks(nd, R)
        ckpt = torch.empty((C, 2, 3, B), dtype=torch.float64, device=dev) if C > 1 else None
        check(h.shen_helm_factor(nd, float(ca), cb_dev.data_ptr(), B, tabs[0].data_ptr(), tabs[1].data_ptr(),
                                 tabs[2].data_ptr(), R, ckpt.data_ptr() if ckpt is not None else None, None, 0,
                                 pivot.data_ptr(), sh), "shen_helm_factor")
    else:
        rows = [(nd + 1) // 2, nd // 2]
        stored = []
        for name in ("low", "d", "e", "tail"):
            for p in (0, 1):
                n = rows[p] - 1 if name == "low" else rows[p]
                stored.append(torch.empty((max(n, 0), B), dtype=torch.float64, device=dev))
        ptrs, keep = ptr_array([b.data_ptr() for b in stored])
        check(h.shen_helm_factor(nd, float(ca), cb_dev.data_ptr(), B, tabs[0].data_ptr(), tabs[1].data_ptr(),
                                 tabs[2].data_ptr(), 0, None, ptrs, 1, pivot.data_ptr(), sh), "shen_helm_factor")
        del keep
    if B > 0:
        _raise_pivot(pivot.cpu().numpy(), "Helmholtz")
    return HelmholtzLU(mats.n_x, mats.family, np.shape(z2), ca, cb_dev, tabs, R, ckpt, method, stored)


# ------------------------------------------------------------------ biharmonic

BIH_NCOL = 18  # 17 constants + 1 pad (16-B aligned rows on the device)


def _bih_table(mats):
    """Per-mode row constants (csrc/shen_rows.cuh BihCol), zeros where the
    reference's band() leaves an entry out (solvers.py:244-268,287-304)."""
    nb = mats.n_bih
    p, q, r, s = tail_factors(nb)
    q0 = mats.fourth_bih.diag
    ar_m2 = -mats.stiff_bih.diagonal(-2)
    ar_0 = -mats.stiff_bih.diagonal(0)
    ar_2 = -mats.stiff_bih.diagonal(2)
    bb0 = mats.mass_bih.diagonal(0)
    bb2 = mats.mass_bih.diagonal(2)
    bb4 = mats.mass_bih.diagonal(4)
    tail2 = p[:nb - 2] * q[2:] + r[:nb - 2] * s[2:]
    tail4 = p[:nb - 4] * q[4:] + r[:nb - 4] * s[4:]
    T = np.zeros((nb, BIH_NCOL))
    k = np.arange(nb)
    T[:, 0] = q0
    T[:, 1] = ar_0
    T[:, 2] = bb0
    v2 = k + 2 <= nb - 1
    T[v2, 3] = tail2
    T[v2, 4] = ar_2
    T[v2, 5] = bb2
    v4 = k + 4 <= nb - 1
    T[v4, 6] = tail4
    T[v4, 7] = bb4
    m2 = k >= 2
    T[m2, 8] = ar_m2
    T[m2, 9] = bb2
    m4 = k >= 4
    T[m4, 10] = bb4
    T[:, 11] = p
    T[:, 12] = r
    T[v2, 13] = q[2:]
    T[v2, 14] = s[2:]
    T[v4, 15] = q[4:]
    T[v4, 16] = s[4:]
    return np.ascontiguousarray(T), q, s


class BiharmonicLU:
    """Device-resident biharmonic factorisation (reference ``BiharmonicLU``,
    solvers.py:129-198)."""

    def __init__(self, n_x, family, z2_shape, xi0, xi1_dev, xi2_dev, tab_dev, q, s, chunk_rows, ckpt, method,
                 stored=None):
        self.n_x = int(n_x)
        self.family = family
        self.z2_shape = tuple(z2_shape)
        self.xi0 = float(xi0)
        self._xi1 = xi1_dev
        self._xi2 = xi2_dev
        self._tab = tab_dev
        self.q = q
        self.s = s
        self.chunk_rows = int(chunk_rows)
        self._ckpt = ckpt
        self.method = method
        self._stored = stored
        self._qs_dev = None
        self._host = None
        self._pairs = None  # device (2, P) int64 mirror pairs (build_biharmonic), or None

    @property
    def n_modes(self) -> int:
        return self.n_x - 3

    @property
    def batch(self) -> int:
        return int(self._xi1.numel())

    def storage_vectors(self) -> int:
        """Stored O(N) vectors per system in the reference layout (solvers.py:158-160)."""
        return 7

    def _factors_dev(self):
        import torch

        if self._stored is not None:
            return self._stored
        nb, B = self.n_modes, self.batch
        dev = self._xi1.device
        rows = [(nb + 1) // 2, nb // 2]
        bufs = []
        for name, off in (("low2", 1), ("low4", 2), ("d", 0), ("e", 0), ("f", 0), ("a", 0), ("b", 0)):
            for p in (0, 1):
                bufs.append(torch.zeros((max(rows[p] - off, 0), B), dtype=torch.float64, device=dev))
        ptrs, keep = ptr_array([b.data_ptr() for b in bufs])
        check(lib().shen_bih_factor(nb, self.xi0, self._xi1.data_ptr(), self._xi2.data_ptr(), B,
                                    self._tab.data_ptr(), 0, None, ptrs, 1, None, dv.stream_handle()),
              "shen_bih_factor(exact)")
        del keep
        return bufs

    def _host_factors(self):
        if self._host is None:
            bufs = [b.cpu().numpy() for b in self._factors_dev()]
            names = ("low2", "low4", "d", "e", "f", "a", "b")
            self._host = {nm: bufs[2 * i:2 * i + 2] for i, nm in enumerate(names)}
        return self._host

    low2 = property(lambda self: self._host_factors()["low2"])
    low4 = property(lambda self: self._host_factors()["low4"])
    d = property(lambda self: self._host_factors()["d"])
    e = property(lambda self: self._host_factors()["e"])
    f = property(lambda self: self._host_factors()["f"])
    a = property(lambda self: self._host_factors()["a"])
    b = property(lambda self: self._host_factors()["b"])

    def solve(self, rhs, out=None):
        """Solve H x = rhs (reference solvers.py:162-170); see HelmholtzLU.solve."""
        return _solve_api(self, rhs, out)

    def solve_into(self, rhs_dev, out_dev, is_complex, j0=0, j1=-1, max_ctas=0):
        nb, B = self.n_modes, self.batch
        if B == 0:
            return out_dev
        if self.method == "stream" and not is_complex and (B % 2 or rhs_dev.data_ptr() % 16):
            return _solve_real_via_complex(self, rhs_dev, out_dev)
        h = lib()
        sh = dv.stream_handle()
        if self.method == "stored":
            import torch

            if self._qs_dev is None:
                self._qs_dev = (torch.from_numpy(np.ascontiguousarray(self.q)).to(out_dev.device),
                                torch.from_numpy(np.ascontiguousarray(self.s)).to(out_dev.device))
            ptrs, keep = ptr_array([b.data_ptr() for b in self._stored])
            check(h.shen_bih_solve_stored(nb, B, self.xi0, self._qs_dev[0].data_ptr(), self._qs_dev[1].data_ptr(),
                                          ptrs, rhs_dev.data_ptr(), out_dev.data_ptr(), int(is_complex), sh),
                  "shen_bih_solve_stored")
            del keep
        elif self.method == "stream" and self._pairs is not None and j0 == 0 and j1 in (-1, B):
            # mirror pairs: one factor recurrence for two systems (bit-identical results)
            ck = self._ckpt.data_ptr() if self._ckpt is not None else None
            scratch = _scratch(self, 1, nb, B, is_complex, out_dev.device)
            P = int(self._pairs.shape[1])
            check(h.shen_bih_solve_stream_pairs(nb, self.xi0, self._xi1.data_ptr(), self._xi2.data_ptr(), B,
                                                self._tab.data_ptr(), self.chunk_rows, ck, rhs_dev.data_ptr(),
                                                out_dev.data_ptr(), scratch, int(is_complex), self._pairs.data_ptr(),
                                                P, max_ctas, sh),
                  "shen_bih_solve_stream_pairs")
        else:
            ck = self._ckpt.data_ptr() if self._ckpt is not None else None
            scratch = _scratch(self, 1, nb, B, is_complex, out_dev.device)
            check(h.shen_bih_solve_stream(nb, self.xi0, self._xi1.data_ptr(), self._xi2.data_ptr(), B,
                                          self._tab.data_ptr(), self.chunk_rows, ck, rhs_dev.data_ptr(),
                                          out_dev.data_ptr(), scratch, int(is_complex), stream_warps(), max_ctas,
                                          j0, j1, sh),
                  "shen_bih_solve_stream")
        return out_dev


def build_biharmonic(mats: MatrixSet, nu: float, dt: float, z2, method: str = "stream") -> BiharmonicLU:
    """Factor the biharmonic operator for every z^2 (reference solvers.py:271-355)."""
    import torch

    if method not in _METHODS:
        raise ValueError(f"unknown method {method!r}")
    if dv.is_torch(z2):
        z2 = z2.detach().cpu().numpy()
    z2 = np.asarray(z2, dtype=float)
    xi0, xi1, xi2 = biharmonic_coefficients(nu, dt, z2)
    x1 = np.ascontiguousarray(np.atleast_1d(xi1).reshape(-1))
    x2 = np.ascontiguousarray(np.atleast_1d(xi2).reshape(-1))
    nb = mats.n_bih
    dev = dv.device()
    T, q, s = _bih_table(mats)
    tab = torch.from_numpy(T).to(dev)
    x1d = torch.from_numpy(x1).to(dev)
    x2d = torch.from_numpy(x2).to(dev)
    B = x1.size
    R = STREAM_ROWS_B
    h = lib()
    sh = dv.stream_handle()
    pivot = torch.empty(2, dtype=torch.int32, device=dev)
    check(h.shen_pivot_reset(pivot.data_ptr(), sh), "shen_pivot_reset")
    ckpt = None
    stored = None
    if method == "stream":
        C = _n_chunks(nb, R)
        ckpt = torch.empty((C, 2, 10, B), dtype=torch.float64, device=dev) if C > 1 else None
        check(h.shen_bih_factor(nb, float(xi0), x1d.data_ptr(), x2d.data_ptr(), B, tab.data_ptr(), R,
                                ckpt.data_ptr() if ckpt is not None else None, None, 0, pivot.data_ptr(), sh),
              "shen_bih_factor")
    else:
        rows = [(nb + 1) // 2, nb // 2]
        stored = []
        for name, off in (("low2", 1), ("low4", 2), ("d", 0), ("e", 0), ("f", 0), ("a", 0), ("b", 0)):
            for p in (0, 1):
                stored.append(torch.zeros((max(rows[p] - off, 0), B), dtype=torch.float64, device=dev))
        ptrs, keep = ptr_array([b.data_ptr() for b in stored])
        check(h.shen_bih_factor(nb, float(xi0), x1d.data_ptr(), x2d.data_ptr(), B, tab.data_ptr(), 0, None,
                                ptrs, 1, pivot.data_ptr(), sh), "shen_bih_factor")
        del keep
    if B > 0:
        _raise_pivot(pivot.cpu().numpy(), "biharmonic")
    lu = BiharmonicLU(mats.n_x, mats.family, np.shape(z2), xi0, x1d, x2d, tab, q, s, R, ckpt, method, stored)
    if method == "stream" and MIRROR_PAIRS:
        pr = mirror_pairs(z2)
        # small batches keep one system per thread: halving the threads of a
        # launch that cannot fill the GPU costs more than the shared work saves
        # (config 1, 1.1k pairs: 44 vs 39 us; config 3, 16.6k pairs: 0.097 vs 0.120 ms)
        if pr is not None and pr.shape[1] >= PAIRS_MIN:
            lu._pairs = torch.from_numpy(np.ascontiguousarray(pr)).to(dev)
    return lu


# ------------------------------------------------------------------ host helpers (tests)

def dense_helmholtz(mats, nu, dt, z2) -> np.ndarray:
    """Dense H (reference solvers.py:361-363); host, tests only."""
    ca, cb = helmholtz_coefficients(nu, dt, float(z2))
    return ca * mats.stiff_dir.dense() + cb * mats.mass_dir.dense()


def dense_biharmonic(mats, nu, dt, z2) -> np.ndarray:
    """Dense biharmonic operator (reference solvers.py:366-369); host, tests only."""
    xi0, xi1, xi2 = biharmonic_coefficients(nu, dt, float(z2))
    return xi0 * mats.fourth_bih.dense() - xi1 * mats.stiff_bih.dense() + xi2 * mats.mass_bih.dense()


def lu_nopivot(a):
    """Dense unpivoted LU (reference solvers.py:372-384); host, tests only."""
    n = a.shape[0]
    u = np.array(a, dtype=float)
    low = np.eye(n)
    for i in range(n - 1):
        piv = u[i, i]
        if abs(piv) < PIVOT_FLOOR:
            raise ZeroPivotError(f"dense elimination pivot ~0 at row {i}")
        mult = u[i + 1:, i] / piv
        low[i + 1:, i] = mult
        u[i + 1:] -= mult[:, None] * u[i]
    return low, u


def solve_field(lu, field):
    """Per-wavenumber solve of a whole SpectralField (reference solvers.py:387-392)."""
    from .transforms import SpectralField

    return SpectralField(lu.solve(field.data), field.grid, field.mesh)

