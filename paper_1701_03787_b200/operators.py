"""Structured wall-normal operators on the device.

``apply(M, x)`` is ``M.apply(x)`` of the reference's ``BandedMatrix``,
``ConstantTailMatrix`` and ``Rank2TailMatrix`` (``matrices.py:62-71,
109-117, 145-152``; this package's ``matrices`` classes or the reference's,
duck-typed) evaluated by ``csrc/shen_apply.cu`` along axis 0 of any
``(rows, ...)`` array, real or complex -- bit-identical to the reference
(same operation order, no contraction).  These products form the stepper's
right-hand sides (``stepper.py:193-220``) and the roundoff checks
(``verify.py:129-136``).

numpy in -> numpy out; torch CUDA tensors stay on the device.  No CPU
fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._device import device, is_torch, stream_handle

__all__ = ["apply", "DeviceOperator", "operator_tables"]


def operator_tables(M):
    """Host tables of one structured matrix, read through the attributes the
    reference's classes and this package's share (``matrices.py:46-152``):
    ``(2, (diag, p, q, r, s))`` for a rank-2 tail, else ``(kind, (offsets,
    band table [n_off][rows], tail | None, tail_start))`` with kind 1 for a
    constant tail and 0 for a plain banded matrix."""
    if hasattr(M, "p") and hasattr(M, "q"):  # rank-2 tail
        return 2, tuple(np.ascontiguousarray(v, dtype=np.float64) for v in (M.diag, M.p, M.q, M.r, M.s))
    banded = M.banded if hasattr(M, "banded") else M
    kind = 1 if hasattr(M, "tail") else 0
    nr, nc = banded.shape
    offs = tuple(int(d) for d in banded.offsets)
    if len(offs) > 6:
        raise ValueError("at most 6 diagonals")
    tab = np.zeros((max(len(offs), 1), nr))
    for i, (d, diag) in enumerate(zip(offs, banded.diagonals)):
        a, b = max(0, -d), min(nr, nc - d)
        tab[i, a:b] = diag
    if kind == 1:
        return 1, (offs, tab, np.ascontiguousarray(M.tail, dtype=np.float64), int(M.tail_start))
    return 0, (offs, tab, None, 0)


class DeviceOperator:
    """Device copy of one structured matrix (tables uploaded once)."""

    def __init__(self, M):
        import torch

        dev = device()
        self.shape = tuple(M.shape)
        self.kind, tabs = operator_tables(M)
        if self.kind == 2:
            self._vecs = [torch.from_numpy(v).to(dev) for v in tabs]
            return
        offs, tab, tail, tail_start = tabs
        self._offs = (ctypes.c_int * max(len(offs), 1))(*offs) if offs else None
        self._n_off = len(offs)
        self._tab = torch.from_numpy(tab).to(dev)
        if self.kind == 1:
            self._tail = torch.from_numpy(tail).to(dev)
            self._tail_start = tail_start

    def __call__(self, x):
        """y = M x along axis 0; numpy or torch CUDA input."""
        import torch

        nr, nc = self.shape
        from_numpy = not is_torch(x)
        if from_numpy:
            a = np.asarray(x)
            cplx = np.iscomplexobj(a)
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)).to(device())
        else:
            cplx = x.is_complex()
            t = x.to(device=device(), dtype=torch.complex128 if cplx else torch.float64).contiguous()
        if t.dim() == 0 or t.shape[0] != nc:
            raise ValueError(f"expected leading size {nc}, got {tuple(t.shape)[:1]}")
        trailing = tuple(t.shape[1:])
        L = int(np.prod(trailing, dtype=np.int64)) if trailing else 1
        y = torch.empty((nr,) + trailing, dtype=t.dtype, device=t.device)
        lib = _lib.lib()
        st = stream_handle()
        if self.kind == 2:
            d, p, q, r, s = (v.data_ptr() for v in self._vecs)
            _lib.check(lib.shen_apply_rank2_tail(nr, L, d, p, q, r, s, t.data_ptr(), y.data_ptr(), int(cplx), st),
                       "shen_apply_rank2_tail")
        elif self.kind == 1:
            _lib.check(lib.shen_apply_const_tail(nr, nc, L, self._n_off, self._offs, self._tab.data_ptr(),
                                                 self._tail.data_ptr(), self._tail_start, t.data_ptr(),
                                                 y.data_ptr(), int(cplx), st), "shen_apply_const_tail")
        else:
            _lib.check(lib.shen_apply_banded(nr, nc, L, self._n_off, self._offs, self._tab.data_ptr(), t.data_ptr(),
                                             y.data_ptr(), int(cplx), st), "shen_apply_banded")
        if from_numpy:
            return y.cpu().numpy()
        return y


_CACHE = {}
_CACHE_MAX = 32  # device copies kept for the most recently used matrices


def apply(M, x):
    """``M.apply(x)`` on the device (reference matrices.py apply semantics).
    The device tables of the last ``_CACHE_MAX`` matrices are kept (least
    recently used dropped), keyed by identity; a kept entry holds its matrix
    so the identity cannot be reused while cached."""
    key = (id(M), device().index)
    op = _CACHE.pop(key, None)
    if op is None or op[0] is not M:
        op = (M, DeviceOperator(M))
    _CACHE[key] = op  # re-inserted: most recently used last
    while len(_CACHE) > _CACHE_MAX:
        _CACHE.pop(next(iter(_CACHE)))
    return op[1](x)
