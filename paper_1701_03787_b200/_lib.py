"""ctypes binding of the in-tree C-ABI library ``libshen_b200.so``.

There is no CPU fallback: if the library is missing, or no CUDA device is
visible, every solver/transform entry point raises ``ShenBackendError``.
Loading the library itself does not need a GPU (cudart is linked
statically), so the symbol table can be checked on a CPU-only machine.
"""

from __future__ import annotations

import ctypes
import os
import threading

__all__ = ["ShenBackendError", "lib", "lib_path", "require_device", "check", "declared_symbols"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# SHEN_LIB_VARIANT=<tag> loads libshen_b200_<tag>.so from the same directory
# (A/B timing of kernel variants built by tools/ab_build.sh; default: the product library)
_variant = os.environ.get("SHEN_LIB_VARIANT", "")
lib_path = os.path.join(_HERE, f"libshen_b200_{_variant}.so" if _variant else "libshen_b200.so")


class ShenBackendError(RuntimeError):
    """The B200 backend (CUDA library or device) is unavailable."""


_c_int64 = ctypes.c_int64
_vp = ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes); mirrors include/shen_b200.h
class ShenBand(ctypes.Structure):
    _fields_ = [("nr", ctypes.c_int), ("nc", ctypes.c_int), ("n_off", ctypes.c_int), ("off", ctypes.c_int * 6),
                ("diag", ctypes.c_void_p)]


class ShenRhsGArgs(ctypes.Structure):
    _fields_ = [("n_dir", ctypes.c_int), ("L", ctypes.c_int64), ("stiff", ShenBand), ("mass", ShenBand),
                ("tail", ctypes.c_void_p), ("tail_start", ctypes.c_int), ("c_stiff", ctypes.c_double),
                ("dt", ctypes.c_double), ("cg", ctypes.c_void_p), ("im_m_re", ctypes.c_void_p),
                ("im_m_im", ctypes.c_void_p), ("im_n_re", ctypes.c_void_p), ("im_n_im", ctypes.c_void_p),
                ("g", ctypes.c_void_p), ("hcy", ctypes.c_void_p), ("hpy", ctypes.c_void_p), ("hcz", ctypes.c_void_p),
                ("hpz", ctypes.c_void_p), ("out", ctypes.c_void_p)]


class ShenRhsUArgs(ctypes.Structure):
    _fields_ = [("n_bih", ctypes.c_int), ("L", ctypes.c_int64), ("d", ctypes.c_void_p), ("p", ctypes.c_void_p),
                ("q", ctypes.c_void_p), ("r", ctypes.c_void_p), ("s", ctypes.c_void_p), ("c_fourth", ctypes.c_double),
                ("stiff", ShenBand), ("mass", ShenBand), ("mixed", ShenBand), ("deriv", ShenBand),
                ("c_stiff", ctypes.c_void_p), ("c_mass", ctypes.c_void_p), ("c_mixed", ctypes.c_void_p),
                ("c_dy_re", ctypes.c_void_p), ("c_dy_im", ctypes.c_void_p), ("c_dz_re", ctypes.c_void_p),
                ("c_dz_im", ctypes.c_void_p), ("u", ctypes.c_void_p), ("hcx", ctypes.c_void_p),
                ("hpx", ctypes.c_void_p), ("hcy", ctypes.c_void_p), ("hpy", ctypes.c_void_p), ("hcz", ctypes.c_void_p),
                ("hpz", ctypes.c_void_p), ("out", ctypes.c_void_p)]


class ShenRecoverArgs(ctypes.Structure):
    _fields_ = [("n_dir", ctypes.c_int), ("L", ctypes.c_int64), ("deriv", ShenBand), ("fac", ctypes.c_void_p),
                ("mmax", ctypes.c_int), ("im_m_re", ctypes.c_void_p), ("im_m_im", ctypes.c_void_p),
                ("im_n_re", ctypes.c_void_p), ("im_n_im", ctypes.c_void_p), ("safe_z2", ctypes.c_void_p),
                ("u", ctypes.c_void_p), ("g", ctypes.c_void_p), ("v", ctypes.c_void_p), ("w", ctypes.c_void_p)]


class ShenWallPlan(ctypes.Structure):
    _fields_ = [("direction", ctypes.c_int), ("family", ctypes.c_int), ("space", ctypes.c_int), ("mass", ctypes.c_int),
                ("N", ctypes.c_int), ("n_out", ctypes.c_int), ("n_in", ctypes.c_int), ("kind", ctypes.c_int),
                ("Ld", ctypes.c_int), ("M", ctypes.c_int), ("nstage", ctypes.c_int), ("radix", ctypes.c_int * 4),
                ("log2_lines", ctypes.c_int), ("rows_smem", ctypes.c_int), ("scale", ctypes.c_double),
                ("nband", ctypes.c_int), ("mmax", ctypes.c_int),
                ("tw", _vp), ("ker_f", _vp), ("ker_i", _vp), ("chirp_f", _vp), ("chirp_i", _vp),
                ("gin_f", _vp), ("gin_i", _vp), ("gout", _vp), ("pinv", _vp), ("mk", _vp),
                ("c2", _vp), ("c4", _vp), ("mfac", _vp), ("rowscale", _vp)]


_SIGS = {
    "shen_version": (ctypes.c_char_p, []),
    "shen_last_error": (ctypes.c_char_p, []),
    "shen_device_count": (ctypes.c_int, []),
    "shen_pivot_reset": (ctypes.c_int, [_vp, _vp]),
    "shen_memcpy2d_async": (ctypes.c_int, [_vp, _c_int64, _vp, _c_int64, _c_int64, _c_int64, ctypes.c_int, _vp]),
    "shen_stream_scratch_bytes": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_int64, ctypes.c_int]),
    "shen_helm_factor": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, _vp, _c_int64, _vp, _vp, _vp,
                                        ctypes.c_int, _vp, _pp, ctypes.c_int, _vp, _vp]),
    "shen_helm_solve_stream": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, _vp, _c_int64, _vp, _vp, _vp,
                                              ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, _c_int64, _c_int64, _vp]),
    "shen_wall_transform": (ctypes.c_int, [ctypes.POINTER(ShenWallPlan), _c_int64, _vp, _vp, _vp]),
    "shen_wall_smem_bytes": (ctypes.c_int64, [ctypes.POINTER(ShenWallPlan)]),
    "shen_helm_solve_stored": (ctypes.c_int, [ctypes.c_int, _c_int64, _pp, _vp, _vp, ctypes.c_int, _vp]),
    "shen_bih_factor": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, _vp, _vp, _c_int64, _vp, ctypes.c_int,
                                       _vp, _pp, ctypes.c_int, _vp, _vp]),
    "shen_bih_solve_stream": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, _vp, _vp, _c_int64, _vp,
                                             ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, _c_int64, _c_int64, _vp]),
    "shen_bih_solve_stream_pairs": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, _vp, _vp, _c_int64, _vp,
                                                   ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_int, _vp, _c_int64,
                                                   ctypes.c_int, _vp]),
    "shen_bih_solve_stored": (ctypes.c_int, [ctypes.c_int, _c_int64, ctypes.c_double, _vp, _vp, _pp, _vp, _vp,
                                             ctypes.c_int, _vp]),
    "shen_apply_banded": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _c_int64, ctypes.c_int, _vp, _vp, _vp, _vp,
                                         ctypes.c_int, _vp]),
    "shen_apply_const_tail": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _c_int64, ctypes.c_int, _vp, _vp, _vp,
                                             ctypes.c_int, _vp, _vp, ctypes.c_int, _vp]),
    "shen_apply_rank2_tail": (ctypes.c_int, [ctypes.c_int, _c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                             ctypes.c_int, _vp]),
    "shen_rhs_g": (ctypes.c_int, [ctypes.POINTER(ShenRhsGArgs), _vp]),
    "shen_rhs_u": (ctypes.c_int, [ctypes.POINTER(ShenRhsUArgs), _vp]),
    "shen_recover_velocity": (ctypes.c_int, [ctypes.POINTER(ShenRecoverArgs), _vp]),
    "shen_cross": (ctypes.c_int, [_c_int64, _vp, _vp, _vp]),
    "shen_plane_fft_supported": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "shen_plane_rfft2": (ctypes.c_int, [_c_int64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "shen_plane_irfft2": (ctypes.c_int, [_c_int64, ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_double, _vp]),
    "shen_plane_rfft2_fac": (ctypes.c_int, [_c_int64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "shen_plane_irfft2_fac": (ctypes.c_int, [_c_int64, ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_double, _vp, _vp,
                                             _vp]),
    "shen_plane_rfft2_scatter": (ctypes.c_int, [_c_int64, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp, _vp, _vp,
                                                _vp, _c_int64, _c_int64, _vp]),
    "shen_plane_irfft2_gather": (ctypes.c_int, [_c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp,
                                                _c_int64, _c_int64, _vp, ctypes.c_double, _vp]),
    "shen_enable_peer_access": (ctypes.c_int, [ctypes.c_int]),
    "shen_xform_extend": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _c_int64, _vp, _vp, _vp]),
    "shen_xform_fwd_post": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_int64, ctypes.c_double,
                                           _vp, _vp, _vp, _vp]),
    "shen_xform_inv_pre": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_int64, _vp,
                                          _vp, _vp, _vp, _vp]),
    "shen_xform_inv_post": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _c_int64, _vp, _vp, _vp, _vp]),
    "shen_xform_mass_solve": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_int64, _vp, _vp, _vp,
                                             _vp]),
}

_lock = threading.Lock()
_lib = None


def declared_symbols():
    return tuple(_SIGS)


def lib():
    """The loaded library (raises ShenBackendError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(lib_path):
                raise ShenBackendError(
                    f"{lib_path} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "or `make -C paper_1701_03787_b200/csrc` (no CPU fallback exists)")
            handle = ctypes.CDLL(lib_path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def require_device():
    """Fail loudly unless a CUDA device is usable from both torch and the library."""
    import torch

    if not torch.cuda.is_available():
        raise ShenBackendError("paper_1701_03787_b200 needs a CUDA (B200) device; there is no CPU fallback")
    handle = lib()
    if handle.shen_device_count() < 1:
        raise ShenBackendError("libshen_b200.so sees no CUDA device")
    return handle


def check(status: int, what: str):
    if status != 0:
        msg = lib().shen_last_error().decode(errors="replace")
        raise ShenBackendError(f"{what} failed (status {status}): {msg}")


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(p) for p in ptrs])
    return ctypes.cast(arr, _pp), arr
