"""The C-ABI library: loads without a GPU and exports every symbol that
include/shen_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

import pytest

from paper_1701_03787_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "shen_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(shen_[a-z0-9_]+)\s*\(", text)))


def test_library_built():
    assert os.path.exists(_lib.lib_path), "run __graft_entry__.build() first"


def test_exports_every_header_symbol():
    handle = ctypes.CDLL(_lib.lib_path)
    syms = _header_symbols()
    assert len(syms) >= 10
    missing = [s for s in syms if not hasattr(handle, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert sorted(_lib.declared_symbols()) == _header_symbols()


def test_load_and_query_without_gpu():
    h = _lib.lib()
    assert b"sm_100a" in h.shen_version()
    n = h.shen_device_count()
    assert n >= 0


def test_argument_errors_are_reported():
    h = _lib.lib()
    # invalid sizes are rejected before any device work
    st = h.shen_helm_factor(1, 0.0, None, 1, None, None, None, 0, None, None, 0, None, None)
    assert st == 1
    assert b"bad args" in h.shen_last_error()


def test_product_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_1701_03787_b200 import solvers
    from paper_1701_03787_b200.matrices import assemble

    with pytest.raises(_lib.ShenBackendError):
        solvers.build_helmholtz(assemble(16, 0), 1e-3, 1e-3, [0.0, 1.0])


def test_every_compute_entry_point_validates_arguments():
    """Bad sizes / NULL pointers are rejected with SHEN_ERR_ARG and a message
    naming the entry point, before any device work (runs without a GPU)."""
    import ctypes

    h = _lib.lib()
    cases = {
        "shen_helm_solve_stream": (1, 0.0, None, 1, None, None, None, 8, None, None, None, None, 1, 0, 0, 0, -1,
                                   None),
        "shen_bih_solve_stream": (1, 0.0, None, None, 1, None, 8, None, None, None, None, 1, 0, 0, 0, -1, None),
        "shen_bih_factor": (1, 0.0, None, None, 1, None, 8, None, None, 0, None, None),
        "shen_bih_solve_stream_pairs": (1, 0.0, None, None, 1, None, 8, None, None, None, None, 1, None, 1, 0, None),
        "shen_xform_extend": (3, 5, 1, None, None, None),
        "shen_xform_fwd_post": (0, 9, 5, 1, 1.0, None, None, None, None),
        "shen_xform_inv_pre": (0, 1, 9, 5, 1, None, None, None, None, None),
        "shen_xform_inv_post": (0, 1, 1, None, None, None, None),
        "shen_xform_mass_solve": (3, 8, 4, 1, None, None, None, None),
        "shen_apply_banded": (4, 4, 1, 9, None, None, None, None, 1, None),
        "shen_apply_const_tail": (4, 4, 1, 1, None, None, None, 2, None, None, 1, None),
        "shen_apply_rank2_tail": (4, 1, None, None, None, None, None, None, None, 1, None),
        "shen_cross": (8, None, None, None),
        "shen_memcpy2d_async": (None, 16, None, 16, 16, 1, 0, None),
        "shen_plane_rfft2": (1, 128, 256, 16, 16, None),  # unsupported plane size
        "shen_plane_irfft2": (1, 256, 256, 24, 8, ctypes.c_double(1.0), None),  # X not 16-B aligned
        "shen_plane_rfft2_fac": (1, 256, 256, 16, 16, None, None),  # no factor table
        "shen_plane_irfft2_fac": (1, 256, 256, 16, 8, ctypes.c_double(1.0), 8, None, None),  # no imaginary table
        # exchange-fused plane FFTs: no rank tables / 9 ranks
        "shen_plane_rfft2_scatter": (1, 256, 256, 16, 2, None, None, None, None, 0, 1, None),
        "shen_plane_irfft2_gather": (1, 256, 256, 9, None, None, None, None, 0, 1, 16, ctypes.c_double(1.0), None),
    }
    for name, args in cases.items():
        st = getattr(h, name)(*args)
        assert st == 1, name
        assert name.encode() in h.shen_last_error() or b"bad args" in h.shen_last_error(), name
    assert h.shen_plane_fft_supported(256, 256) == 1 and h.shen_plane_fft_supported(64, 32) == 0
    # a row table that points outside its owner's buffer, or planes past the total, are rejected
    bases = (ctypes.c_void_p * 2)(4096, 8192)
    rows = (ctypes.c_int64 * 2)(128, 128)
    owner = (ctypes.c_int * 256)(*([0] * 128 + [1] * 128))
    local = (ctypes.c_int * 256)(*(list(range(128)) * 2))
    local_bad = (ctypes.c_int * 256)(*([128] + list(range(1, 128)) + list(range(128))))
    owner_bad = (ctypes.c_int * 256)(*([2] + [0] * 127 + [1] * 128))
    for ow, lo, plane0, total in ((owner, local_bad, 0, 4), (owner_bad, local, 0, 4), (owner, local, 3, 4)):
        assert h.shen_plane_rfft2_scatter(2, 256, 256, 16, 2, bases, rows, ow, lo, plane0, total, None) == 1
        assert h.shen_plane_irfft2_gather(2, 256, 256, 2, bases, rows, ow, lo, plane0, total, 16,
                                          ctypes.c_double(1.0), None) == 1
    for name, cls in (("shen_rhs_g", _lib.ShenRhsGArgs), ("shen_rhs_u", _lib.ShenRhsUArgs),
                      ("shen_recover_velocity", _lib.ShenRecoverArgs)):
        a = cls()
        a.L = 4
        if hasattr(a, "n_dir"):
            a.n_dir = 4
        if hasattr(a, "n_bih"):
            a.n_bih = 4
        assert getattr(h, name)(ctypes.byref(a), None) == 1, name
        assert getattr(h, name)(None, None) == 1, name
