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
