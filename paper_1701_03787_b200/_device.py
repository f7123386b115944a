"""Host <-> device plumbing for the drop-in API (torch is used only for
device memory, streams and copies)."""

from __future__ import annotations

import numpy as np

from ._lib import require_device

__all__ = ["device", "stream_handle", "to_device_f64", "as_rhs", "is_torch"]


def device():
    import torch

    require_device()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    import torch

    return torch.cuda.current_stream().cuda_stream


def is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def to_device_f64(arr):
    """float64 contiguous device tensor from a numpy array / scalar / tensor."""
    import torch

    if is_torch(arr):
        return arr.to(device=device(), dtype=torch.float64).contiguous()
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.float64))
    return torch.from_numpy(a).to(device())


def as_rhs(rhs):
    """(device tensor in float64/complex128, is_complex, came_from_numpy).

    The result dtype follows the reference: ``np.result_type(rhs, float)``
    (solvers.py:106) -- complex inputs become complex128, everything else
    float64."""
    import torch

    if is_torch(rhs):
        cplx = rhs.is_complex()
        t = rhs.to(device=device(), dtype=torch.complex128 if cplx else torch.float64).contiguous()
        return t, cplx, False
    a = np.asarray(rhs)
    cplx = np.iscomplexobj(a)
    a = np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)
    t = torch.from_numpy(a)
    if t.numel() > 0:
        t = t.pin_memory()
    return t.to(device(), non_blocking=True), cplx, True
