"""Checkpoint wire format of the reference stepper, for device-resident state
(reference ``stepper.py:352-401``).

Byte-compatible with ``chebchan.stepper.save_checkpoint`` /
``load_checkpoint``: header ``<8siiiiddddddqi`` (magic ``CHCHKPT1``,
version 1, n_x, n_y, n_z, l_y, l_z, nu, dt, t, beta, kappa, family) followed by
the little-endian complex128 arrays u, v, w, g, h_curr x 3, h_prev x 3.

The state's arrays may live on the device: ``save_checkpoint`` streams them
to the file through two page-locked staging buffers (the device-to-host copy
of array i+1 overlaps the write of array i); ``load_checkpoint(path,
device=True)`` returns CUDA tensors.  ``FlowState`` / ``StepperConfig``
mirror the reference's dataclasses (duck-typed: the reference's own objects
are accepted by ``save_checkpoint``).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from ._device import is_torch
from .mesh import PointFamily, Space, build_mesh, family_code, wavenumber_grid
from .transforms import SpectralField

__all__ = ["FlowState", "StepperConfig", "save_checkpoint", "load_checkpoint", "HEADER"]

HEADER = "<8siiiiddddddqi"
_MAGIC = b"CHCHKPT1"


@dataclass
class StepperConfig:
    """The two fields a checkpoint carries (reference ``StepperConfig``)."""

    nu: float
    dt: float


@dataclass
class FlowState:
    """Reference ``FlowState`` (stepper.py:68-80); field data numpy or torch."""

    u_hat: SpectralField
    v_hat: SpectralField
    w_hat: SpectralField
    g_hat: SpectralField
    h_curr: tuple
    h_prev: tuple
    beta: float
    t: float
    kappa: int


def _arrays(state):
    out = [state.u_hat.data, state.v_hat.data, state.w_hat.data, state.g_hat.data]
    out += [f.data for f in state.h_curr]
    out += [f.data for f in state.h_prev]
    return out


def save_checkpoint(path, state, config):
    """Write ``state`` in the reference's format (stepper.py:355-370)."""
    mesh = state.u_hat.mesh
    header = struct.pack(HEADER, _MAGIC, 1, mesh.n_x, mesh.n_y, mesh.n_z, mesh.l_y, mesh.l_z, config.nu, config.dt,
                         state.t, state.beta, state.kappa, family_code(mesh.family))
    arrays = _arrays(state)
    with open(path, "wb") as fh:
        fh.write(header)
        if not any(is_torch(a) and a.is_cuda for a in arrays):
            for a in arrays:
                a = a.cpu().numpy() if is_torch(a) else a
                fh.write(np.ascontiguousarray(a, dtype="<c16").tobytes())
            return
        import torch

        biggest = max(int(a.numel() if is_torch(a) else np.size(a)) for a in arrays)
        stage = [torch.empty(biggest, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
        events = [None, None]
        copy = torch.cuda.Stream()

        def issue(i):
            a = arrays[i]
            if not is_torch(a):
                a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128))
            buf = stage[i % 2][: a.numel()]
            copy.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(copy):
                buf.copy_(a.reshape(-1).to(torch.complex128), non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            events[i % 2] = (ev, buf)

        issue(0)
        for i in range(len(arrays)):
            ev, buf = events[i % 2]
            ev.synchronize()
            if i + 1 < len(arrays):
                issue(i + 1)  # overlaps the write below (other staging buffer)
            fh.write(buf.numpy().tobytes())


def load_checkpoint(path, device: bool = False):
    """Read a checkpoint (stepper.py:373-401): (state, config, mesh); with
    ``device=True`` the arrays are returned as CUDA tensors."""
    size = struct.calcsize(HEADER)
    with open(path, "rb") as fh:
        raw = fh.read(size)
        if len(raw) != size:
            raise ValueError(f"not a recognized checkpoint file: {path}")
        (magic, version, n_x, n_y, n_z, l_y, l_z, nu, dt, t, beta, kappa, fam) = struct.unpack(HEADER, raw)
        if magic != _MAGIC or version != 1:
            raise ValueError(f"not a recognized checkpoint file: {path}")
        family = PointFamily.GAUSS if fam == 0 else PointFamily.GAUSS_LOBATTO
        mesh = build_mesh(n_x, n_y, n_z, l_y, l_z, family)
        grid_dir = wavenumber_grid(mesh, Space.DIRICHLET)
        grid_bih = wavenumber_grid(mesh, Space.BIHARMONIC)
        yz = mesh.spectral_shape_yz

        def read(grid):
            shape = (grid.n_modes,) + yz
            count = int(np.prod(shape))
            data = fh.read(16 * count)
            if len(data) != 16 * count:
                raise ValueError(f"truncated checkpoint file: {path}")
            arr = np.frombuffer(data, dtype="<c16").reshape(shape).copy()
            if device:
                import torch

                from ._device import device as _dev

                arr = torch.from_numpy(arr).to(_dev())
            return SpectralField(arr, grid, mesh)

        u_hat = read(grid_bih)
        v_hat, w_hat, g_hat = read(grid_dir), read(grid_dir), read(grid_dir)
        h_curr = tuple(read(grid_dir) for _ in range(3))
        h_prev = tuple(read(grid_dir) for _ in range(3))
    return FlowState(u_hat, v_hat, w_hat, g_hat, h_curr, h_prev, beta, t, kappa), StepperConfig(nu, dt), mesh
