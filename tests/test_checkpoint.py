"""Checkpoint wire format (checkpoint.py) against files written by the
reference's save_checkpoint (tests/golden/checkpoint_f*.bin): reading them
recovers the state exactly, writing the same state reproduces the bytes --
from host arrays here, from device tensors in the GPU test."""

import os

import numpy as np
import pytest

from paper_1701_03787_b200 import checkpoint as C

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _check_state(state, g, k):
    d = (lambda x: x.cpu().numpy()) if hasattr(state.u_hat.data, "cpu") else (lambda x: x)
    assert np.array_equal(d(state.u_hat.data), g[k + "_u"])
    assert np.array_equal(d(state.v_hat.data), g[k + "_v"])
    assert np.array_equal(d(state.w_hat.data), g[k + "_w"])
    assert np.array_equal(d(state.g_hat.data), g[k + "_g"])
    for i in range(3):
        assert np.array_equal(d(state.h_curr[i].data), g[f"{k}_hc{i}"])
        assert np.array_equal(d(state.h_prev[i].data), g[f"{k}_hp{i}"])
    assert (state.beta, state.t, state.kappa) == (0.25, 1.5, 7)


@pytest.mark.parametrize("fi", [0, 1])
def test_read_and_rewrite_reference_checkpoint(golden, tmp_path, fi):
    g = golden("rhs.npz")
    path = os.path.join(GOLD, f"checkpoint_f{fi}.bin")
    state, cfg, mesh = C.load_checkpoint(path)
    assert (cfg.nu, cfg.dt) == (1e-2, 1e-3) and (mesh.n_x, mesh.n_y, mesh.n_z) == (16, 8, 8)
    _check_state(state, g, f"f{fi}")
    out = tmp_path / "re.bin"
    C.save_checkpoint(out, state, cfg)
    assert out.read_bytes() == open(path, "rb").read()


def test_bad_files(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOTACHKP" + b"\0" * 100)
    with pytest.raises(ValueError):
        C.load_checkpoint(p)
    good = open(os.path.join(GOLD, "checkpoint_f0.bin"), "rb").read()
    p.write_bytes(good[:-16])
    with pytest.raises(ValueError, match="truncated"):
        C.load_checkpoint(p)


@pytest.mark.gpu
def test_device_state_round_trip(golden, tmp_path):
    """load to CUDA tensors, save from them (staged, overlapped D2H): same bytes."""
    g = golden("rhs.npz")
    path = os.path.join(GOLD, "checkpoint_f1.bin")
    state, cfg, _ = C.load_checkpoint(path, device=True)
    assert state.u_hat.data.is_cuda
    _check_state(state, g, "f1")
    out = tmp_path / "dev.bin"
    C.save_checkpoint(out, state, cfg)
    assert out.read_bytes() == open(path, "rb").read()
