"""Plane FFT kernels (shen_plane_fft.cu) against numpy and cuFFT: accuracy on
a few planes, then timing at the config-3 size (257 planes of 256 x 256) and
at the nonlinear term's 8-field batch.  Writes gpurun_out/plane_fft.json."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import _lib  # noqa: E402
from paper_1701_03787_b200._device import stream_handle  # noqa: E402

NY = NZ = 256
lib = _lib.lib()


def rfft2(x):
    X = torch.empty((x.shape[0], NY, NZ // 2 + 1), dtype=torch.complex128, device=x.device)
    _lib.check(lib.shen_plane_rfft2(x.shape[0], NY, NZ, x.data_ptr(), X.data_ptr(), stream_handle()), "rfft2")
    return X


def irfft2(X, scale):
    x = torch.empty((X.shape[0], NY, NZ), dtype=torch.float64, device=X.device)
    _lib.check(lib.shen_plane_irfft2(X.shape[0], NY, NZ, X.data_ptr(), x.data_ptr(), ctypes.c_double(scale),
                                     stream_handle()), "irfft2")
    return x


res = {}
rng = np.random.default_rng(0)
xs = rng.uniform(-1, 1, (5, NY, NZ))
x = torch.from_numpy(xs).cuda()
X = rfft2(x).cpu().numpy()
want = np.fft.rfft2(xs)
res["rfft2_max_rel"] = float(np.abs(X - want).max() / np.abs(want).max())
Xs = want + 1j * 0  # Hermitian-consistent input
Xs = Xs.copy()
Xs[:, :, 0] += 0.3j * rng.standard_normal((5, NY))  # imaginary parts numpy ignores
Xs[:, :, -1] += 0.3j * rng.standard_normal((5, NY))
back = irfft2(torch.from_numpy(Xs).cuda(), 1.0 / (NY * NZ)).cpu().numpy()
wantb = np.fft.irfft2(Xs, s=(NY, NZ))
res["irfft2_max_rel"] = float(np.abs(back - wantb).max() / np.abs(wantb).max())
Xr = rng.standard_normal((5, NY, NZ // 2 + 1)) + 1j * rng.standard_normal((5, NY, NZ // 2 + 1))
back = irfft2(torch.from_numpy(Xr).cuda(), 1.0).cpu().numpy()
wantr = np.fft.irfft2(Xr, s=(NY, NZ), norm="forward")
res["irfft2_general_max_rel"] = float(np.abs(back - wantr).max() / np.abs(wantr).max())
print(res, flush=True)


def timeit(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


for P in (257, 8 * 257):
    x = torch.rand((P, NY, NZ), dtype=torch.float64, device="cuda")
    X = torch.fft.rfft2(x)
    byts = P * NY * (NZ * 8 + (NZ // 2 + 1) * 16)
    for name, fn in (("shen_rfft2", lambda: rfft2(x)), ("cufft_rfft2", lambda: torch.fft.rfft2(x)),
                     ("shen_irfft2", lambda: irfft2(X, 1.0)),
                     ("cufft_irfft2", lambda: torch.fft.irfft2(X, s=(NY, NZ), norm="forward"))):
        ms = timeit(fn)
        res[f"{name}_P{P}"] = {"ms": ms, "GBps": byts / ms / 1e6}
        print(name, P, f"{ms * 1e3:.1f} us  {byts / ms / 1e6:.0f} GB/s", flush=True)
json.dump(res, open("gpurun_out/plane_fft.json", "w"), indent=1)
