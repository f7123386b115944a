"""Per-CTA phase durations of the plane rfft2 kernel (257 planes of 256 x 256),
from the %globaltimer stamps of a -DSHEN_PF_TIMING variant library
(bash tools/ab_build_tu.sh ts shen_plane_fft paper_1701_03787_b200/csrc/shen_plane_fft.cu
-DSHEN_PF_TIMING; run with SHEN_LIB_VARIANT=ts)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import _lib  # noqa: E402
from paper_1701_03787_b200._device import stream_handle  # noqa: E402

_lib._SIGS["shen_pf_ts_read"] = (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t])
P = int(sys.argv[1]) if len(sys.argv) > 1 else 257
x = torch.rand((P, 256, 256), dtype=torch.float64, device="cuda")
X = torch.empty((P, 256, 129), dtype=torch.complex128, device="cuda")
lib = _lib.lib()
for _ in range(3):
    _lib.check(lib.shen_plane_rfft2(P, 256, 256, x.data_ptr(), X.data_ptr(), stream_handle()), "rfft2")
torch.cuda.synchronize()
buf = np.zeros((1 << 16, 10), dtype=np.int64)
assert lib.shen_pf_ts_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
b = buf[: 16 * P]
t0 = b[:, 0].min()
d = np.diff(b[:, :7], axis=1)
names = ["load", "z", "y1+barrier", "remote ld", "dft+st", "final wait"]
print("mean ns:", " ".join(f"{n} {d[:, i].mean():.0f}" for i, n in enumerate(names)))
print("p90 ns: ", " ".join(f"{n} {np.percentile(d[:, i], 90):.0f}" for i, n in enumerate(names)))
life = b[:, 6] - b[:, 0]
print(f"life mean {life.mean():.0f} ns, span {(b[:, 6].max() - t0) / 1e3:.1f} us, "
      f"first-wave starts {np.sort(b[:, 0] - t0)[:8]} ... last start {(b[:, 0].max() - t0) / 1e3:.1f} us")
per_sm = np.bincount(b[:, 9].astype(int), minlength=148)
print("CTAs per SM min/max", per_sm.min(), per_sm.max(), "SMs used", int((per_sm > 0).sum()))
# concurrency over time
ev = np.concatenate([np.stack([b[:, 0], np.ones(len(b))], 1), np.stack([b[:, 6], -np.ones(len(b))], 1)])
ev = ev[np.argsort(ev[:, 0], kind="stable")]
conc = np.cumsum(ev[:, 1])
print("max concurrent CTAs", int(conc.max()), "time-avg concurrent",
      float((conc[:-1] * np.diff(ev[:, 0])).sum() / (ev[-1, 0] - ev[0, 0])))
