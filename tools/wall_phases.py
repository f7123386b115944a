"""Per-CTA phase durations of the fused forward wall-normal kernel at C3
size, from the clock64 stamps of a -DSHEN_WALL_TIMING variant library
(bash tools/ab_build_tu.sh ts shen_wall paper_1701_03787_b200/csrc/shen_wall.cu
-DSHEN_WALL_TIMING; run with SHEN_LIB_VARIANT=ts)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import _lib, transforms as T  # noqa: E402
_lib._SIGS["shen_wall_ts_read"] = (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t])

N, L = 257, 256 * 129
g = torch.Generator(device="cuda").manual_seed(0)
lines = torch.complex(torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64),
                      torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64))
for fam in (0, 1):
    for sp in (1, 2):
        for mass in (True, False):
            for _ in range(3):
                T.wall_forward(lines, 256, fam, sp, mass)
            torch.cuda.synchronize()
            buf = np.zeros((1 << 16, 6), dtype=np.int64)
            assert _lib.lib().shen_wall_ts_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
            ntile = int((buf[:, 4] > 0).sum())
            b = buf[:ntile]
            d = np.diff(b[:, :5], axis=1)
            span = (b[:, 4].max() - b[:, 0].min())
            per_sm = np.bincount(b[:, 5].astype(int))
            print(f"fam {fam} sp {sp} mass {int(mass)}: tiles {ntile}, per-SM {per_sm.min()}-{per_sm.max()}, "
                  f"mean cycles load {d[:,0].mean():.0f} dft {d[:,1].mean():.0f} stencil/mass {d[:,2].mean():.0f} "
                  f"store {d[:,3].mean():.0f} | life {(b[:,4]-b[:,0]).mean():.0f} | span {span} cyc", flush=True)
