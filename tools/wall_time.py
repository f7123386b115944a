"""Time the wall-normal stage (fused kernel vs the GEMM and cuFFT routes) at
BASELINE config 3 size: (257 points, 256 x 129 Fourier lines)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import transforms as T  # noqa: E402

N, L = 257, 256 * 129
g = torch.Generator(device="cuda").manual_seed(0)
lines = torch.complex(torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64),
                      torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64))
res = {}
for method in [a for a in sys.argv[1:] if not a.startswith("--")] or ["wall"]:
    T.XFORM_METHOD = method
    for fam in (0, 1):
        for sp in (1, 2):
            for kind in ("fwd", "fsp", "inv"):
                if kind in ("fwd", "fsp"):
                    fn = lambda: T.wall_forward(lines, 256, fam, sp, kind == "fwd")  # noqa: E731
                    nin, nout = N, 256 - 1 if sp == 1 else 256 - 3
                else:
                    coef = lines[: (255 if sp == 1 else 253)].contiguous()
                    fn = lambda: T.wall_inverse(coef, 256, fam, sp, 65536)  # noqa: E731
                    nin, nout = (255 if sp == 1 else 253), N
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                gbs = (nin + nout) * L * 16 / (ms * 1e6)
                res[f"{method}_f{fam}_s{sp}_{kind}"] = {"ms": ms, "GBps_alg": gbs}
                print(method, fam, sp, kind, f"{ms*1e3:.1f} us  {gbs:.0f} GB/s", flush=True)
import os
tag = os.environ.get("SHEN_LIB_VARIANT", "") or "product"
json.dump(res, open(f"gpurun_out/wall_time_{tag}.json", "w"), indent=1)
