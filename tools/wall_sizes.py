"""Wall-normal stage time per route (fused kernel vs extension + cuFFT + post
kernels) across n_x, both families, Dirichlet forward (with mass solve) and
inverse, on 8192 Fourier lines."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import transforms as T  # noqa: E402

L = 8192
res = {}
for n_x in (64, 128, 256, 512, 1024, 2048):
    N = n_x + 1
    g = torch.Generator(device="cuda").manual_seed(0)
    lines = torch.complex(torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64),
                          torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64))
    coef = lines[: n_x - 1].contiguous()
    for fam in (0, 1):
        for route in ("wall", "fft"):
            T.XFORM_METHOD = route
            for kind, fn in (("fwd", lambda: T.wall_forward(lines, n_x, fam, 1, True)),
                             ("inv", lambda: T.wall_inverse(coef, n_x, fam, 1, 1))):
                try:
                    for _ in range(2):
                        fn()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(5):
                        fn()
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / 5
                except Exception as e:  # noqa: BLE001
                    ms = float("nan")
                    print("error", n_x, fam, route, kind, e)
                res[f"n{n_x}_f{fam}_{route}_{kind}"] = ms
                print(f"n_x={n_x:5d} fam={fam} {route:4s} {kind}: {ms * 1e3:9.1f} us  "
                      f"({(N + n_x - 1) * L * 16 / (ms * 1e6):7.0f} GB/s alg)", flush=True)
json.dump(res, open("gpurun_out/wall_sizes.json", "w"), indent=1)
