"""Multi-tile-per-CTA check of the persistent wall kernels (debugging aid)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import transforms as T  # noqa: E402

which = sys.argv[1]
L = int(sys.argv[2])
N = 257
g = torch.Generator(device="cuda").manual_seed(0)
lines = torch.complex(torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64),
                      torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64))
if which == "inv":
    x, _ = T.wall_inverse(lines[:255].contiguous(), 256, 0, 1, 1)
else:
    x = T.wall_forward(lines, 256, 0, 1, True)
torch.cuda.synchronize()
print(which, L, "ok", float(x.abs().max()))
