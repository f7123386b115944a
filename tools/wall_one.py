"""One forward and one inverse wall-normal launch at config-3 size (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import transforms as T  # noqa: E402

fam = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sp = int(sys.argv[2]) if len(sys.argv) > 2 else 2
N, L = 257, 256 * 129
g = torch.Generator(device="cuda").manual_seed(0)
lines = torch.complex(torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64),
                      torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64))
for _ in range(2):
    c = T.wall_forward(lines, 256, fam, sp, True)
    x, _n = T.wall_inverse(c, 256, fam, sp, 65536)
torch.cuda.synchronize()
print("ok", c.shape, x.shape)
