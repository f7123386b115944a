"""One config-4 Helmholtz solve through the chunk-split pair kernel (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import solvers as S  # noqa: E402
from paper_1701_03787_b200.matrices import assemble  # noqa: E402
from paper_1701_03787_b200.mesh import channel_z2  # noqa: E402

mats = assemble(1024, 0)
z2 = channel_z2(2048, 2048)
lu = S.build_helmholtz(mats, 1 / 2000, 1e-4, z2)
g = torch.Generator(device="cuda").manual_seed(1)
rhs = torch.complex(torch.randn((mats.n_dir, z2.size), generator=g, device="cuda", dtype=torch.float64),
                    torch.randn((mats.n_dir, z2.size), generator=g, device="cuda", dtype=torch.float64))
out = torch.empty_like(rhs)
S.HELM_SPLIT = 1
lu.solve_into(rhs, out, True)
torch.cuda.synchronize()
