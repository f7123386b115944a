import sys; sys.path.insert(0, ".")
import numpy as np, torch, time
from paper_1701_03787_b200 import operators as P
from paper_1701_03787_b200.matrices import assemble
mats = assemble(256, 0)
for name in ("stiff_dir", "mass_dir", "stiff_bih"):
    M = getattr(mats, name)
    x = torch.randn(M.shape[1], 1, dtype=torch.complex128, device="cuda")
    for _ in range(3): y = P.apply(M, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): y = P.apply(M, x)
    e1.record(); torch.cuda.synchronize()
    print(name, "ms per apply (incl. launch):", e0.elapsed_time(e1) / 20)
