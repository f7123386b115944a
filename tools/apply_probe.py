"""Time the structured apply (operators.apply) on a few lines (staged kernel)
and on the config-3 Fourier lines (one thread per (line, parity))."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1701_03787_b200 import operators as P  # noqa: E402
from paper_1701_03787_b200.matrices import assemble  # noqa: E402

mats = assemble(256, 0)
for L in (1, 256 * 129):
    for name in ("stiff_dir", "mass_dir", "stiff_bih", "deriv_dir_to_cheb", "fourth_bih"):
        M = getattr(mats, name)
        x = torch.randn(M.shape[1], L, dtype=torch.complex128, device="cuda")
        for _ in range(3):
            y = P.apply(M, x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            y = P.apply(M, x)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        gb = (M.shape[0] + M.shape[1]) * L * 16 / 1e9
        print(f"L={L} {name}: {ms * 1e3:.1f} us per apply  {gb / ms * 1e3:.0f} GB/s", flush=True)
