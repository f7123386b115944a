"""Forward wall-normal stage as fused kernel (stencil + in-kernel mass solve)
vs fused scalar product + the standalone mass-solve kernel (one thread per
(line, parity) over all lines), vs the cuFFT route, per n_x and family."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import transforms as T  # noqa: E402
from paper_1701_03787_b200.wall import wall_plan  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for L in (8192, 33024):
    for n_x in (128, 256, 512, 1024, 2048):
        N = n_x + 1
        g = torch.Generator(device="cuda").manual_seed(0)
        lines = torch.complex(torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64),
                              torch.randn((N, L), generator=g, device="cuda", dtype=torch.float64))
        for fam in (0, 1):
            for sp in (1, 2):
                T.XFORM_METHOD = "wall"
                pl = wall_plan(n_x, fam, sp, 0, True, T._cheb_scale(N, fam))
                tl = pl.struct.log2_lines if pl is not None else -1
                route = T._split_mass
                T._split_mass = lambda *a: False  # the fused kernel with its in-kernel mass solve
                fused = timed(lambda: T.wall_forward(lines, n_x, fam, sp, True))
                T._split_mass = route
                fsp = timed(lambda: T.wall_forward(lines, n_x, fam, sp, False))
                s = T.wall_forward(lines, n_x, fam, sp, False)
                mass = timed(lambda: T._mass_pass(s, sp, n_x, fam, out=torch.empty_like(s)))
                T.XFORM_METHOD = "fft"
                fft = timed(lambda: T.wall_forward(lines, n_x, fam, sp, True))
                print(f"L={L} n_x={n_x:5d} fam={fam} sp={sp} log2TL={tl}: fused {fused:8.1f}  fsp {fsp:8.1f} + mass {mass:7.1f} = "
                      f"{fsp + mass:8.1f}   fft route {fft:8.1f} us", flush=True)
        del lines
