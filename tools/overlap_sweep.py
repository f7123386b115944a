"""Sweep the SM split of a concurrent Helmholtz + biharmonic streaming solve
(config 4 slab): H on max_ctas = x SMs on one stream, B on the rest on another.
Prints ms per pair for each x (device-timed)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1701_03787_b200 import solvers as S  # noqa: E402
from paper_1701_03787_b200.matrices import assemble  # noqa: E402
from paper_1701_03787_b200.mesh import channel_z2  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
splits = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [40, 48, 56, 64, 72, 80]
mats = assemble(1024, 0)
z2 = np.ascontiguousarray(channel_z2(2048, 2048)[:rows])
hlu = S.build_helmholtz(mats, 1 / 2000, 1e-4, z2)
blu = S.build_biharmonic(mats, 1 / 2000, 1e-4, z2)
B = z2.size
g = torch.Generator(device="cuda").manual_seed(1)
fh = torch.randn((mats.n_dir, B), dtype=torch.complex128, device="cuda", generator=g)
fb = torch.randn((mats.n_bih, B), dtype=torch.complex128, device="cuda", generator=g)
xh, xb = torch.empty_like(fh), torch.empty_like(fb)
sms = torch.cuda.get_device_properties(0).multi_processor_count
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def seq():
    hlu.solve_into(fh, xh, True)
    blu.solve_into(fb, xb, True)


def pair(x):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        hlu.solve_into(fh, xh, True, max_ctas=x)
    with torch.cuda.stream(s2):
        blu.solve_into(fb, xb, True, max_ctas=sms - x)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("sequential", round(timeit(seq), 2), "ms", flush=True)
ref = xh[:, ::97].clone(), xb[:, ::97].clone()  # sampled columns (memory)
for x in splits:
    t = timeit(lambda: pair(x))
    ok = torch.equal(xh[:, ::97], ref[0]) and torch.equal(xb[:, ::97], ref[1])
    print("H on", x, "SMs, B on", sms - x, ":", round(t, 2), "ms", "identical" if ok else "MISMATCH", flush=True)
