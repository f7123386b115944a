"""Device-timed fused RHS assembly (rhs.py) on a config-4 kx slab: ms per
call and achieved HBM GB/s on algorithmic bytes (rhs_g: 5 complex inputs +
1 output per unknown = 96 B; rhs_u: 7 + 1 = 128 B), next to the oracle port
(numpy, reference arithmetic) on a small slab on one core."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import shen_oracle as O  # noqa: E402
from paper_1701_03787_b200 import rhs as H  # noqa: E402
from paper_1701_03787_b200.matrices import assemble  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n_y, n_z, n_x, nu, dt = 2048, 2048, 1024, 1 / 2000, 1e-4
m = (2 * np.pi * np.fft.fftfreq(n_y, 1.0 / n_y) / (2 * np.pi))[:rows, None]
n = (2 * np.pi * np.fft.rfftfreq(n_z, 1.0 / n_z) / np.pi)[None, :]
z2 = m ** 2 + n ** 2
mats = assemble(n_x, 0)
L = z2.size
g = torch.Generator(device="cuda").manual_seed(0)


PAD = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # bytes of skew between the arrays (DRAM-partition probe)


def rnd(r):
    if not PAD:
        return torch.randn((r, rows, n.shape[1]), dtype=torch.complex128, device="cuda", generator=g)
    cnt = r * rows * n.shape[1]
    buf = torch.empty(cnt + PAD * (1 + len(_keep)) // 16, dtype=torch.complex128, device="cuda")
    _keep.append(buf)
    off = PAD * len(_keep) // 16
    t = buf[off:off + cnt].view(r, rows, n.shape[1])
    t.copy_(torch.randn((r, rows, n.shape[1]), dtype=torch.complex128, device="cuda", generator=g))
    return t


_keep = []


u, gg = rnd(mats.n_bih), rnd(mats.n_dir)
hc = [rnd(mats.n_dir) for _ in range(3)]
hp = [rnd(mats.n_dir) for _ in range(3)]
asm = H.RhsAssembler(mats, nu, dt, z2, m, n)
res = {}
for name, fn, nrow, nbytes in (("rhs_g", lambda: asm.rhs_g(gg, hc, hp), mats.n_dir, 96),
                               ("rhs_u", lambda: asm.rhs_u(u, hc, hp), mats.n_bih, 128)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    unk = nrow * L
    res[name] = {"ms": ms, "unknowns_per_s": unk / (ms / 1e3), "GBps_alg": nbytes * unk / (ms / 1e3) / 1e9,
                 "alg_bytes_per_unknown": nbytes}
# CPU oracle on 4 kx rows, one core
sl = slice(0, 4)
hc_h = [h[:, sl].cpu().numpy() for h in hc]
hp_h = [h[:, sl].cpu().numpy() for h in hp]
t0 = time.perf_counter()
hab = O.ab2(hc_h, hp_h)
O.assemble_rhs_g(mats, nu, dt, z2[sl], m[sl], n, gg[:, sl].cpu().numpy(), hab)
O.assemble_rhs_u(mats, nu, dt, z2[sl], m[sl], n, u[:, sl].cpu().numpy(), hab)
t = time.perf_counter() - t0
res["cpu_oracle_unknowns_per_s"] = (mats.n_dir + mats.n_bih) * 4 * n.shape[1] / t
res["config"] = f"config-4 plane, kx rows 0..{rows - 1} ({L} lines), n_x = {n_x}"
print(json.dumps(res))
