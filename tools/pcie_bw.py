"""Pinned host <-> device copy bandwidth on this box: 1-D copies one way and
both ways concurrently, and the 2-D column-slab copies the pipelined solve
uses (bytes per direction / s)."""
import sys
import time

sys.path.insert(0, ".")

import torch

from paper_1701_03787_b200 import _lib

n = 1 << 30  # 1 GiB per buffer
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D 1-D      {n / t / 1e9:6.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H 1-D      {n / t / 1e9:6.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t = timed(both)
print(f"H2D+D2H 1-D  {n / t / 1e9:6.1f} GB/s each way")
# 2-D: 1023 rows, pitch 4 MiB, 16 slabs of 256 KiB per row
lib = _lib.lib()
rows, pitch = 256, 4 << 20
w = pitch // 16


def both2d():
    for k in range(16):
        with torch.cuda.stream(s1):
            lib.shen_memcpy2d_async(d_a.data_ptr() + k * w, pitch, h_in.data_ptr() + k * w, pitch, w, rows, 0,
                                    s1.cuda_stream)
        with torch.cuda.stream(s2):
            lib.shen_memcpy2d_async(h_out.data_ptr() + k * w, pitch, d_b.data_ptr() + k * w, pitch, w, rows, 1,
                                    s2.cuda_stream)


t = timed(both2d)
print(f"H2D+D2H 2-D  {rows * pitch / t / 1e9:6.1f} GB/s each way (16 column slabs)")
