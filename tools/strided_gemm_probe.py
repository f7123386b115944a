"""Does torch.matmul write into / read from row-strided views without copies
(cuBLAS leading dimensions)?  Times the variants for the transform GEMMs."""
import torch

N, L = 257, 33024
n = 255
M = torch.randn(n, N, dtype=torch.float64, device="cuda")
X = torch.randn(N, 2 * L, dtype=torch.float64, device="cuda")
out = torch.empty(2 * n, 2 * L, dtype=torch.float64, device="cuda")


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


full = torch.empty(n, 2 * L, dtype=torch.float64, device="cuda")
print("contiguous out      %.3f ms" % t(lambda: torch.matmul(M, X, out=full)))
view = out[0::2]
ptr = view.data_ptr()
print("strided out         %.3f ms" % t(lambda: torch.matmul(M, X, out=view)), "same storage:", view.data_ptr() == ptr)
print("correct:", torch.allclose(out[0::2], full))
half = M[:, : N // 2 + 1].contiguous()
Xh = X[: N // 2 + 1].contiguous()
print("half-K contiguous   %.3f ms" % t(lambda: torch.matmul(half[0::2].contiguous(), Xh)))
Xs = X[0::2]
print("strided input rows  %.3f ms" % t(lambda: torch.matmul(M[:, 0::2].contiguous(), Xs)))
