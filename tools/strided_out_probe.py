"""Does torch.matmul write a row-strided out= view in place (cuBLAS ldc), or via a temporary + copy?"""
import torch

A = torch.randn(128, 129, dtype=torch.float64, device="cuda")
B = torch.randn(129, 66048, dtype=torch.float64, device="cuda")
C = torch.zeros(256, 66048, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.matmul(A, B, out=C[0::2])
torch.cuda.synchronize()
ref = A @ B
print("max err", (C[0::2] - ref).abs().max().item(), "odd rows untouched", C[1::2].abs().max().item())
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    torch.matmul(A, B, out=C[0::2])
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8))
