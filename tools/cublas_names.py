"""cuBLAS kernel choices for the block's GEMM shapes (run under ncu to read the names)."""
import torch

dev = torch.device("cuda", 0)
for m, n, k, ta, tb in ((16384, 28672, 4096, 0, 0), (16384, 4096, 28672, 0, 1), (4096, 28672, 16384, 1, 0),
                        (8192, 8192, 8192, 0, 0), (16384, 4096, 4096, 0, 0)):
    a = torch.randn((k, m) if ta else (m, k), device=dev, dtype=torch.bfloat16)
    b = torch.randn((n, k) if tb else (k, n), device=dev, dtype=torch.bfloat16)
    A = a.t() if ta else a
    B = b.t() if tb else b
    for _ in range(2):
        torch.matmul(A, B)
torch.cuda.synchronize()
