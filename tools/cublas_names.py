"""Which cuBLAS kernels (tile / cluster encoded in the name) run at the step's GEMM shapes."""
import torch
shapes = [(4096, 1024, 1024), (4096, 3072, 1024), (4096, 4096, 1024), (4096, 1024, 4096), (8192, 8192, 8192)]
for M, N, K in shapes:
    x = torch.randn(M, K, device="cuda").bfloat16(); w = torch.randn(N, K, device="cuda").bfloat16()
    for _ in range(3):
        torch.matmul(x, w.t())
torch.cuda.synchronize()
