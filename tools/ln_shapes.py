import sys, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)
rows, cols = 4096, 1024
x = torch.randn(rows, cols, device="cuda").bfloat16(); g = torch.randn(cols, device="cuda").bfloat16()
dy = torch.randn(rows, cols, device="cuda").bfloat16(); dx = torch.empty_like(x)
mean = torch.zeros(rows, device="cuda"); rstd = torch.ones(rows, device="cuda")
dg = torch.zeros(cols, device="cuda"); db = torch.zeros(cols, device="cuda")
for _ in range(3):
    k.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dx_add=dx)
    k.colsum(dy, dg)
torch.cuda.synchronize(); print("ok")
