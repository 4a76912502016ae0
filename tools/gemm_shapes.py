"""Run a few pipeline GEMM shapes in isolation (for ncu captures)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)
b, s, A, d = 8, 512, 16, 64
H = A * d
qkv = torch.randn(b * s, 3 * H, device="cuda").bfloat16()
S = torch.empty(b, A, s, s, device="cuda", dtype=torch.bfloat16)
x = torch.randn(b * s, H, device="cuda").bfloat16()
w = torch.randn(H, H, device="cuda").bfloat16()
y = torch.empty(b * s, H, device="cuda", dtype=torch.bfloat16)
w1 = torch.randn(4 * H, H, device="cuda").bfloat16()
y1 = torch.empty(b * s, 4 * H, device="cuda", dtype=torch.bfloat16)
which = sys.argv[1:] or ["score", "proj", "fc1"]
for it in range(3):
    if "score" in which:
        k.gemm_raw(M=s, N=s, K=d, A=qkv, lda=3 * H, a_s=(d, s * 3 * H), B=qkv[:, H:], ldb=3 * H,
                   b_s=(d, s * 3 * H), batch1=A, batch2=b, Cout=S, ldc=s, c_s=(s * s, A * s * s))
    if "proj" in which:
        k.linear_fwd(x, w, y)
    if "fc1" in which:
        k.linear_fwd(x, w1, y1)
torch.cuda.synchronize()
print("ok")
