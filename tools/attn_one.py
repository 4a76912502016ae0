"""A few attention launches at the bench shape (b32 h16 s512) for ncu captures."""
import sys, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)
b, h, s = 32, 16, 512
H = h * 64
qkv = (torch.randn(b * s, 3 * H, device="cuda") * 0.5).bfloat16()
out = torch.empty(b * s, H, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, h, s, device="cuda")
dout = torch.randn(b * s, H, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
for _ in range(3):
    k.attn_fwd(qkv, out, lse, b, s, h, False)
    k.attn_bwd(qkv, out, dout, lse, dqkv, b, s, h, False)
torch.cuda.synchronize()
print("done")
