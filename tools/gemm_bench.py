"""GEMM throughput at the BERT-large / GPT-2 XL shapes vs cuBLAS (torch.matmul)."""
import sys, json
import torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k

_lib.init_device(0)
def timeit(fn, iters=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3

shapes = [("qkv", 4096, 3072, 1024), ("proj", 4096, 1024, 1024), ("fc1", 4096, 4096, 1024),
          ("fc2", 4096, 1024, 4096), ("head", 4096, 30528, 1024), ("big", 8192, 8192, 8192),
          ("gpt_fc1", 8192, 6400, 1600), ("gpt_fc2", 8192, 1600, 6400)]
rows = []
for name, M, N, K in shapes:
    x = torch.randn(M, K, device="cuda").bfloat16(); w = torch.randn(N, K, device="cuda").bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn(M, N, device="cuda").bfloat16(); dx = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
    dw = torch.empty(N, K, device="cuda")
    fl = 2 * M * N * K
    r = {"name": name, "M": M, "N": N, "K": K}
    r["fwd"] = fl / timeit(lambda: k.linear_fwd(x, w, y)) / 1e12
    r["dgrad"] = fl / timeit(lambda: k.linear_dgrad(dy, w, dx)) / 1e12
    r["wgrad"] = fl / timeit(lambda: k.linear_wgrad(dy, x, dw)) / 1e12
    r["cublas_fwd"] = fl / timeit(lambda: torch.matmul(x, w.t(), out=y)) / 1e12
    rows.append(r); print(json.dumps({a: (round(b, 1) if isinstance(b, float) else b) for a, b in r.items()}), flush=True)
