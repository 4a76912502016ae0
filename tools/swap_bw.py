"""Swap-engine link bandwidth on the B200 host link: pinned D2H / H2D copies on
a copy stream (the memopt swap path, kernels.copy via torch non_blocking
copies as in runtime/stage.py), alone and while a GEMM stream keeps the SMs
busy, at activation-sized transfers."""
import json, sys, time
import torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)
res = []
cs = torch.cuda.Stream()
gs = torch.cuda.Stream()
x = torch.randn(8192, 8192, device="cuda").bfloat16()
w = torch.randn(8192, 8192, device="cuda").bfloat16()
y = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
for mb in (8, 64, 256):
    n = mb << 20
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    for busy in (False, True):
        for direction in ("d2h", "h2d"):
            reps = 20
            torch.cuda.synchronize()
            if busy:
                with torch.cuda.stream(gs):
                    for _ in range(6):
                        k.gemm_raw(M=8192, N=8192, K=8192, A=x, lda=8192, B=w, ldb=8192, Cout=y, ldc=8192)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            with torch.cuda.stream(cs):
                e0.record(cs)
                for _ in range(reps):
                    if direction == "d2h":
                        host.copy_(dev, non_blocking=True)
                    else:
                        dev.copy_(host, non_blocking=True)
                e1.record(cs)
            torch.cuda.synchronize()
            gbs = reps * n / (e0.elapsed_time(e1) / 1e3) / 1e9
            res.append({"MiB": mb, "dir": direction, "with_gemm": busy, "GB/s": round(gbs, 1)})
            print(json.dumps(res[-1]), flush=True)
# both directions at once (full duplex)
n = 256 << 20
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty_like(d1)
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty_like(h1).pin_memory()
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(cs):
        h1.copy_(d1, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps({"MiB": 256, "dir": "duplex", "GB/s each way": round(10 * n / dt / 1e9, 1)}))
