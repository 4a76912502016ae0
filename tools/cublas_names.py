"""Which cuBLAS kernels (tile / cluster encoded in the name) run at the step's GEMM shapes,
and their CUDA-event TFLOP/s (torch.profiler lists the kernel names)."""
import torch
from torch.profiler import ProfilerActivity, profile

shapes = [(24576, 1024, 1024), (24576, 3072, 1024), (24576, 4096, 1024), (24576, 1024, 4096),
          (4096, 1024, 1024), (4096, 3072, 1024), (8192, 8192, 8192)]
for M, N, K in shapes:
    x = torch.randn(M, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    for _ in range(3):
        torch.matmul(x, w.t())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        torch.matmul(x, w.t())
    e1.record()
    torch.cuda.synchronize()
    tf = 2 * M * N * K / (e0.elapsed_time(e1) / 20 * 1e-3) / 1e12
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.matmul(x, w.t())
        torch.cuda.synchronize()
    names = sorted({e.name for e in prof.events() if e.device_type.name == "CUDA"})
    print(f"{M}x{N}x{K}: {tf:.0f} TFLOP/s {names}", flush=True)
