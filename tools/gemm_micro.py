"""Pure-GPU GEMM throughput: launches captured in a CUDA graph, replayed, event-timed."""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)

def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3

shapes = [(4096, 4096, 1024), (4096, 4096, 4096), (8192, 8192, 8192), (4096, 1024, 1024), (4096, 3072, 1024), (16384, 4096, 1024), (16384, 1024, 4096), (16384, 3072, 1024)]
for M, N, K in shapes:
    x = torch.randn(M, K, device="cuda").bfloat16(); w = torch.randn(N, K, device="cuda").bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * K
    row = {"shape": (M, N, K)}
    for bn, cg in ((256, 4), (256, 2), (128, 2), (256, 1)):
        t = graph_time(lambda: k.gemm_raw(M=M, N=N, K=K, A=x, lda=K, B=w, ldb=K, Cout=y, ldc=N, block_n=bn, cta_group=cg))
        row[f"{bn}x{cg}"] = round(fl / t / 1e12)
    t = graph_time(lambda: torch.matmul(x, w.t(), out=y))
    row["cublas"] = round(fl / t / 1e12)
    print(json.dumps(row), flush=True)
