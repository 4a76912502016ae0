"""LayerNorm backward A/B at the bench shapes: ln_dx + column reduction (+ the
separate bias colsum) vs the one-pass fused kernel (CUDA-graph replay, events).

    python tools/ln_micro.py
"""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)


def graph_time(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


for rows, cols in ((16384, 1024), (4096, 1024), (16384, 1600), (1024, 768), (8192, 2048)):
    x = torch.randn(rows, cols, device="cuda").bfloat16()
    dy = torch.randn(rows, cols, device="cuda").bfloat16()
    dx = torch.randn(rows, cols, device="cuda").bfloat16()
    g = torch.randn(cols, device="cuda").bfloat16()
    mean = torch.randn(rows, device="cuda"); rstd = torch.rand(rows, device="cuda") + 0.5
    dg = torch.zeros(cols, device="cuda"); db = torch.zeros(cols, device="cuda")
    dbias = torch.zeros(cols, device="cuda")
    def old():
        k.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dx_add=dx)
        k.colsum(dx, dbias)
    def fused():
        k.layernorm_bwd_fused(dy, x, g, mean, rstd, dx, dg, db, dx_add=dx, dbias=dbias)
    t_old, t_new = graph_time(old), graph_time(fused)
    alg = 8 * rows * cols  # read dy, x, dx_add, write dx (bf16)
    print(json.dumps({"rows": rows, "cols": cols, "old_us": round(t_old * 1e6, 1),
                      "fused_us": round(t_new * 1e6, 1), "speedup": round(t_old / t_new, 2),
                      "fused_GBps_alg": round(alg / t_new / 1e9)}), flush=True)
