"""A/B of the LayerNorm kernels between library builds at the bench shapes
(b=64 / b=32 BERT-large rows x 1024): fused backward and forward, algorithmic GB/s.
    python tools/ln_ab.py path/to/_dawnpiper.so"""
import json, sys
from pathlib import Path
import torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib
if len(sys.argv) > 1:
    _lib.SO_PATH = Path(sys.argv[1]).resolve()
from paper_2505_05856_b200 import kernels as k
_lib.init_device(0)


def graph_time(fn, reps=30):
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


row = {"so": _lib.SO_PATH.name}
for rows, cols in ((32768, 1024), (16384, 1024)):
    x = torch.randn(rows, cols, device="cuda").bfloat16()
    dy = torch.randn(rows, cols, device="cuda").bfloat16()
    dx = torch.randn(rows, cols, device="cuda").bfloat16()
    y = torch.empty_like(x)
    g = torch.randn(cols, device="cuda").bfloat16(); bt = torch.randn(cols, device="cuda").bfloat16()
    mean = torch.randn(rows, device="cuda"); rstd = torch.rand(rows, device="cuda") + 0.5
    dg = torch.zeros(cols, device="cuda"); db = torch.zeros(cols, device="cuda")
    dbias = torch.zeros(cols, device="cuda")
    t = graph_time(lambda: k.layernorm_bwd_fused(dy, x, g, mean, rstd, dx, dg, db, dx_add=dx, dbias=dbias))
    row[f"bwd{rows}_GBps"] = round(8 * rows * cols / t / 1e9)
    t = graph_time(lambda: k.layernorm_fwd(x, g, bt, y, mean, rstd))
    row[f"fwd{rows}_GBps"] = round(4 * rows * cols / t / 1e9)
print(json.dumps(row), flush=True)
