"""A/B GEMM throughput of two builds of the library on the same box:
    python tools/gemm_ab.py path/to/_dawnpiper.so  (prints JSON lines)
BERT-large b=32 shapes through the executor's entry points (plain, bias,
GELU+aux, residual epilogues; f32 wgrad), CUDA-graph replay, event-timed."""
import json, sys
from pathlib import Path
import torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib
if len(sys.argv) > 1:
    _lib.SO_PATH = Path(sys.argv[1]).resolve()
from paper_2505_05856_b200 import kernels as k
_lib.init_device(0)


def graph_time(fn, reps=20):
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


M = int(__import__("os").environ.get("GEMM_AB_M", "24576"))
row = {"so": str(_lib.SO_PATH.name)}
for name, N, K in (("qkv", 3072, 1024), ("proj", 1024, 1024), ("fc1", 4096, 1024), ("fc2", 1024, 4096), ("big", 8192, 8192)):
    m = M if name != "big" else 8192
    x = torch.randn(m, K, device="cuda").bfloat16()
    w = torch.randn(N, K, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda").bfloat16()
    y = torch.empty(m, N, device="cuda", dtype=torch.bfloat16)
    aux = torch.empty_like(y)
    res = torch.randn(m, N, device="cuda").bfloat16()
    dy = torch.randn(m, N, device="cuda").bfloat16()
    dw = torch.empty(N, K, device="cuda")
    fl = 2 * m * N * K
    row[f"{name}_plain"] = round(fl / graph_time(lambda: k.gemm_raw(M=m, N=N, K=K, A=x, lda=K, B=w, ldb=K, Cout=y, ldc=N)) / 1e12)
    if name == "fc1":
        row[f"{name}_gelu_aux"] = round(fl / graph_time(lambda: k.linear_fwd(x, w, y, bias=bias, gelu=True, aux=aux)) / 1e12)
    if name == "fc2":
        row[f"{name}_res"] = round(fl / graph_time(lambda: k.linear_fwd(x, w, y, bias=bias, residual=res)) / 1e12)
    if name in ("fc1", "qkv"):
        row[f"{name}_wgrad"] = round(fl / graph_time(lambda: k.linear_wgrad(dy, x, dw)) / 1e12)
    if name in ("fc2", "big"):
        row[f"{name}_cublas"] = round(fl / graph_time(lambda: torch.matmul(x, w.t(), out=y)) / 1e12)
print(json.dumps(row), flush=True)
