"""Clock-normalised GEMM comparison: our tcgen05 GEMM vs cuBLAS, each run for
~2 s in CUDA-graph loops while nvidia-smi samples the SM clock and power, so
throughput can be compared per MHz (under the 1 kW cap the clock depends on
the kernel's power draw).  Prints JSON lines."""
import json, statistics, sys, time
import torch
sys.path.insert(0, ".")
from bench import Clocks
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)


def run(fn, fl, seconds=2.0, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay(); torch.cuda.synchronize()
    c = Clocks(0); c.start(); time.sleep(0.3)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < seconds:
        g.replay(); n += 1
        if n % 4 == 0:
            torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    clk = c.stop()
    tf = fl * reps * n / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return {"tflops": round(tf), "sm_mhz": clk.get("sm_mhz"), "power_w_max": clk.get("power_w_max"),
            "tflops_per_ghz": round(tf / (clk["sm_mhz"] / 1e3)) if clk.get("sm_mhz") else None}


for M, N, K in ((16384, 4096, 1024), (16384, 1024, 4096), (8192, 8192, 8192)):
    x = torch.randn(M, K, device="cuda").bfloat16(); w = torch.randn(N, K, device="cuda").bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * K
    for rnd in range(2):
        ours = run(lambda: k.gemm_raw(M=M, N=N, K=K, A=x, lda=K, B=w, ldb=K, Cout=y, ldc=N), fl)
        cub = run(lambda: torch.matmul(x, w.t(), out=y), fl)
        print(json.dumps({"shape": [M, N, K], "round": rnd, "ours": ours, "cublas": cub}), flush=True)
