"""Fused attention fwd/bwd throughput at the bench shape (CUDA-graph replay, event-timed),
next to torch SDPA (cuDNN / flash backends) for scale."""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
if len(sys.argv) > 1:  # A/B: another build of the library
    from pathlib import Path
    _lib.SO_PATH = Path(sys.argv[1]).resolve()
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


for b, h, s, causal in ((8, 16, 512, False), (4, 25, 1024, True), (16, 16, 512, False), (32, 16, 512, False)):
    H = h * 64
    qkv = (torch.randn(b * s, 3 * H, device="cuda") * 0.5).bfloat16()
    out = torch.empty(b * s, H, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, h, s, device="cuda")
    dout = torch.randn(b * s, H, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv)
    fl = 4 * b * h * s * s * 64 * (0.5 if causal else 1.0)
    row = {"b": b, "h": h, "s": s, "causal": causal}
    t = graph_time(lambda: k.attn_fwd(qkv, out, lse, b, s, h, causal))
    row["fwd_us"] = round(t * 1e6, 1); row["fwd_tflops"] = round(fl / t / 1e12)
    t = graph_time(lambda: k.attn_bwd(qkv, out, dout, lse, dqkv, b, s, h, causal))
    row["bwd_us"] = round(t * 1e6, 1); row["bwd_tflops"] = round(2.5 * fl / t / 1e12)
    q, kk, v = [qkv[:, i * H:(i + 1) * H].reshape(b, s, h, 64).transpose(1, 2) for i in range(3)]
    from torch.nn.attention import sdpa_kernel, SDPBackend
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                t = graph_time(lambda: torch.nn.functional.scaled_dot_product_attention(q, kk, v, is_causal=causal))
            row[f"{name}_fwd_tflops"] = round(fl / t / 1e12)
            qq, k2, vv = [x.detach().clone().requires_grad_(True) for x in (q, kk, v)]
            with sdpa_kernel([be]):
                o = torch.nn.functional.scaled_dot_product_attention(qq, k2, vv, is_causal=causal)
                go = torch.randn_like(o)
                t = graph_time(lambda: torch.autograd.grad(o, (qq, k2, vv), go, retain_graph=True))
            row[f"{name}_bwd_tflops"] = round(2.5 * fl / t / 1e12)
        except Exception as e:  # noqa: BLE001
            row[name] = str(e)[:80]
    print(json.dumps(row), flush=True)
