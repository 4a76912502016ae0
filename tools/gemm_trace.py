"""Where GEMM time goes, per role (debug trace in gemm.cu): wait cycles per CTA for
the TMA producer (empty slots), the MMA issuer (full slots / free accumulator),
the epilogue (accumulator ready) and its busy time, at the pipeline's shapes."""
import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import _lib, kernels as k
_lib.init_device(0)
lib = _lib.lib()
lib.dpn_gemm_debug_trace.argtypes = [ctypes.c_void_p]
lib.dpn_gemm_debug_trace.restype = None
tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
bf = torch.bfloat16
M = 4096
cases = [  # name, M, N, K, a_mn, b_mn, f32, epilogue kwargs
    ("qkv fwd", M, 3072, 1024, 0, 0, 0, "bias"),
    ("proj fwd", M, 1024, 1024, 0, 0, 0, "bias_res"),
    ("fc1 fwd", M, 4096, 1024, 0, 0, 0, "gelu_aux"),
    ("fc2 fwd", M, 1024, 4096, 0, 0, 0, "bias_res"),
    ("fc2 dgrad", M, 4096, 1024, 0, 1, 0, "gelu_grad"),
    ("fc1 dgrad", M, 1024, 4096, 0, 1, 0, "acc"),
    ("fc1 wgrad", 4096, 1024, M, 1, 1, 1, ""),
    ("proj wgrad", 1024, 1024, M, 1, 1, 1, ""),
    ("big", 8192, 8192, 8192, 0, 0, 0, ""),
    ("fc1 plain", M, 4096, 1024, 0, 0, 0, ""),
    ("fc1 bias", M, 4096, 1024, 0, 0, 0, "bias"),
    ("fc1 gelu", M, 4096, 1024, 0, 0, 0, "gelu"),
    ("fc1 b32", 16384, 4096, 1024, 0, 0, 0, "gelu_aux"),
    ("fc2dg b32", 16384, 4096, 1024, 0, 1, 0, "gelu_grad"),
    ("fc2dg plain", 16384, 4096, 1024, 0, 1, 0, ""),
    ("fc2dg resadd", 16384, 4096, 1024, 0, 1, 0, "res"),
    ("fc2dg gg-ldg", 16384, 4096, 1024, 0, 1, 0, "gelu_grad_direct"),
    ("fc1 b32 ldg", 16384, 4096, 1024, 0, 0, 0, "gelu_aux_direct"),
    ("qkv b48", 24576, 3072, 1024, 0, 0, 0, "bias"),
    ("proj b48", 24576, 1024, 1024, 0, 0, 0, "bias_res"),
    ("fc2 b48", 24576, 1024, 4096, 0, 0, 0, "bias_res"),
    ("fc1dg b48", 24576, 1024, 4096, 0, 1, 0, "acc"),
    ("big plain", 8192, 8192, 8192, 0, 1, 0, ""),
]
for name, m, n, kk, amn, bmn, f32, epi in cases:
    A = torch.randn(kk, m, device="cuda").to(bf) if amn else torch.randn(m, kk, device="cuda").to(bf)
    B = torch.randn(kk, n, device="cuda").to(bf) if bmn else torch.randn(n, kk, device="cuda").to(bf)
    C = torch.empty(m, n, device="cuda", dtype=torch.float32 if f32 else bf)
    kw = {}
    if "bias" in epi or epi.startswith("gelu_aux"):
        kw["bias"] = torch.randn(n, device="cuda").to(bf)
    if epi.endswith("_direct"):
        kw["epilogue"] = 1
        epi = epi[:-len("_direct")]
    if epi in ("bias_res", "acc", "res"):
        kw["residual"] = torch.randn(m, n, device="cuda").to(bf)
    if epi == "gelu_aux":
        kw.update(gelu=True, aux=torch.empty(m, n, device="cuda", dtype=bf))
    if epi == "gelu":
        kw.update(gelu=True)
    if epi == "gelu_grad":
        kw.update(residual=torch.randn(m, n, device="cuda").to(bf), residual_mode=1)
    call = lambda: k.gemm_raw(M=m, N=n, K=kk, A=A, lda=A.stride(0), a_mn=bool(amn), B=B, ldb=B.stride(0),
                              b_mn=bool(bmn), Cout=C, ldc=n, **kw)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    tr.zero_()
    lib.dpn_gemm_debug_trace(tr.data_ptr())
    call()
    torch.cuda.synchronize()
    lib.dpn_gemm_debug_trace(None)
    t = tr.view(148, 8).float()
    act = t[:, 4] > 0
    a = t[act].mean(0) / 1000
    lead = t[act & (t[:, 1] > 0)].mean(0) / 1000
    tf = 2 * m * n * kk / (us * 1e-6) / 1e12
    print(f"{name:11s} {us:7.1f} us {tf:6.0f} TF | kcyc: run {a[4]:6.1f} prod-wait-empty {a[0]:6.1f} "
          f"mma-wait-full {lead[1]:6.1f} mma-wait-acc {lead[2]:6.1f} epi-wait {a[3]:6.1f} epi-busy {a[6]:6.1f} "
          f"pdl {a[5]:5.1f} ctas {int(act.sum())}", flush=True)
