"""Thin Python entry points over the C ABI, taking torch CUDA tensors.

torch is used only as the owner of device memory and streams; every op here is
one call into `_dawnpiper.so` (no torch compute).  Shapes/strides are checked
on the host side before the call; the C side re-checks what it relies on.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from ._lib import GemmArgs, check, lib

BF16 = torch.bfloat16
F32 = torch.float32


class _Instrument:
    """Launch accounting for bench.py: counts every kernel launched through
    the C ABI and, when `gemm_events` is a list, brackets each GEMM with CUDA
    events on its own stream (flops, start, end)."""

    def __init__(self):
        self.launches = 0
        self.gemm_events = None
        self.gemm_flops = 0  # algorithmic 2*M*N*K*batch of every GEMM issued


INSTR = _Instrument()


_WS = {}


def _dev_index(device) -> int:
    d = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    return d.index if d.index is not None else torch.cuda.current_device()


def _workspace(device, floats: int, stream) -> torch.Tensor:
    """Per-(device, stream) f32 scratch for two-phase reductions / attention.
    Kernels on one stream use it in stream order; streams never share one.
    The buffer is allocated in that stream's order (None = the current stream,
    a raw handle is wrapped), so the caching allocator never hands its memory
    to another stream while kernels on this one may still use it."""
    ts = _torch_stream(stream)
    if ts is None:
        ts = torch.cuda.ExternalStream(int(stream), device=torch.device("cuda", _dev_index(device)))
    key = (_dev_index(device), ts.cuda_stream)
    t = _WS.get(key)
    if t is None or t.numel() < floats:
        with torch.cuda.stream(ts):
            t = torch.empty(max(floats, 1 << 20), dtype=F32, device=torch.device("cuda", key[0]))
        _WS[key] = t
    return t


def release_workspaces(device=None) -> None:
    """Drop the cached scratch buffers (all devices, or one). Callers that create
    short-lived streams (per-trial executors) call this when they are done: the
    cache is keyed by stream handle, so it would otherwise keep one buffer per
    stream the pool ever handed out."""
    want = None if device is None else _dev_index(device)
    for key in [k for k in _WS if want is None or k[0] == want]:
        del _WS[key]


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def _torch_stream(stream):
    if stream is None:
        return torch.cuda.current_stream()
    return stream if isinstance(stream, torch.cuda.Stream) else None


def _p(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _s(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def gemm_raw(*, M, N, K, A, lda, B, ldb, Cout, ldc, a_mn=False, b_mn=False, batch1=1, batch2=1,
             a_s=(0, 0), b_s=(0, 0), c_s=(0, 0), bias=None, residual=None, ldr=None, r_s=None,
             aux=None, alpha=1.0, gelu=False, accumulate=False, block_n=0, split_k=0,
             cta_group=0, residual_mode=0, epilogue=0, colsum=None, stream=None) -> None:
    """C[z] = epi(alpha * A[z] B[z]^T); see include/dawnpiper.h for the layout rules.
    colsum: optional f32 [N]: += the column sums of the stored bf16 C (fused bias gradient)."""
    assert colsum is None or colsum.dtype == F32
    rs = (r_s if r_s is not None else c_s) if residual is not None else (0, 0)
    g = GemmArgs(M, N, K, batch1, batch2,
                 A.data_ptr(), lda, a_s[0], a_s[1], a_mn,
                 B.data_ptr(), ldb, b_s[0], b_s[1], b_mn,
                 Cout.data_ptr(), ldc, c_s[0], c_s[1], 0 if Cout.dtype == F32 else 1, accumulate,
                 None if bias is None else bias.data_ptr(),
                 None if residual is None else residual.data_ptr(),
                 (ldr if ldr is not None else ldc) if residual is not None else 0, rs[0], rs[1],
                 residual_mode, None if aux is None else aux.data_ptr(), alpha, gelu, block_n,
                 split_k, cta_group, epilogue, None if colsum is None else colsum.data_ptr())
    INSTR.launches += 1
    INSTR.gemm_flops += 2 * int(M) * int(N) * int(K) * int(batch1) * int(batch2)
    ev = INSTR.gemm_events
    if ev is not None:
        ts = _torch_stream(stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ts)
        check(lib().dpn_gemm(C.byref(g), _s(stream)), "dpn_gemm")
        e1.record(ts)
        ev.append((2 * int(M) * int(N) * int(K) * int(batch1) * int(batch2), e0, e1,
                   (int(M), int(N), int(K), int(batch1) * int(batch2), int(a_mn), int(b_mn), Cout.dtype == F32)))
    else:
        check(lib().dpn_gemm(C.byref(g), _s(stream)), "dpn_gemm")


# ---- dense-layer shapes -----------------------------------------------------------


def linear_fwd(x, w, out, bias=None, residual=None, gelu=False, aux=None, stream=None):
    """out[M, N] = x[M, K] @ w[N, K]^T (+ bias) (+ residual), optional GELU."""
    M, K = x.shape
    N = w.shape[0]
    gemm_raw(M=M, N=N, K=K, A=x, lda=x.stride(0), B=w, ldb=w.stride(0), Cout=out,
             ldc=out.stride(0), bias=bias, residual=residual,
             ldr=None if residual is None else residual.stride(0), aux=aux, gelu=gelu,
             stream=stream)


def linear_dgrad(dy, w, dx, accumulate_into=None, gelu_of=None, dbias=None, stream=None):
    """dx[M, K] = dy[M, N] @ w[N, K]  (w used MN-major: no transpose copy).
    accumulate_into: a bf16 [M, K] tensor added to the result (may be dx);
    gelu_of: pre-activation f [M, K]: dx *= gelu'(f) (fused GELU backward);
    dbias: f32 [K]: += column sums of the stored dx (the bias gradient of the
    linear that produced f, fused into this epilogue)."""
    M, N = dy.shape
    K = w.shape[1]
    assert accumulate_into is None or gelu_of is None
    res = accumulate_into if gelu_of is None else gelu_of
    gemm_raw(M=M, N=K, K=N, A=dy, lda=dy.stride(0), B=w, ldb=w.stride(0), b_mn=True, Cout=dx,
             ldc=dx.stride(0), residual=res, ldr=None if res is None else res.stride(0),
             residual_mode=0 if gelu_of is None else 1, colsum=dbias, stream=stream)


def linear_wgrad(dy, x, dw, accumulate=False, stream=None):
    """dw[N, K] (f32) = dy[M, N]^T @ x[M, K]  (both operands MN-major)."""
    M, N = dy.shape
    K = x.shape[1]
    gemm_raw(M=N, N=K, K=M, A=dy, lda=dy.stride(0), a_mn=True, B=x, ldb=x.stride(0), b_mn=True,
             Cout=dw, ldc=dw.stride(0), accumulate=accumulate, stream=stream)


# ---- node kernels -----------------------------------------------------------------


def attn_fwd(qkv, out, lse, batch, seq, heads, causal, scale=None, stream=None):
    """Fused attention forward from the [b*s, 3H] QKV buffer (head_dim 64)."""
    d = 64
    INSTR.launches += 1
    check(lib().dpn_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), batch, seq, heads, d,
                             scale if scale is not None else d ** -0.5, int(causal), _s(stream)),
          "dpn_attn_fwd")


def attn_bwd(qkv, out, dout, lse, dqkv, batch, seq, heads, causal, scale=None, dbias=None,
             stream=None):
    """Fused attention backward -> dqkv [b*s, 3H] (dQ | dK | dV).
    dbias: f32 [3H]: += column sums of dqkv (the QKV projection's bias gradient)."""
    assert dbias is None or (dbias.dtype == torch.float32 and dbias.data_ptr() % 16 == 0)
    d = 64
    H = heads * d
    INSTR.launches += 3
    ws = _workspace(qkv.device, batch * seq * H + batch * heads * seq, stream)
    check(lib().dpn_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                             dqkv.data_ptr(), ws.data_ptr(), ws.numel(), batch, seq, heads, d,
                             scale if scale is not None else d ** -0.5, int(causal),
                             None if dbias is None else dbias.data_ptr(), _s(stream)),
          "dpn_attn_bwd")


def attn_fwd_cross(q, kv, out, lse, batch, q_seq, kv_seq, heads, scale=None, stream=None):
    """Fused cross-attention forward: q [b*t, H], kv [b*s, 2H] (K | V) -> out, lse [b, A, t]."""
    d = 64
    INSTR.launches += 1
    check(lib().dpn_attn_fwd_cross(q.data_ptr(), kv.data_ptr(), out.data_ptr(), lse.data_ptr(), batch,
                                   q_seq, kv_seq, heads, d, scale if scale is not None else d ** -0.5,
                                   _s(stream)), "dpn_attn_fwd_cross")


def attn_bwd_cross(q, kv, out, dout, lse, dq, dkv, batch, q_seq, kv_seq, heads, scale=None,
                   stream=None):
    """Fused cross-attention backward -> dq [b*t, H], dkv [b*s, 2H]."""
    d = 64
    H = heads * d
    INSTR.launches += 3
    ws = _workspace(q.device, batch * q_seq * H + batch * heads * q_seq, stream)
    check(lib().dpn_attn_bwd_cross(q.data_ptr(), kv.data_ptr(), out.data_ptr(), dout.data_ptr(),
                                   lse.data_ptr(), dq.data_ptr(), dkv.data_ptr(), ws.data_ptr(),
                                   ws.numel(), batch, q_seq, kv_seq, heads, d,
                                   scale if scale is not None else d ** -0.5, _s(stream)),
          "dpn_attn_bwd_cross")


def layernorm_fwd(x, gamma, beta, y, mean, rstd, eps=1e-5, stream=None):
    rows, cols = x.shape
    INSTR.launches += 1
    check(lib().dpn_layernorm_fwd(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(),
                                  mean.data_ptr(), rstd.data_ptr(), rows, cols, eps, _s(stream)),
          "dpn_layernorm_fwd")


def layernorm_bwd(dy, x, gamma, mean, rstd, dx, dgamma, dbeta, dx_add=None, stream=None):
    rows, cols = x.shape
    INSTR.launches += 2
    check(lib().dpn_layernorm_bwd(dy.data_ptr(), x.data_ptr(), gamma.data_ptr(), mean.data_ptr(),
                                  rstd.data_ptr(), dx.data_ptr(), _p(dx_add), dgamma.data_ptr(),
                                  dbeta.data_ptr(), rows, cols, None, 0, _s(stream)),
          "dpn_layernorm_bwd")


def layernorm_bwd_fused(dy, x, gamma, mean, rstd, dx, dgamma, dbeta, dx_add=None, dbias=None,
                        stream=None):
    """One-pass LayerNorm backward (dx, dgamma, dbeta and optionally the next
    linear's bias gradient = column sums of the final dx)."""
    rows, cols = x.shape
    INSTR.launches += 1
    check(lib().dpn_layernorm_bwd_fused(dy.data_ptr(), x.data_ptr(), gamma.data_ptr(),
                                        mean.data_ptr(), rstd.data_ptr(), dx.data_ptr(), _p(dx_add),
                                        dgamma.data_ptr(), dbeta.data_ptr(), _p(dbias), rows, cols,
                                        _s(stream)), "dpn_layernorm_bwd_fused")


def softmax_fwd(s, p, q_len, alpha, causal, stream=None):
    cols = s.shape[-1]
    rows = s.numel() // cols
    INSTR.launches += 1
    check(lib().dpn_softmax_fwd(s.data_ptr(), p.data_ptr(), rows, cols, q_len, alpha, int(causal),
                                _s(stream)), "dpn_softmax_fwd")


def softmax_bwd(p, dp, ds, alpha, stream=None):
    cols = p.shape[-1]
    rows = p.numel() // cols
    INSTR.launches += 1
    check(lib().dpn_softmax_bwd(p.data_ptr(), dp.data_ptr(), ds.data_ptr(), rows, cols, alpha,
                                _s(stream)), "dpn_softmax_bwd")


def gelu_fwd(x, y, stream=None):
    INSTR.launches += 1
    check(lib().dpn_gelu_fwd(x.data_ptr(), y.data_ptr(), x.numel(), _s(stream)), "dpn_gelu_fwd")


def gelu_bwd(dy, x, dx, stream=None):
    INSTR.launches += 1
    check(lib().dpn_gelu_bwd(dy.data_ptr(), x.data_ptr(), dx.data_ptr(), x.numel(), _s(stream)),
          "dpn_gelu_bwd")


def add(a, b, out, stream=None):
    INSTR.launches += 1
    check(lib().dpn_add(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.numel(), _s(stream)), "dpn_add")


def cast_f32_bf16(x, y, stream=None):
    INSTR.launches += 1
    check(lib().dpn_cast_f32_bf16(x.data_ptr(), y.data_ptr(), x.numel(), _s(stream)),
          "dpn_cast_f32_bf16")


def colsum(x, out, stream=None):
    rows, cols = x.shape
    INSTR.launches += 1
    check(lib().dpn_colsum(x.data_ptr(), rows, cols, x.stride(0), out.data_ptr(), None, 0,
                           _s(stream)), "dpn_colsum")


def xent(logits, labels, vocab, grad_scale, loss_sum, dlogits, loss_scale=1.0, stream=None):
    rows, ld = logits.shape
    INSTR.launches += 1
    check(lib().dpn_xent(logits.data_ptr(), ld, labels.data_ptr(), rows, vocab, grad_scale,
                         loss_scale, loss_sum.data_ptr(), dlogits.data_ptr(), _s(stream)), "dpn_xent")


def embed_fwd(ids, tok, pos, out, seq, stream=None):
    rows = ids.numel()
    INSTR.launches += 1
    check(lib().dpn_embed_fwd(ids.data_ptr(), tok.data_ptr(), pos.data_ptr(), out.data_ptr(), rows,
                              seq, tok.shape[1], _s(stream)), "dpn_embed_fwd")


def embed_bwd(ids, dout, dtok, dpos, seq, stream=None):
    rows = ids.numel()
    INSTR.launches += 1
    check(lib().dpn_embed_bwd(ids.data_ptr(), dout.data_ptr(), dtok.data_ptr(), dpos.data_ptr(),
                              rows, seq, dout.shape[1], _s(stream)), "dpn_embed_bwd")


def adamw(w, m, v, g, out_bf16, lr, beta1, beta2, eps, wd, step, stream=None):
    INSTR.launches += 1
    check(lib().dpn_adamw(w.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(),
                          out_bf16.data_ptr(), w.numel(), lr, beta1, beta2, eps, wd, step,
                          _s(stream)), "dpn_adamw")


def adamw_dstep(w, m, v, g, out_bf16, lr, beta1, beta2, eps, wd, step_dev, stream=None):
    """AdamW with a device-resident step counter (CUDA-graph replayable)."""
    INSTR.launches += 2
    check(lib().dpn_adamw_dstep(w.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(),
                                out_bf16.data_ptr(), w.numel(), lr, beta1, beta2, eps, wd,
                                step_dev.data_ptr(), _s(stream)), "dpn_adamw_dstep")


def memset(t, value=0, nbytes=None, stream=None):
    n = nbytes if nbytes is not None else t.numel() * t.element_size()
    check(lib().dpn_memset_async(t.data_ptr(), value, n, _s(stream)), "dpn_memset_async")


def swap_out(host_dst, dev_src, copy_stream, ready_event=None):
    """Swap engine D2H (memopt `swap`): host_dst (pinned) <- dev_src on
    copy_stream after ready_event (recorded on the compute stream)."""
    n = dev_src.numel() * dev_src.element_size()
    check(lib().dpn_swap_out(host_dst.data_ptr(), dev_src.data_ptr(), n, _s(copy_stream),
                             ready_event.cuda_event if ready_event is not None else None, None),
          "dpn_swap_out")
    return n


def swap_in(dev_dst, host_src, copy_stream, ready_event=None):
    """Swap engine H2D prefetch: dev_dst <- host_src (pinned) on copy_stream
    after ready_event."""
    n = dev_dst.numel() * dev_dst.element_size()
    check(lib().dpn_swap_in(dev_dst.data_ptr(), host_src.data_ptr(), n, _s(copy_stream),
                            ready_event.cuda_event if ready_event is not None else None, None),
          "dpn_swap_in")
    return n


def copy_d2d(dst, src, nbytes=None, dst_dev=0, src_dev=0, stream=None):
    n = nbytes if nbytes is not None else src.numel() * src.element_size()
    check(lib().dpn_p2p_copy(dst.data_ptr(), dst_dev, src.data_ptr(), src_dev, n, _s(stream)),
          "dpn_p2p_copy")


# ---- CNN nodes (AmoebaNet-D) --------------------------------------------------------


def relu_fwd(x, y, stream=None):
    INSTR.launches += 1
    check(lib().dpn_relu_fwd(x.data_ptr(), y.data_ptr(), x.numel(), _s(stream)), "dpn_relu_fwd")


def relu_bwd(dy, y, dx, stream=None):
    INSTR.launches += 1
    check(lib().dpn_relu_bwd(dy.data_ptr(), y.data_ptr(), dx.data_ptr(), dy.numel(), _s(stream)),
          "dpn_relu_bwd")


def dwconv3_fwd(x, w, y, b, H, W, C, stride, stream=None):
    INSTR.launches += 1
    check(lib().dpn_dwconv3_fwd(x.data_ptr(), w.data_ptr(), y.data_ptr(), b, H, W, C, stride,
                                _s(stream)), "dpn_dwconv3_fwd")


def dwconv3_bwd(x, w, dy, dx, dw, b, H, W, C, stride, stream=None):
    INSTR.launches += (dx is not None) + (dw is not None)
    check(lib().dpn_dwconv3_bwd(x.data_ptr(), w.data_ptr(), dy.data_ptr(), _p(dx), _p(dw), b, H, W, C,
                                stride, _s(stream)), "dpn_dwconv3_bwd")


def bn_fwd(x, gamma, beta, y, stats, eps=1e-5, stream=None):
    P, C_ = x.shape
    INSTR.launches += 2
    check(lib().dpn_bn_fwd(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(),
                           stats.data_ptr(), P, C_, eps, _s(stream)), "dpn_bn_fwd")


def bn_bwd(dy, x, stats, gamma, dx, dgamma, dbeta, workspace, eps=1e-5, stream=None):
    P, C_ = x.shape
    INSTR.launches += 2
    check(lib().dpn_bn_bwd(dy.data_ptr(), x.data_ptr(), stats.data_ptr(), gamma.data_ptr(),
                           dx.data_ptr(), dgamma.data_ptr(), dbeta.data_ptr(), workspace.data_ptr(),
                           P, C_, eps, _s(stream)), "dpn_bn_bwd")


def pool3_fwd(x, y, argmax, b, H, W, C, stride, mode, stream=None):
    INSTR.launches += 1
    check(lib().dpn_pool3_fwd(x.data_ptr(), y.data_ptr(), _p(argmax), b, H, W, C, stride, mode,
                              _s(stream)), "dpn_pool3_fwd")


def pool3_bwd(dy, argmax, dx, b, H, W, C, stride, mode, stream=None):
    INSTR.launches += 1
    check(lib().dpn_pool3_bwd(dy.data_ptr(), _p(argmax), dx.data_ptr(), b, H, W, C, stride, mode,
                              _s(stream)), "dpn_pool3_bwd")


def copy_cols(src, lds, dst, ldd, rows, cols, accumulate=False, stream=None):
    INSTR.launches += 1
    check(lib().dpn_copy_cols(src.data_ptr(), lds, dst.data_ptr(), ldd, rows, cols, int(accumulate),
                              _s(stream)), "dpn_copy_cols")


def im2col3(x, cols, b, H, W, C, stride, stream=None):
    INSTR.launches += 1
    check(lib().dpn_im2col3(x.data_ptr(), cols.data_ptr(), b, H, W, C, stride, _s(stream)),
          "dpn_im2col3")


def gap_fwd(x, y, b, HW, C, stream=None):
    INSTR.launches += 1
    check(lib().dpn_gap_fwd(x.data_ptr(), y.data_ptr(), b, HW, C, _s(stream)), "dpn_gap_fwd")


def gap_bwd(dy, dx, b, HW, C, stream=None):
    INSTR.launches += 1
    check(lib().dpn_gap_bwd(dy.data_ptr(), dx.data_ptr(), b, HW, C, _s(stream)), "dpn_gap_bwd")
