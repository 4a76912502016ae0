"""Numerics of every CUDA kernel against a plain PyTorch fp32 reference.

Tolerances: bf16 outputs are compared at rel 2e-2 of the output scale (the
north-star bf16 tolerance); fp32 outputs of bf16 GEMMs at 5e-3 relative.
"""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def dev():
    from paper_2505_05856_b200 import _lib
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    _lib.init_device(torch.cuda.current_device())
    torch.manual_seed(0)
    yield


def K():
    from paper_2505_05856_b200 import kernels
    return kernels


def close(got, want, rel=2e-2):
    got = got.float()
    want = want.float()
    scale = want.abs().max().item() + 1e-6
    err = (got - want).abs().max().item()
    assert err <= rel * scale, f"max err {err:.4g} vs scale {scale:.4g}"


def rnd(*shape, dtype=torch.bfloat16, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(dtype)


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("M,N,K_,bn,cg", [(256, 256, 128, 0, 0), (300, 200, 96, 0, 0), (128, 64, 64, 64, 1),
                                           (512, 768, 1024, 256, 1), (384, 1024, 512, 128, 1),
                                           (77, 136, 40, 0, 0), (512, 768, 1024, 256, 2),
                                           (384, 1024, 512, 128, 2), (700, 520, 200, 256, 2),
                                           (200, 384, 64, 128, 2), (512, 1024, 512, 256, 4),
                                           (700, 520, 200, 256, 4), (1024, 768, 1024, 256, 4)])
@pytest.mark.parametrize("epi", [0, 1])
def test_gemm_layouts(a_mn, b_mn, M, N, K_, bn, cg, epi):
    k = K()
    A = rnd(M, K_)
    B = rnd(N, K_)
    As = A.t().contiguous() if a_mn else A
    Bs = B.t().contiguous() if b_mn else B
    lda = As.stride(0)
    ldb = Bs.stride(0)
    if (a_mn and M % 8) or (b_mn and N % 8) or (not a_mn and K_ % 8) or (not b_mn and K_ % 8):
        pytest.skip("TMA needs 16-byte strides")
    C = torch.empty(M, (N + 7) // 8 * 8, device="cuda", dtype=torch.float32)
    k.gemm_raw(M=M, N=N, K=K_, A=As, lda=lda, a_mn=a_mn, B=Bs, ldb=ldb, b_mn=b_mn, Cout=C,
               ldc=C.stride(0), block_n=bn, cta_group=cg, epilogue=epi)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    close(C[:, :N], ref, rel=5e-3)


@pytest.mark.parametrize("mode", ["plain", "bias", "bias_res", "gelu_aux", "gelu_grad"])
@pytest.mark.parametrize("M,N,K_,bn,cg", [(512, 384, 256, 0, 0), (300, 200, 96, 0, 0),
                                           (77, 136, 40, 0, 0), (1024, 1024, 1024, 256, 2),
                                           (384, 512, 128, 128, 1), (640, 320, 192, 128, 2),
                                           (1024, 1024, 1024, 256, 4), (640, 320, 192, 256, 4)])
@pytest.mark.parametrize("epi", [0, 1])
def test_gemm_bf16_epilogues(mode, M, N, K_, bn, cg, epi):
    """bf16 outputs through the TMA-staged epilogue (epi 0) and the direct-store
    one (epi 1), with tails in M and N, every epilogue combination the executor uses."""
    k = K()
    A, B = rnd(M, K_), rnd(N, K_, scale=0.05)
    ldc = (N + 7) // 8 * 8
    bias, res = rnd(N), rnd(M, ldc)
    out = torch.zeros(M, ldc, device="cuda", dtype=torch.bfloat16)
    aux = torch.zeros_like(out)
    kw = {}
    pre = A.float() @ B.float().t()
    if mode in ("bias", "bias_res", "gelu_aux"):
        kw["bias"] = bias
        pre = pre + bias.float()
    if mode == "bias_res":
        kw["residual"] = res
        pre = pre + res[:, :N].float()
    if mode == "gelu_aux":
        kw.update(gelu=True, aux=aux)
    if mode == "gelu_grad":
        kw.update(residual=res, residual_mode=1)
    k.gemm_raw(M=M, N=N, K=K_, A=A, lda=K_, B=B, ldb=K_, Cout=out, ldc=ldc, block_n=bn, cta_group=cg,
               epilogue=epi, **kw)
    torch.cuda.synchronize()
    if mode == "gelu_aux":
        close(aux[:, :N], pre)
        close(out[:, :N], torch.nn.functional.gelu(pre, approximate="tanh"))
    elif mode == "gelu_grad":
        fr = res[:, :N].float().requires_grad_()
        torch.nn.functional.gelu(fr, approximate="tanh").backward(pre)
        close(out[:, :N], fr.grad)
    else:
        close(out[:, :N], pre)
    if ldc > N:  # pad columns untouched
        assert torch.all(out[:, N:] == 0)


def test_gemm_epilogue_bias_residual_gelu_aux():
    k = K()
    M, N, K_ = 512, 384, 256
    A, B = rnd(M, K_), rnd(N, K_, scale=0.05)
    bias, res = rnd(N), rnd(M, N)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    aux = torch.empty_like(out)
    k.gemm_raw(M=M, N=N, K=K_, A=A, lda=K_, B=B, ldb=K_, Cout=out, ldc=N, bias=bias, residual=res,
               aux=aux, gelu=True, alpha=0.5)
    torch.cuda.synchronize()
    pre = 0.5 * (A.float() @ B.float().t()) + bias.float() + res.float()
    close(aux, pre)
    close(out, torch.nn.functional.gelu(pre, approximate="tanh"))


def test_gemm_f32_accumulate():
    k = K()
    M, N, K_ = 256, 512, 384
    A, B = rnd(M, K_), rnd(N, K_)
    C = torch.randn(M, N, device="cuda")
    C0 = C.clone()
    k.gemm_raw(M=M, N=N, K=K_, A=A, lda=K_, B=B, ldb=K_, Cout=C, ldc=N, accumulate=True)
    torch.cuda.synchronize()
    close(C, C0 + A.float() @ B.float().t(), rel=5e-3)


def test_gemm_batched_attention_layout():
    """QK^T and PV straight out of a fused [b*s, 3H] qkv buffer, per (batch, head)."""
    k = K()
    b, s, A_, d = 2, 256, 4, 64
    H = A_ * d
    qkv = rnd(b * s, 3 * H)
    q = qkv[:, :H].reshape(b, s, A_, d).permute(0, 2, 1, 3).float()
    kk = qkv[:, H:2 * H].reshape(b, s, A_, d).permute(0, 2, 1, 3).float()
    v = qkv[:, 2 * H:].reshape(b, s, A_, d).permute(0, 2, 1, 3).float()
    S = torch.empty(b, A_, s, s, device="cuda", dtype=torch.bfloat16)
    k.gemm_raw(M=s, N=s, K=d, A=qkv, lda=3 * H, a_s=(d, s * 3 * H), B=qkv[:, H:], ldb=3 * H,
               b_s=(d, s * 3 * H), batch1=A_, batch2=b, Cout=S, ldc=s, c_s=(s * s, A_ * s * s))
    torch.cuda.synchronize()
    close(S, q @ kk.transpose(-1, -2))
    P = torch.softmax(S.float(), -1).to(torch.bfloat16)
    O = torch.empty(b * s, H, device="cuda", dtype=torch.bfloat16)
    # PV: A = P (K-major over keys), B = V MN-major (d contiguous)
    k.gemm_raw(M=s, N=d, K=s, A=P, lda=s, a_s=(s * s, A_ * s * s), B=qkv[:, 2 * H:], ldb=3 * H,
               b_mn=True, b_s=(d, s * 3 * H), batch1=A_, batch2=b, Cout=O, ldc=H,
               c_s=(d, s * H))
    torch.cuda.synchronize()
    ref = (P.float() @ v).permute(0, 2, 1, 3).reshape(b * s, H)
    close(O, ref)


def test_linear_helpers():
    k = K()
    M, N, K_ = 384, 512, 256
    x, w, b = rnd(M, K_), rnd(N, K_, scale=0.05), rnd(N)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    k.linear_fwd(x, w, y, bias=b)
    dy = rnd(M, N)
    dx = torch.empty(M, K_, device="cuda", dtype=torch.bfloat16)
    k.linear_dgrad(dy, w, dx)
    dw = torch.empty(N, K_, device="cuda")
    k.linear_wgrad(dy, x, dw)
    torch.cuda.synchronize()
    close(y, x.float() @ w.float().t() + b.float())
    close(dx, dy.float() @ w.float())
    close(dw, dy.float().t() @ x.float(), rel=5e-3)


@pytest.mark.parametrize("cols", [768, 1024, 1600])
def test_layernorm(cols):
    k = K()
    rows = 333
    x = rnd(rows, cols, scale=2.0)
    g, b = rnd(cols), rnd(cols)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    k.layernorm_fwd(x, g, b, y, mean, rstd)
    xr = x.float().requires_grad_()
    gr = g.float().requires_grad_()
    br = b.float().requires_grad_()
    yr = torch.nn.functional.layer_norm(xr, (cols,), gr, br, 1e-5)
    torch.cuda.synchronize()
    close(y, yr)
    dy = rnd(rows, cols)
    add = rnd(rows, cols)
    yr.backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.zeros(cols, device="cuda")
    db = torch.zeros(cols, device="cuda")
    k.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, db, dx_add=add)
    torch.cuda.synchronize()
    close(dx, xr.grad + add.float())
    close(dg, gr.grad, rel=5e-3)
    close(db, br.grad, rel=5e-3)


@pytest.mark.parametrize("rows,cols", [(333, 128), (16384, 1024), (1000, 768), (2048, 1600),
                                       (7, 1024), (8192, 2048)])
@pytest.mark.parametrize("add", [False, True])
def test_layernorm_bwd_fused(rows, cols, add):
    """One-pass LayerNorm backward (dx, dgamma, dbeta, + the bias gradient of
    the linear producing the LN input = column sums of the final dx) against
    the fp32 torch reference."""
    k = K()
    x = rnd(rows, cols, scale=2.0)
    g, b = rnd(cols), rnd(cols)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    k.layernorm_fwd(x, g, b, y, mean, rstd)
    xr = x.float().requires_grad_()
    gr = g.float().requires_grad_()
    br = b.float().requires_grad_()
    yr = torch.nn.functional.layer_norm(xr, (cols,), gr, br, 1e-5)
    dy = rnd(rows, cols)
    yr.backward(dy.float())
    dxa = rnd(rows, cols) if add else None
    dx = dxa.clone() if add else torch.empty_like(x)   # in place over dx_add, as the executor does
    dg = torch.full((cols,), 0.5, device="cuda")       # accumulates into what is there
    db = torch.zeros(cols, device="cuda")
    dbias = torch.full((cols,), -1.0, device="cuda")
    k.layernorm_bwd_fused(dy, x, g, mean, rstd, dx, dg, db, dx_add=dx if add else None, dbias=dbias)
    torch.cuda.synchronize()
    want_dx = xr.grad + (dxa.float() if add else 0)
    close(dx, want_dx)
    close(dg, gr.grad + 0.5, rel=5e-3)
    close(db, br.grad, rel=5e-3)
    close(dbias, dx.float().sum(0) - 1.0, rel=5e-3)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("cols", [128, 512, 1024])
def test_softmax(causal, cols):
    k = K()
    z, q = 3, cols
    s = rnd(z, q, cols, scale=3.0)
    p = torch.empty_like(s)
    alpha = 1 / math.sqrt(64)
    k.softmax_fwd(s, p, q, alpha, causal)
    sr = (s.float() * alpha)
    if causal:
        mask = torch.ones(q, cols, device="cuda").triu(1).bool()
        sr = sr.masked_fill(mask, float("-inf"))
    pr = torch.softmax(sr, -1)
    torch.cuda.synchronize()
    close(p, pr)
    dp = rnd(z, q, cols)
    ds = torch.empty_like(s)
    k.softmax_bwd(p, dp, ds, alpha)
    pf = p.float()
    ref = alpha * pf * (dp.float() - (dp.float() * pf).sum(-1, keepdim=True))
    torch.cuda.synchronize()
    close(ds, ref)


def test_gelu_add_cast_colsum():
    k = K()
    x = rnd(1000, 64)
    y = torch.empty_like(x)
    k.gelu_fwd(x, y)
    dy = rnd(1000, 64)
    dx = torch.empty_like(x)
    k.gelu_bwd(dy, x, dx)
    xr = x.float().requires_grad_()
    yr = torch.nn.functional.gelu(xr, approximate="tanh")
    yr.backward(dy.float())
    o = torch.empty_like(x)
    k.add(x, dy, o)
    f = torch.randn(4096, device="cuda")
    fb = torch.empty(4096, device="cuda", dtype=torch.bfloat16)
    k.cast_f32_bf16(f, fb)
    cs = torch.zeros(64, device="cuda")
    k.colsum(dy, cs)
    torch.cuda.synchronize()
    close(y, yr)
    close(dx, xr.grad)
    close(o, x.float() + dy.float())
    assert torch.equal(fb, f.to(torch.bfloat16))
    close(cs, dy.float().sum(0), rel=5e-3)


@pytest.mark.parametrize("vocab,ld", [(1000, 1000), (30520, 30528), (30522, 30528), (50257, 50304)])
def test_xent(vocab, ld):
    k = K()
    rows = 257
    logits = rnd(rows, ld, scale=2.0)
    labels = torch.randint(0, vocab, (rows,), device="cuda", dtype=torch.int32)
    loss = torch.zeros(1, device="cuda")
    dl = torch.empty_like(logits)
    k.xent(logits, labels, vocab, 1.0 / rows, loss, dl)
    lr = logits[:, :vocab].float().requires_grad_()
    ref = torch.nn.functional.cross_entropy(lr, labels.long(), reduction="sum")
    (ref / rows).backward()
    torch.cuda.synchronize()
    assert abs(loss.item() - ref.item()) <= 1e-3 * abs(ref.item())
    close(dl[:, :vocab], lr.grad)
    assert dl[:, vocab:].abs().sum().item() == 0


def test_embed():
    k = K()
    V, H, S, B = 500, 256, 64, 3
    tok, pos = rnd(V, H), rnd(S, H)
    ids = torch.randint(0, V, (B * S,), device="cuda", dtype=torch.int32)
    out = torch.empty(B * S, H, device="cuda", dtype=torch.bfloat16)
    k.embed_fwd(ids, tok, pos, out, S)
    ref = tok.float()[ids.long()] + pos.float().repeat(B, 1)
    dout = rnd(B * S, H)
    dt = torch.zeros(V, H, device="cuda")
    dp = torch.zeros(S, H, device="cuda")
    k.embed_bwd(ids, dout, dt, dp, S)
    rt = torch.zeros(V, H, device="cuda").index_add_(0, ids.long(), dout.float())
    rp = dout.float().reshape(B, S, H).sum(0)
    torch.cuda.synchronize()
    close(out, ref)
    close(dt, rt, rel=1e-4)
    close(dp, rp, rel=1e-4)


def test_adamw():
    k = K()
    n = 4096
    w = torch.randn(n, device="cuda")
    g = torch.randn(n, device="cuda")
    m, v = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    out = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    wr = w.clone().requires_grad_()
    opt = torch.optim.AdamW([wr], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)
    for step in (1, 2, 3):
        k.adamw(w, m, v, g, out, 1e-3, 0.9, 0.999, 1e-8, 0.01, step)
        wr.grad = g.clone()
        opt.step()
    torch.cuda.synchronize()
    assert torch.allclose(w, wr.detach(), rtol=1e-5, atol=1e-6)
    assert torch.equal(out, w.to(torch.bfloat16))


@pytest.mark.parametrize("split", [2, 3, 0])
@pytest.mark.parametrize("accumulate", [False, True])
@pytest.mark.parametrize("epi", [0, 1])
def test_gemm_split_k_wgrad(split, accumulate, epi):
    """Split-K partials reduced with red.add.f32 (wgrad shapes with few tiles)."""
    k = K()
    M, N, Kd = 256, 384, 1000
    dy, x = rnd(Kd, M), rnd(Kd, N)
    dw = torch.randn(M, N, device="cuda")
    base = dw.clone()
    k.gemm_raw(M=M, N=N, K=Kd, A=dy, lda=M, a_mn=True, B=x, ldb=N, b_mn=True, Cout=dw, ldc=N,
               accumulate=accumulate, split_k=split, epilogue=epi)
    torch.cuda.synchronize()
    ref = dy.float().t() @ x.float() + (base if accumulate else 0)
    close(dw, ref, rel=5e-3)


def test_colsum_shapes():
    k = K()
    for rows, cols in ((4096, 1024), (4096, 3072), (4096, 4096), (100, 64), (4096, 30528)):
        x = rnd(rows, cols)
        out = torch.zeros(cols, device="cuda")
        k.colsum(x, out)
        torch.cuda.synchronize()
        close(out, x.float().sum(0), rel=5e-3)


def test_gemm_fused_gelu_backward():
    """dgrad epilogue residual_mode 1: dx = (dy @ w) * gelu'(f)."""
    k = K()
    M, N, Kd = 512, 768, 256
    dy, w, f = rnd(M, Kd), rnd(Kd, N, scale=0.05), rnd(M, N)
    dx = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    k.linear_dgrad(dy, w, dx, gelu_of=f)
    fr = f.float().requires_grad_()
    torch.nn.functional.gelu(fr, approximate="tanh").backward(dy.float() @ w.float())
    torch.cuda.synchronize()
    close(dx, fr.grad)


@pytest.mark.parametrize("M,N,Kd", [(512, 768, 256), (300, 520, 200), (4096, 4096, 1024)])
def test_gemm_fused_colsum(M, N, Kd):
    """colsum epilogue: the column sums of the stored bf16 dx are added to an f32
    accumulator (fc1's bias gradient fused into fc2's dgrad), with ragged M / N."""
    k = K()
    dy, w, f = rnd(M, Kd), rnd(Kd, N, scale=0.05), rnd(M, N)
    dx = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    db = torch.randn(N, device="cuda")
    db0 = db.clone()
    k.linear_dgrad(dy, w, dx, gelu_of=f, dbias=db)
    torch.cuda.synchronize()
    close(db - db0, dx.float().sum(0), rel=5e-3)  # sums of the stored values
    fr = f.float().requires_grad_()
    torch.nn.functional.gelu(fr, approximate="tanh").backward(dy.float() @ w.float())
    close(db - db0, fr.grad.sum(0))
    # plain bf16 GEMM with bias + colsum (no residual)
    x, wt, b = rnd(M, Kd), rnd(N, Kd, scale=0.05), rnd(N)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cs = torch.zeros(N, device="cuda")
    k.gemm_raw(M=M, N=N, K=Kd, A=x, lda=Kd, B=wt, ldb=Kd, Cout=y, ldc=N, bias=b, colsum=cs)
    torch.cuda.synchronize()
    close(cs, y.float().sum(0), rel=5e-3)


def _attn_ref(qkv, b, s, A, causal):
    H = A * 64
    q = qkv[:, :H].float().reshape(b, s, A, 64).transpose(1, 2)
    k = qkv[:, H:2 * H].float().reshape(b, s, A, 64).transpose(1, 2)
    v = qkv[:, 2 * H:].float().reshape(b, s, A, 64).transpose(1, 2)
    sc = q @ k.transpose(-1, -2) / 8.0
    if causal:
        sc = sc.masked_fill(torch.ones(s, s, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
    lse = torch.logsumexp(sc, -1)
    o = torch.softmax(sc, -1) @ v
    return o.transpose(1, 2).reshape(b * s, H), lse


# the last two cases have more (tile, head, batch) units than SMs: the persistent
# kernels walk several units per CTA (CTA-global barrier phases, buffer reuse)
@pytest.mark.parametrize("b,s,A,causal", [(2, 128, 2, False), (2, 512, 3, False), (1, 512, 2, True),
                                          (3, 64, 2, False), (2, 192, 2, True), (2, 1024, 1, True),
                                          (8, 512, 16, False), (4, 1024, 8, True)])
def test_fused_attention_forward(b, s, A, causal):
    k = K()
    qkv = rnd(b * s, 3 * A * 64, scale=1.5)
    out = torch.empty(b * s, A * 64, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, A, s, device="cuda")
    k.attn_fwd(qkv, out, lse, b, s, A, causal)
    torch.cuda.synchronize()
    o_ref, lse_ref = _attn_ref(qkv, b, s, A, causal)
    close(out, o_ref)
    assert (lse - lse_ref).abs().max().item() < 2e-2


@pytest.mark.parametrize("causal", [False, True])
def test_fused_attention_forward_rescale(causal):
    """Keys of later tiles carry far larger logits, so each key half's running
    max grows by more than 2^8 mid-row: the O accumulators in TMEM are rescaled
    in place (the rare path of the split-key forward)."""
    k = K()
    b, s, A = 2, 512, 4
    H = A * 64
    qkv = rnd(b * s, 3 * H, scale=1.0)
    kv = qkv.view(b, s, 3 * H)
    for t in range(1, s // 128):  # K rows of tile t scaled up by 2.5^t
        kv[:, t * 128:(t + 1) * 128, H:2 * H] *= 2.5 ** t
    out = torch.empty(b * s, H, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, A, s, device="cuda")
    k.attn_fwd(qkv, out, lse, b, s, A, causal)
    torch.cuda.synchronize()
    o_ref, lse_ref = _attn_ref(qkv, b, s, A, causal)
    close(out, o_ref)
    assert ((lse - lse_ref).abs() / lse_ref.abs().clamp_min(1)).max().item() < 2e-2


@pytest.mark.parametrize("b,s,A,causal", [(2, 128, 2, False), (2, 512, 2, False), (1, 512, 2, True),
                                          (3, 64, 2, False), (2, 192, 1, True), (1, 1024, 1, True),
                                          (8, 512, 16, False), (4, 1024, 8, True)])
def test_fused_attention_backward(b, s, A, causal):
    k = K()
    H = A * 64
    qkv = rnd(b * s, 3 * H, scale=1.5)
    out = torch.empty(b * s, H, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, A, s, device="cuda")
    k.attn_fwd(qkv, out, lse, b, s, A, causal)
    dout = rnd(b * s, H)
    dqkv = torch.empty_like(qkv)
    dbias = torch.randn(3 * H, device="cuda")
    db0 = dbias.clone()
    k.attn_bwd(qkv, out, dout, lse, dqkv, b, s, A, causal, dbias=dbias)
    torch.cuda.synchronize()
    x = qkv.float().requires_grad_()
    o_ref, _ = _attn_ref(x, b, s, A, causal)
    o_ref.backward(dout.float())
    for part in range(3):
        close(dqkv[:, part * H:(part + 1) * H], x.grad[:, part * H:(part + 1) * H])
        # fused QKV bias gradient: column sums of dQ | dK | dV, against the fp32
        # reference's; the dK sums are exactly zero (softmax rows of dS sum to 0),
        # so the tolerance is relative to the sums of |d| rather than to the sums
        g = x.grad[:, part * H:(part + 1) * H]
        err = ((dbias - db0)[part * H:(part + 1) * H] - g.sum(0)).abs().max().item()
        assert err <= 1e-2 * g.abs().sum(0).max().item(), f"part {part}: max err {err:.4g}"


@pytest.mark.parametrize("b,t,s,A", [(2, 128, 512, 2), (3, 64, 192, 2), (16, 128, 512, 16)])
def test_fused_cross_attention(b, t, s, A):
    """T5 cross-attention: queries from the decoder (t), keys / values from the
    encoder output (s), separate buffers, forward and backward."""
    k = K()
    H = A * 64
    q = rnd(b * t, H, scale=1.5)
    kv = rnd(b * s, 2 * H, scale=1.5)
    out = torch.empty(b * t, H, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, A, t, device="cuda")
    k.attn_fwd_cross(q, kv, out, lse, b, t, s, A)
    dout = rnd(b * t, H)
    dq = torch.empty_like(q)
    dkv = torch.empty_like(kv)
    k.attn_bwd_cross(q, kv, out, dout, lse, dq, dkv, b, t, s, A)
    torch.cuda.synchronize()
    qr = q.float().requires_grad_()
    kvr = kv.float().requires_grad_()
    qh = qr.reshape(b, t, A, 64).transpose(1, 2)
    kh = kvr[:, :H].reshape(b, s, A, 64).transpose(1, 2)
    vh = kvr[:, H:].reshape(b, s, A, 64).transpose(1, 2)
    sc = qh @ kh.transpose(-1, -2) / 8.0
    o_ref = (torch.softmax(sc, -1) @ vh).transpose(1, 2).reshape(b * t, H)
    close(out, o_ref)
    assert (lse - torch.logsumexp(sc, -1)).abs().max().item() < 2e-2
    o_ref.backward(dout.float())
    close(dq, qr.grad)
    close(dkv[:, :H], kvr.grad[:, :H])
    close(dkv[:, H:], kvr.grad[:, H:])
