"""CNN node kernels (AmoebaNet-D) against plain PyTorch fp32 references."""
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def K():
    from paper_2505_05856_b200 import _lib, kernels
    _lib.init_device(0)
    return kernels


def close(got, want, rel=2e-2):
    got, want = got.float(), want.float()
    scale = want.abs().max().item() + 1e-6
    err = (got - want).abs().max().item()
    assert err <= rel * scale, f"max err {err:.4g} vs scale {scale:.4g}"


def nhwc(t):  # [b, C, H, W] -> [b*H*W, C]
    b, C, H, W = t.shape
    return t.permute(0, 2, 3, 1).reshape(b * H * W, C)


def nchw(t, b, H, W):
    return t.reshape(b, H, W, -1).permute(0, 3, 1, 2)


def test_relu():
    k = K()
    x = torch.randn(1000, 64, device="cuda").bfloat16()
    y = torch.empty_like(x)
    k.relu_fwd(x, y)
    dy = torch.randn_like(x)
    dx = torch.empty_like(x)
    k.relu_bwd(dy, y, dx)
    torch.cuda.synchronize()
    assert torch.equal(y, torch.relu(x))
    assert torch.equal(dx, torch.where(x > 0, dy, torch.zeros_like(dy)))


@pytest.mark.parametrize("b,H,W,C,stride", [(2, 14, 14, 64, 1), (2, 15, 13, 32, 2), (1, 56, 56, 128, 2),
                                            (3, 7, 7, 256, 1)])
def test_dwconv3(b, H, W, C, stride):
    k = K()
    x = torch.randn(b, C, H, W, device="cuda")
    w = torch.randn(C, 1, 3, 3, device="cuda") * 0.3
    xb, wb = x.bfloat16(), w.bfloat16()
    ref = F.conv2d(xb.float(), wb.float(), stride=stride, padding=1, groups=C)
    Ho, Wo = ref.shape[2], ref.shape[3]
    y = torch.empty(b * Ho * Wo, C, device="cuda", dtype=torch.bfloat16)
    k.dwconv3_fwd(nhwc(xb).contiguous(), wb.reshape(C, 9).contiguous(), y, b, H, W, C, stride)
    torch.cuda.synchronize()
    close(y, nhwc(ref))
    # backward
    xr = xb.float().requires_grad_()
    wr = wb.float().requires_grad_()
    out = F.conv2d(xr, wr, stride=stride, padding=1, groups=C)
    g = torch.randn_like(out).bfloat16()
    out.backward(g.float())
    dx = torch.empty(b * H * W, C, device="cuda", dtype=torch.bfloat16)
    dw = torch.zeros(C, 9, device="cuda")
    k.dwconv3_bwd(nhwc(xb).contiguous(), wb.reshape(C, 9).contiguous(), nhwc(g).contiguous(), dx, dw,
                  b, H, W, C, stride)
    torch.cuda.synchronize()
    close(dx, nhwc(xr.grad))
    close(dw, wr.grad.reshape(C, 9), rel=1e-2)


@pytest.mark.parametrize("P,C", [(4096, 64), (1000, 256), (25088, 128), (98, 1024)])
def test_batchnorm(P, C):
    k = K()
    x = (torch.randn(P, C, device="cuda") * 2 + 0.5).bfloat16()
    gamma = (torch.rand(C, device="cuda") + 0.5).bfloat16()
    beta = torch.randn(C, device="cuda").bfloat16()
    y = torch.empty_like(x)
    st = torch.empty(2, C, device="cuda")
    k.bn_fwd(x, gamma, beta, y, st)
    xr = x.float().requires_grad_()
    gr = gamma.float().requires_grad_()
    br = beta.float().requires_grad_()
    ref = F.batch_norm(xr, None, None, gr, br, training=True, eps=1e-5)
    torch.cuda.synchronize()
    close(y, ref)
    dy = torch.randn_like(x)
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.full((C,), 0.25, device="cuda")
    db = torch.full((C,), -0.5, device="cuda")
    ws = torch.empty(2 * C, device="cuda")
    k.bn_bwd(dy, x, st, gamma, dx, dg, db, ws)
    torch.cuda.synchronize()
    close(dx, xr.grad)
    close(dg - 0.25, gr.grad, rel=1e-2)
    close(db + 0.5, br.grad, rel=1e-2)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("b,H,W,C,stride", [(2, 14, 14, 64, 1), (2, 15, 13, 32, 2), (1, 28, 28, 128, 2)])
def test_pool3(mode, b, H, W, C, stride):
    k = K()
    x = torch.randn(b, C, H, W, device="cuda").bfloat16()
    xr = x.float().requires_grad_()
    if mode == 0:
        ref = F.max_pool2d(xr, 3, stride, 1)
    else:
        ref = F.avg_pool2d(xr, 3, stride, 1, count_include_pad=False)
    Ho, Wo = ref.shape[2], ref.shape[3]
    y = torch.empty(b * Ho * Wo, C, device="cuda", dtype=torch.bfloat16)
    arg = torch.empty(b * Ho * Wo, C, device="cuda", dtype=torch.uint8) if mode == 0 else None
    k.pool3_fwd(nhwc(x).contiguous(), y, arg, b, H, W, C, stride, mode)
    torch.cuda.synchronize()
    close(y, nhwc(ref.detach()))
    g = torch.randn_like(ref).bfloat16()
    ref.backward(g.float())
    dx = torch.empty(b * H * W, C, device="cuda", dtype=torch.bfloat16)
    k.pool3_bwd(nhwc(g).contiguous(), arg, dx, b, H, W, C, stride, mode)
    torch.cuda.synchronize()
    close(dx, nhwc(xr.grad))


def test_copy_cols_concat():
    k = K()
    a, b_ = torch.randn(300, 64, device="cuda").bfloat16(), torch.randn(300, 128, device="cuda").bfloat16()
    out = torch.empty(300, 192, device="cuda", dtype=torch.bfloat16)
    k.copy_cols(a, 64, out, 192, 300, 64)
    k.copy_cols(b_, 128, out[:, 64:], 192, 300, 128)
    torch.cuda.synchronize()
    assert torch.equal(out, torch.cat([a, b_], 1))
    g = torch.randn_like(a)
    g0 = g.float().clone()
    k.copy_cols(out, 192, g, 64, 300, 64, accumulate=True)
    torch.cuda.synchronize()
    close(g, g0 + a.float())


def test_im2col_stem_matches_conv():
    k = K()
    b, H, W, C, Co, stride = 2, 32, 32, 8, 64, 2
    x = torch.randn(b, C, H, W, device="cuda").bfloat16()
    w = (torch.randn(Co, C, 3, 3, device="cuda") * 0.1).bfloat16()
    Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
    cols = torch.empty(b * Ho * Wo, 9 * C, device="cuda", dtype=torch.bfloat16)
    k.im2col3(nhwc(x).contiguous(), cols, b, H, W, C, stride)
    wk = w.permute(0, 2, 3, 1).reshape(Co, 9 * C).contiguous()  # [Co, (r, s, c)]
    y = torch.empty(b * Ho * Wo, Co, device="cuda", dtype=torch.bfloat16)
    k.linear_fwd(cols, wk, y)
    torch.cuda.synchronize()
    ref = F.conv2d(x.float(), w.float(), stride=stride, padding=1)
    close(y, nhwc(ref))


def test_global_average_pool():
    k = K()
    b, HW, C = 4, 49, 256
    x = torch.randn(b * HW, C, device="cuda").bfloat16()
    y = torch.empty(b, C, device="cuda", dtype=torch.bfloat16)
    k.gap_fwd(x, y, b, HW, C)
    dy = torch.randn(b, C, device="cuda").bfloat16()
    dx = torch.empty_like(x)
    k.gap_bwd(dy, dx, b, HW, C)
    torch.cuda.synchronize()
    close(y, x.float().reshape(b, HW, C).mean(1))
    close(dx, (dy.float() / HW).repeat_interleave(HW, 0))
