"""The FP32 operator kernel on the tensor cores (qsync_gemm_f32, 3xTF32 split):
FP32-level accuracy against float64 for every operand layout the Linear and
its backward use, with alpha / bias / accumulate; the split itself is exact
(hi + lo reproduces x to 2^-22); and the FP32-planned Linear / training step
run on it (training devices stay FP32, replayer.cpp:96-101)."""
import pytest
import torch

from paper_2407_02327_b200 import _lib, ops

pytestmark = pytest.mark.gpu


def _nrel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-300))


@pytest.mark.parametrize("M,N,K", [(4096, 768, 768), (256, 3072, 768), (130, 200, 64), (64, 1024, 1024),
                                   (768, 768, 4096), (768, 768, 2), (33, 5, 7)])
@pytest.mark.parametrize("layout", [0, 2, 3])
def test_gemm_f32_accuracy(M, N, K, layout):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K + layout)
    a = torch.randn(M, K, device="cuda", generator=g)
    b = torch.randn(N, K, device="cuda", generator=g) / K ** 0.5
    bias = torch.randn(N, device="cuda", generator=g)
    a_op = a.t().contiguous() if layout & 1 else a
    b_op = b.t().contiguous() if layout & 2 else b
    c = ops.gemm_f32(a_op, b_op, bias=bias, a_mn=bool(layout & 1), b_mn=bool(layout & 2))
    ref = a.double() @ b.double().t() + bias.double()
    err = _nrel(c, ref)
    # measured 6e-6 (K = 768) .. 3e-5 (K = 4096): the tensor core's FP32 accumulation
    # (truncating alignment, growing with K) + the dropped lo*lo term; 1xTF32 is ~1e-3
    assert err < 1e-4, err
    # accumulate + alpha (the wgrad form)
    base = torch.randn(M, N, device="cuda", generator=g)
    out = base.clone()
    ops.gemm_f32(a_op, b_op, alpha=0.5, out=out, accumulate=True, a_mn=bool(layout & 1), b_mn=bool(layout & 2))
    assert _nrel(out, base.double() + 0.5 * (a.double() @ b.double().t())) < 1e-4


def test_split_is_exact_to_tf32_residual():
    x = torch.randn(257, 96, device="cuda") * 1e3
    out = torch.empty(257, 3 * 96, device="cuda")
    _lib.call("qsync_split_tf32x3", x.data_ptr(), 257, 96, 0, 0, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    hi, hi2, lo = out[:, :96], out[:, 96:192], out[:, 192:]
    assert torch.equal(hi, hi2)
    assert int((hi.view(torch.int32) & 0x1FFF).abs().max()) == 0  # TF32: low 13 mantissa bits clear
    assert int((lo.view(torch.int32) & 0x1FFF).abs().max()) == 0
    r = (x.double() - hi.double() - lo.double()).abs() / x.double().abs().clamp_min(1e-30)
    assert float(r.max()) <= 2.0 ** -21
    xt = torch.empty(257, 3 * 96, device="cuda")
    _lib.call("qsync_split_tf32x3", x.t().contiguous().data_ptr(), 257, 96, 1, 1, xt.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    assert torch.equal(xt[:, :96], hi) and torch.equal(xt[:, 96:192], lo) and torch.equal(xt[:, 192:], hi)


def test_fp32_qlinear_on_tensor_cores():
    from paper_2407_02327_b200.qlinear import FP32, qlinear
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(512, 768, device="cuda", generator=g).requires_grad_(True)
    w = (torch.rand(3072, 768, device="cuda", generator=g) * 2 - 1).div_(768 ** 0.5).requires_grad_(True)
    b = torch.randn(3072, device="cuda", generator=g).requires_grad_(True)
    n0 = ops.launch_count()
    y = qlinear(x, w, b, FP32)
    dy = torch.randn_like(y)
    y.backward(dy)
    assert ops.launch_count() - n0 >= 6  # split + GEMM for fwd, dgrad and wgrad
    x64, w64 = x.detach().double(), w.detach().double()
    assert y.dtype == torch.float32 and _nrel(y, x64 @ w64.t() + b.detach().double()) < 1e-4
    assert _nrel(x.grad, dy.double() @ w64) < 1e-4
    assert _nrel(w.grad, dy.double().t() @ x64) < 1e-4
    assert _nrel(b.grad, dy.double().sum(0)) < 1e-6


@pytest.mark.parametrize("geom", [
    # (N, H, C, Cout, R, stride, pad): the ResNet-50 kinds -- 7x7/2 stem (C = 3),
    # 1x1/1 (read in place), 3x3/1, 3x3/2, 1x1/2 downsample, odd channel counts
    (2, 32, 3, 64, 7, 2, 3), (2, 14, 64, 256, 1, 1, 0), (2, 14, 64, 64, 3, 1, 1),
    (2, 15, 128, 128, 3, 2, 1), (2, 14, 256, 512, 1, 2, 0), (1, 9, 5, 7, 3, 1, 1)])
def test_fp32_conv_on_tensor_cores(geom):
    """FP32-planned Conv2d (im2col + 3xTF32 GEMM, col2im dgrad, GEMM wgrad) against
    float64 autograd: forward, dgrad and wgrad within 1e-5 of the norm."""
    import torch.nn.functional as F

    from paper_2407_02327_b200.qconv import qconv2d
    N, H, C, Co, R, st, pd = geom
    g = torch.Generator(device="cuda").manual_seed(sum(geom))
    x = torch.randn(N, H, H, C, device="cuda", generator=g, requires_grad=True)
    w = (torch.randn(Co, R, R, C, device="cuda", generator=g) / (R * R * C) ** 0.5).requires_grad_(True)
    b = torch.randn(Co, device="cuda", generator=g, requires_grad=True)
    y = qconv2d(x, w, b, (st, st), (pd, pd), "FP32")
    gy = torch.randn(y.shape, device="cuda", generator=g)
    dx, dw, db = torch.autograd.grad(y, (x, w, b), gy)
    xd, wd, bd = (t.detach().double().requires_grad_(True) for t in (x, w, b))
    yr = F.conv2d(xd.permute(0, 3, 1, 2), wd.permute(0, 3, 1, 2), bd, st, pd).permute(0, 2, 3, 1)
    dxr, dwr, dbr = torch.autograd.grad(yr, (xd, wd, bd), gy.double())
    assert y.dtype == torch.float32 and y.shape == yr.shape
    for got, ref in ((y, yr), (dx, dxr), (dw, dwr), (db, dbr)):
        assert _nrel(got, ref) < 1e-5
