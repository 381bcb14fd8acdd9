"""Conv2d (config 3, ResNet-50 layer shapes at small batch): im2col / col2im vs
the oracle bit for bit, the INT8 conv forward bit-exact (int8 column matrix,
int32 GEMM, dequant epilogue), FP16 forward and both backwards within tolerance."""
import numpy as np
import pytest
import torch

from paper_2407_02327_b200 import ops
from paper_2407_02327_b200.qconv import qconv2d
from paper_2407_02327_b200.qlinear import FP16, INT8

DEV = "cuda"

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[1, 0], ids=["tma_im2col", "gather"])
def conv_impl(request):
    """Both implicit-conv operand loaders: TMA im2col mode and cp.async lanes."""
    ops.conv_set_impl(request.param)
    yield request.param
    ops.conv_set_impl(1)

# (N, H, W, C, Cout, R, stride, pad): stem 7x7/2, res2 3x3, res3 1x1/2 downsample, res5 3x3
CASES = [(1, 32, 32, 3, 64, 7, 2, 3), (2, 14, 14, 64, 64, 3, 1, 1), (2, 28, 28, 128, 256, 1, 2, 0),
         (2, 7, 7, 512, 512, 3, 1, 1), (3, 9, 11, 16, 48, 3, 2, 1)]


def _inputs(case, seed):
    N, H, W, C, Co, R, s, p = case
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(N, H, W, C)).astype(np.float32)
    w = (rng.uniform(-1, 1, size=(Co, R, R, C)) / np.sqrt(R * R * C)).astype(np.float32)
    b = (rng.normal(size=Co) * 0.1).astype(np.float32)
    return x, w, b


@pytest.mark.parametrize("case", CASES)
def test_im2col_col2im_bit_exact(case, cpuref):
    N, H, W, C, Co, R, s, p = case
    x, _, _ = _inputs(case, 1)
    xq, _ = cpuref.quantize_per_tensor(x)
    A, (P, Q) = ops.im2col(torch.from_numpy(xq).cuda(), R, R, (s, s), (p, p))
    Aref, _ = cpuref.im2col(xq, R, R, (s, s), (p, p), ld=A.shape[1])
    assert np.array_equal(A.cpu().numpy(), Aref)
    x16 = x.astype(np.float16)
    A16, _ = ops.im2col(torch.from_numpy(x16).cuda(), R, R, (s, s), (p, p))
    Aref16, _ = cpuref.im2col(x16, R, R, (s, s), (p, p), ld=A16.shape[1])
    assert np.array_equal(A16.cpu().numpy().view(np.uint16), Aref16.view(np.uint16))
    dcol = np.random.default_rng(2).normal(size=A.shape).astype(np.float32)
    dx = ops.col2im(torch.from_numpy(dcol).cuda(), x.shape, R, R, (s, s), (p, p))
    dx_ref = cpuref.col2im(dcol, x.shape, R, R, (s, s), (p, p))
    np.testing.assert_allclose(dx.cpu().numpy(), dx_ref, rtol=1e-5, atol=1e-5)


def _run(case, precision, seed=3):
    N, H, W, C, Co, R, s, p = case
    x, w, b = _inputs(case, seed)
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    wt = torch.from_numpy(w).cuda().requires_grad_(True)
    bt = torch.from_numpy(b).cuda().requires_grad_(True)
    y = qconv2d(xt, wt, bt, (s, s), (p, p), precision)
    g = np.random.default_rng(seed + 1).normal(size=tuple(y.shape)).astype(np.float32)
    y.backward(torch.from_numpy(g).cuda().to(y.dtype))
    torch.cuda.synchronize()
    return x, w, b, g, y, xt.grad, wt.grad, bt.grad


def _rel(a, b):
    a = a.detach().float().cpu().numpy() if torch.is_tensor(a) else a
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-12)


@pytest.mark.parametrize("case", CASES)
def test_int8_conv_vs_oracle(case, cpuref):
    N, H, W, C, Co, R, s, p = case
    x, w, b, g, y, dx, dw, db = _run(case, INT8)
    # forward: same quantized column matrix, exact int32 GEMM, same epilogue -> bit-exact
    xq, sx = cpuref.quantize_per_tensor(x)
    K = R * R * C
    kp = (K + 15) // 16 * 16
    A, (P, Q) = cpuref.im2col(xq, R, R, (s, s), (p, p), ld=kp)
    w2 = np.zeros((Co, kp), np.float32)
    w2[:, :K] = w.reshape(Co, K)
    wq, sw = cpuref.quantize_per_channel(w2)
    acc = cpuref.gemm_s8_tn(A, wq)
    y_ref = cpuref.dequant_epilogue(acc, sx, sw, b).reshape(N, P, Q, Co)
    assert np.array_equal(y.detach().cpu().numpy(), y_ref)
    # backward (FP16 compute): dgrad via col2im, wgrad against the quantized columns
    g2 = g.reshape(-1, Co)
    g16 = g2.astype(np.float16)
    w16 = w2.astype(np.float16)
    dcol = cpuref.gemm_f16_tn(g16, np.ascontiguousarray(w16.T))
    dx_ref = cpuref.col2im(dcol, x.shape, R, R, (s, s), (p, p))
    assert _rel(dx, dx_ref) < 1e-2
    dw_ref = cpuref.gemm_f16_tn(np.ascontiguousarray(g16.T), np.ascontiguousarray(A.T.astype(np.float16)),
                                float(sx))[:, :K].reshape(w.shape)
    assert _rel(dw, dw_ref) < 1e-3
    assert _rel(db, g2.sum(0)) < 1e-4


@pytest.mark.parametrize("case", CASES[:4])
def test_fp16_conv_vs_torch_fp32(case):
    N, H, W, C, Co, R, s, p = case
    x, w, b, g, y, dx, dw, db = _run(case, FP16)
    xt = torch.from_numpy(x).cuda().permute(0, 3, 1, 2).requires_grad_(True)
    wt = torch.from_numpy(w).cuda().permute(0, 3, 1, 2).requires_grad_(True)
    bt = torch.from_numpy(b).cuda().requires_grad_(True)
    ref = torch.nn.functional.conv2d(xt, wt, bt, s, p)
    ref.backward(torch.from_numpy(g).cuda().permute(0, 3, 1, 2))
    assert y.dtype == torch.float16
    assert _rel(y, ref.permute(0, 2, 3, 1).detach().cpu().numpy()) < 1e-2
    assert _rel(dx, xt.grad.permute(0, 2, 3, 1).cpu().numpy()) < 1e-2
    assert _rel(dw, wt.grad.permute(0, 2, 3, 1).cpu().numpy()) < 1e-2
    assert _rel(db, bt.grad.cpu().numpy()) < 1e-3


@pytest.mark.parametrize("geom", [(2, 14, 14, 128, 256, 3, 1, 1), (2, 15, 15, 128, 128, 3, 2, 1),
                                  (3, 7, 7, 256, 512, 1, 1, 0), (1, 28, 28, 128, 64, 1, 2, 0),
                                  (2, 9, 11, 128, 200, 3, 1, 1),
                                  # 64-byte channel runs: two taps per 128-byte K-slice
                                  (2, 14, 14, 64, 64, 3, 1, 1), (2, 15, 15, 64, 128, 3, 2, 1),
                                  (3, 9, 9, 64, 256, 1, 1, 0), (2, 12, 12, 64, 96, 1, 2, 0),
                                  (1, 11, 7, 192, 64, 3, 1, 1)])
def test_implicit_conv_int8_bit_exact_vs_im2col(geom, conv_impl):
    """Implicit-GEMM forward (A gathered by the producer warp) == im2col + GEMM:
    same int8 operands, same K order -> identical int32 accumulators and epilogue."""
    N, H, W, C, Co, R, st, pd = geom
    torch.manual_seed(sum(geom))
    x = torch.randint(-127, 128, (N, H, W, C), dtype=torch.int8, device=DEV)
    w2 = torch.randint(-127, 128, (Co, R * R * C), dtype=torch.int8, device=DEV)
    sa = torch.tensor([0.0123], device=DEV)
    sb = torch.rand(Co, device=DEV) * 0.01
    bias = torch.randn(Co, device=DEV)
    assert ops.implicit_conv_ok(C, torch.int8)
    y, (P, Q) = ops.conv_fwd_implicit(x, w2, R, R, (st, st), (pd, pd), sa, sb, bias)
    A, (P2, Q2) = ops.im2col(x, R, R, (st, st), (pd, pd))
    _, y_ref = ops.gemm_s8(A, w2, sa, sb, bias)
    assert (P, Q) == (P2, Q2)
    assert torch.equal(y, y_ref)


@pytest.mark.parametrize("geom", [(2, 14, 14, 64, 256, 3, 1, 1), (2, 28, 28, 128, 128, 3, 2, 1),
                                  (4, 7, 7, 64, 96, 1, 1, 0), (2, 10, 10, 32, 64, 3, 1, 1)])
def test_implicit_conv_fp16_matches_im2col(geom, conv_impl):
    N, H, W, C, Co, R, st, pd = geom
    torch.manual_seed(sum(geom))
    x = torch.randn(N, H, W, C, device=DEV).half()
    w2 = (torch.randn(Co, R * R * C, device=DEV) / (R * R * C) ** 0.5).half()
    y, _ = ops.conv_fwd_implicit(x, w2, R, R, (st, st), (pd, pd), out_dtype=torch.float16)
    A, _ = ops.im2col(x, R, R, (st, st), (pd, pd))
    y_ref = ops.gemm_f16(A, w2, out_dtype=torch.float16)
    assert torch.equal(y, y_ref)  # same operands, same K order, same accumulation


@pytest.mark.parametrize("geom", [(2, 10, 13, 128, 128, 1, 3, 1, 2, 0, 1), (1, 12, 9, 64, 64, 3, 1, 2, 1, 1, 0),
                                  (2, 11, 11, 128, 256, 5, 5, 2, 2, 2, 2)])
def test_implicit_conv_asymmetric_geometry(geom, conv_impl):
    """R != S, different strides and pads per axis: the TMA im2col map's W/H
    ordering and bounding box match im2col (oracle-pinned) bit for bit."""
    N, H, W, C, Co, R, S, sh, sw, ph, pw = geom
    torch.manual_seed(sum(geom))
    x = torch.randn(N, H, W, C, device=DEV).half()
    w2 = (torch.randn(Co, R * S * C, device=DEV) / (R * S * C) ** 0.5).half()
    y, (P, Q) = ops.conv_fwd_implicit(x, w2, R, S, (sh, sw), (ph, pw), out_dtype=torch.float16)
    A, (P2, Q2) = ops.im2col(x, R, S, (sh, sw), (ph, pw))
    assert (P, Q) == (P2, Q2)
    assert torch.equal(y, ops.gemm_f16(A, w2, out_dtype=torch.float16))
    dy = torch.randn(N, P, Q, Co, device=DEV).half()
    wt = w2.view(Co, R, S, C)
    xt = x.double().permute(0, 3, 1, 2).requires_grad_(True)
    wd = wt.double().permute(0, 3, 1, 2).requires_grad_(True)
    torch.nn.functional.conv2d(xt, wd, None, (sh, sw), (ph, pw)).backward(dy.double().permute(0, 3, 1, 2))
    dx = ops.conv_dgrad_implicit(dy, wt, (N, H, W, C), (sh, sw), (ph, pw))
    assert _nrel(dx, xt.grad.permute(0, 2, 3, 1)) < 1e-5
    dw = ops.conv_wgrad_implicit(x, dy.view(-1, Co), R, S, (sh, sw), (ph, pw))
    assert _nrel(dw.view(Co, R, S, C), wd.grad.permute(0, 2, 3, 1)) < 1e-5


def test_implicit_conv_rejects_narrow_channels():
    x = torch.zeros(1, 8, 8, 3, dtype=torch.int8, device=DEV)
    w2 = torch.zeros(16, 27, dtype=torch.int8, device=DEV)
    with pytest.raises(Exception, match="64 bytes"):
        ops.conv_fwd_implicit(x, w2, 3, 3, (1, 1), (1, 1), torch.ones(1, device=DEV), torch.ones(16, device=DEV))


DGRAD_GEOMS = [(2, 14, 14, 64, 64, 3, 1, 1), (2, 15, 15, 128, 128, 3, 2, 1), (2, 16, 16, 64, 128, 3, 2, 1),
               (1, 28, 28, 256, 128, 1, 2, 0), (3, 7, 7, 200, 64, 1, 1, 0), (2, 9, 11, 24, 192, 3, 1, 1),
               (1, 32, 32, 3, 64, 7, 2, 3)]


def _f64_conv_grads(x16, w16, dy16, st, pd):
    """Float64 autograd of conv2d on the FP16 values (the GEMMs accumulate
    exact FP16 products in FP32: tolerance 1e-5 relative to the norm)."""
    xt = x16.double().permute(0, 3, 1, 2).requires_grad_(True)
    wt = w16.double().permute(0, 3, 1, 2).requires_grad_(True)
    y = torch.nn.functional.conv2d(xt, wt, None, st, pd)
    y.backward(dy16.double().permute(0, 3, 1, 2))
    return xt.grad.permute(0, 2, 3, 1), wt.grad.permute(0, 2, 3, 1)


def _nrel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))


@pytest.mark.parametrize("geom", DGRAD_GEOMS)
def test_implicit_dgrad_vs_f64(geom, conv_impl):
    """Implicit dgrad (dY taps gathered by the producer warp, W read in place
    through a 3-D TMA map) == conv2d's input gradient; strided convs keep only
    the taps on the stride grid."""
    N, H, W, C, Co, R, st, pd = geom
    if not ops.implicit_dgrad_ok(C, Co):  # (the op itself also takes strided geometries)
        pytest.skip("geometry outside the implicit dgrad (C % 8)")
    torch.manual_seed(sum(geom))
    P, Q = ops.conv_out_size(H, W, R, R, (st, st), (pd, pd))
    x16 = torch.randn(N, H, W, C, device=DEV).half()
    w16 = (torch.randn(Co, R, R, C, device=DEV) / (R * R * C) ** 0.5).half()
    dy16 = torch.randn(N, P, Q, Co, device=DEV).half()
    dx = ops.conv_dgrad_implicit(dy16, w16, (N, H, W, C), (st, st), (pd, pd))
    dx_ref, _ = _f64_conv_grads(x16, w16, dy16, (st, st), (pd, pd))
    assert dx.shape == (N, H, W, C) and dx.dtype == torch.float32
    assert _nrel(dx, dx_ref) < 1e-5
    # and the col2im path on the same operands
    dcol = ops.gemm_f16(dy16.view(-1, Co), w16.view(Co, -1).contiguous(), out_dtype=torch.float32, b_mn=True) \
        if (R * R * C) % 8 == 0 else None
    if dcol is not None:
        dx2 = ops.col2im(dcol, (N, H, W, C), R, R, (st, st), (pd, pd))
        assert _nrel(dx, dx2) < 1e-5  # different FP32 summation order of the taps


WGRAD_GEOMS = [(2, 14, 14, 64, 64, 3, 1, 1), (2, 15, 15, 128, 256, 3, 2, 1), (3, 7, 7, 64, 200, 1, 1, 0),
               (1, 28, 28, 128, 64, 1, 2, 0), (8, 56, 56, 64, 64, 3, 1, 1)]


@pytest.mark.parametrize("geom", WGRAD_GEOMS)
def test_implicit_wgrad_vs_f64(geom, conv_impl):
    """Implicit wgrad (column matrix gathered as the MN-major B operand, K = pixels
    split across SMs and reduce-added) == conv2d's weight gradient; accumulate
    and the device alpha behave as in qsync_gemm_f16."""
    N, H, W, C, Co, R, st, pd = geom
    torch.manual_seed(sum(geom))
    P, Q = ops.conv_out_size(H, W, R, R, (st, st), (pd, pd))
    x16 = torch.randn(N, H, W, C, device=DEV).half()
    w16 = torch.zeros(Co, R, R, C, device=DEV).half()
    dy16 = torch.randn(N, P, Q, Co, device=DEV).half()
    _, dw_ref = _f64_conv_grads(x16, w16, dy16, (st, st), (pd, pd))
    dw = ops.conv_wgrad_implicit(x16, dy16.view(-1, Co), R, R, (st, st), (pd, pd))
    assert dw.shape == (Co, R * R * C)
    # K = N*P*Q FP16 products summed in FP32 (tensor-core partial sums, split-K
    # partials reduce-added): 1e-5 of the norm up to ~4k pixels, 1e-4 beyond
    tol = 1e-5 if N * P * Q <= 4096 else 1e-4
    assert _nrel(dw.view(Co, R, R, C), dw_ref) < tol
    base = torch.randn(Co, R * R * C, device=DEV)
    out = base.clone()
    alpha = torch.tensor([0.25], device=DEV)
    ops.conv_wgrad_implicit(x16, dy16.view(-1, Co), R, R, (st, st), (pd, pd), out=out, accumulate=True,
                            alpha_dev=alpha)
    exp = base.double() + 0.25 * dw_ref.reshape(Co, -1)
    assert _nrel(out, exp) < tol


@pytest.mark.parametrize("precision", [INT8, FP16])
def test_qconv_backward_implicit_matches_col_path(precision, monkeypatch):
    """The autograd op with implicit dgrad/wgrad == the same op forced onto the
    materialised im2col / col2im path."""
    torch.manual_seed(5)
    x = torch.randn(2, 14, 14, 128, device=DEV, requires_grad=True)
    w = torch.randn(128, 3, 3, 128, device=DEV) * 0.03
    w.requires_grad_(True)
    g = torch.randn(2, 7, 7, 128, device=DEV)

    def run():
        x.grad = None
        w.grad = None
        y = qconv2d(x, w, None, (2, 2), (1, 1), precision)
        y.backward(g.to(y.dtype))
        return x.grad.clone(), w.grad.clone()

    dx_i, dw_i = run()
    monkeypatch.setattr(ops, "implicit_dgrad_ok", lambda *a: False)
    monkeypatch.setattr(ops, "implicit_wgrad_ok", lambda *a: False)
    dx_c, dw_c = run()
    assert _nrel(dx_i, dx_c) < 1e-5
    assert _nrel(dw_i, dw_c) < 1e-5
