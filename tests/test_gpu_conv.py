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
                                  (2, 9, 11, 128, 200, 3, 1, 1)])
def test_implicit_conv_int8_bit_exact_vs_im2col(geom):
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
                                  (4, 7, 7, 64, 96, 1, 1, 0)])
def test_implicit_conv_fp16_matches_im2col(geom):
    N, H, W, C, Co, R, st, pd = geom
    torch.manual_seed(sum(geom))
    x = torch.randn(N, H, W, C, device=DEV).half()
    w2 = (torch.randn(Co, R * R * C, device=DEV) / (R * R * C) ** 0.5).half()
    y, _ = ops.conv_fwd_implicit(x, w2, R, R, (st, st), (pd, pd), out_dtype=torch.float16)
    A, _ = ops.im2col(x, R, R, (st, st), (pd, pd))
    y_ref = ops.gemm_f16(A, w2, out_dtype=torch.float16)
    assert torch.equal(y, y_ref)  # same operands, same K order, same accumulation


def test_implicit_conv_rejects_narrow_channels():
    x = torch.zeros(1, 8, 8, 3, dtype=torch.int8, device=DEV)
    w2 = torch.zeros(16, 27, dtype=torch.int8, device=DEV)
    with pytest.raises(Exception, match="128 bytes"):
        ops.conv_fwd_implicit(x, w2, 3, 3, (1, 1), (1, 1), torch.ones(1, device=DEV), torch.ones(16, device=DEV))
