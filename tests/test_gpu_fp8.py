"""GPU tests of the FP8 (E4M3) rung: quantizers bit-exact vs torch's CPU
float8_e4m3fn conversion of x / s (s = absmax / 448, IEEE), the tcgen05
kind::f8f6f4 GEMM vs an FP64 product of the dequantized operands (FP32
accumulation: 1e-5 of the output scale), and the FP8 Linear fwd + FP16 bwd vs
an FP32 torch reference of the same quantized operands."""
import pytest
import torch

from paper_2407_02327_b200 import ops
from paper_2407_02327_b200.qlinear import FP8, qlinear

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _ref_fp8(x_cpu, s):
    return (x_cpu / s).to(torch.float8_e4m3fn)


@pytest.mark.parametrize("shape", [(4096, 768), (333, 1000), (7,)])
def test_quantize_fp8_per_tensor_bit_exact(shape):
    torch.manual_seed(1)
    x = torch.randn(shape, device=DEV) * 3
    q, s = ops.quantize_fp8(x)
    am = x.abs().max().item()
    assert s.item() == torch.tensor(am, dtype=torch.float32).div(448.0).item()
    ref = _ref_fp8(x.cpu(), s.cpu())
    assert torch.equal(q.cpu().view(torch.uint8), ref.view(torch.uint8))


def test_quantize_fp8_rows_bit_exact():
    torch.manual_seed(2)
    w = torch.randn(300, 768, device=DEV) * torch.rand(300, 1, device=DEV)
    w[5] = 0
    q, s = ops.quantize_fp8_rows(w)
    am = w.abs().amax(dim=1).cpu()
    s_ref = torch.where(am > 0, am / 448.0, torch.ones_like(am))
    assert torch.equal(s.cpu(), s_ref)
    ref = (w.cpu() / s_ref[:, None]).to(torch.float8_e4m3fn)
    assert torch.equal(q.cpu().view(torch.uint8), ref.view(torch.uint8))


@pytest.mark.parametrize("mnk", [(4096, 3072, 768), (300, 200, 144), (8192, 1024, 1024)])
def test_gemm_f8_vs_fp64(mnk):
    M, N, K = mnk
    torch.manual_seed(sum(mnk))
    a, sa = ops.quantize_fp8(torch.randn(M, K, device=DEV))
    b, sb = ops.quantize_fp8_rows(torch.randn(N, K, device=DEV))
    bias = torch.randn(N, device=DEV)
    y = ops.gemm_f8(a, b, sa, sb, bias)
    ad = a.float().double() * sa.double()
    bd = b.float().double() * sb.double()[:, None]
    ref = ad @ bd.T + bias.double()
    assert ((y.double() - ref).abs().max() / ref.abs().max()).item() < 1e-5
    y16 = ops.gemm_f8(a, b, sa, sb, bias, out_dtype=torch.float16)
    assert ((y16.double() - ref).abs().max() / ref.abs().max()).item() < 2e-3


def test_fp8_linear_fwd_bwd():
    torch.manual_seed(4)
    M, N, K = 512, 768, 1024
    x = torch.randn(M, K, device=DEV, requires_grad=True)
    w = (torch.randn(N, K, device=DEV) / K ** 0.5).requires_grad_(True)
    b = torch.randn(N, device=DEV, requires_grad=True)
    y = qlinear(x, w, b, FP8)
    assert y.dtype == torch.float32
    xq, xs = ops.quantize_fp8(x.detach())
    wq, ws = ops.quantize_fp8_rows(w.detach())
    xd, wd = xq.float() * xs, wq.float() * ws[:, None]
    ref = xd @ wd.T + b.detach()
    assert ((y - ref).abs().max() / ref.abs().max()).item() < 1e-5
    g = torch.randn_like(y)
    y.backward(g)
    g16 = g.half().float()
    dx_ref = g16 @ w.detach().half().float()
    dw_ref = g16.T @ xd
    assert ((x.grad - dx_ref).abs().max() / dx_ref.abs().max()).item() < 1e-2
    assert ((w.grad - dw_ref).abs().max() / dw_ref.abs().max()).item() < 1e-3
    torch.testing.assert_close(b.grad, g.sum(0), rtol=1e-4, atol=1e-3)
