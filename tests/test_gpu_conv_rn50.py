"""Config 3 parity at the REAL ResNet-50 geometries (224x224 input, batch 8 --
every distinct Conv2d shape of the 53 layers: the 7x7/2 stem with C = 3, the
1x1 / 3x3 convolutions of res2..res5, the strided 3x3 and 1x1/2 downsample
convolutions).  Through the planned op (qconv.qconv2d: implicit GEMM where the
channel run allows, im2col otherwise):

* INT8 forward bit-exact against the oracle (oracle/cpu_ref.c): per-tensor int8
  input, im2col, per-channel int8 weights, int32 GEMM, dequant + bias epilogue;
* the INT8 op's FP16 backward against float64 autograd of the same operands
  (dgrad: FP16(dY) with FP16(W); wgrad: FP16(dY) with the saved int8 input times
  s_x): 1e-5 / 1e-4 of the norm (FP32 accumulation over up to 100k pixels);
* the FP16 op forward against float64 on the FP16 operands (1e-3, FP16 output)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2407_02327_b200.qconv import qconv2d
from paper_2407_02327_b200.qlinear import FP16, INT8

pytestmark = pytest.mark.gpu
BATCH = 8


def resnet50_geometries(batch=BATCH):
    """Distinct (N, H, W, C, Cout, R, stride, pad) of ResNet-50's convolutions at 224^2."""
    convs = [(batch, 224, 224, 3, 64, 7, 2, 3)]
    h, cin = 56, 64
    for width, blocks, stride in [(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)]:
        for b in range(blocks):
            s = stride if b == 0 else 1
            ho = h // s
            convs.append((batch, h, h, cin, width, 1, 1, 0))
            convs.append((batch, h, h, width, width, 3, s, 1))
            convs.append((batch, ho, ho, width, 4 * width, 1, 1, 0))
            if b == 0:
                convs.append((batch, h, h, cin, 4 * width, 1, s, 0))
            cin, h = 4 * width, ho
    out = []
    for c in convs:
        if c not in out:
            out.append(c)
    return out


GEOMS = resnet50_geometries()


def _nrel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))


def _ids(g):
    N, H, W, C, Co, R, s, p = g
    return f"{H}x{W}_{C}to{Co}_k{R}s{s}"


def test_geometry_count():
    assert len(GEOMS) >= 20 and GEOMS[0][3] == 3  # the stem and every distinct body conv


@pytest.mark.parametrize("geom", GEOMS, ids=[_ids(g) for g in GEOMS])
def test_rn50_int8_conv_vs_oracle(geom, cpuref):
    N, H, W, C, Co, R, s, p = geom
    rng = np.random.default_rng(sum(geom))
    x = rng.normal(size=(N, H, W, C)).astype(np.float32)
    w = (rng.uniform(-1, 1, size=(Co, R, R, C)) / np.sqrt(R * R * C)).astype(np.float32)
    b = (rng.normal(size=Co) * 0.1).astype(np.float32)
    xt = torch.from_numpy(x).cuda().requires_grad_(C != 3)
    wt = torch.from_numpy(w).cuda().requires_grad_(True)
    bt = torch.from_numpy(b).cuda()
    y = qconv2d(xt, wt, bt, (s, s), (p, p), INT8)
    # ---- forward: bit-exact against the oracle's quantize + im2col + int32 GEMM + epilogue
    xq, sx = cpuref.quantize_per_tensor(x.reshape(1, -1))
    xq = xq.reshape(x.shape)
    K = R * R * C
    kp = (K + 15) // 16 * 16
    A, (P, Q) = cpuref.im2col(xq, R, R, (s, s), (p, p), ld=kp)
    w2 = np.zeros((Co, kp), np.float32)
    w2[:, :K] = w.reshape(Co, K)
    wq, sw = cpuref.quantize_per_channel(w2)
    y_ref = cpuref.dequant_epilogue(cpuref.gemm_s8_tn(A, wq), sx, sw, b).reshape(N, P, Q, Co)
    assert y.shape == (N, P, Q, Co) and y.dtype == torch.float32
    assert np.array_equal(y.detach().cpu().numpy(), y_ref)
    # ---- backward (FP16): float64 autograd of the same FP16 operands
    g = torch.from_numpy(rng.normal(size=(N, P, Q, Co)).astype(np.float32)).cuda()
    y.backward(g)
    g16 = g.half().double().permute(0, 3, 1, 2)
    xin = (torch.from_numpy(xq).cuda().double() * float(sx)).permute(0, 3, 1, 2).requires_grad_(True)
    w16 = wt.detach().half().double().permute(0, 3, 1, 2).requires_grad_(True)
    F.conv2d(xin, w16, None, s, p).backward(g16)
    assert _nrel(wt.grad.permute(0, 3, 1, 2), w16.grad) < (1e-5 if N * P * Q <= 4096 else 1e-4)
    if C != 3:
        assert _nrel(xt.grad.permute(0, 3, 1, 2), xin.grad) < 1e-5


@pytest.mark.parametrize("geom", GEOMS, ids=[_ids(g) for g in GEOMS])
def test_rn50_fp16_conv_forward_vs_f64(geom):
    N, H, W, C, Co, R, s, p = geom
    torch.manual_seed(sum(geom))
    x = torch.randn(N, H, W, C, device="cuda").half()
    w = (torch.rand(Co, R, R, C, device="cuda") * 2 - 1).div_((R * R * C) ** 0.5)
    b = torch.randn(Co, device="cuda") * 0.1
    y = qconv2d(x, w, b, (s, s), (p, p), FP16)
    ref = F.conv2d(x.double().permute(0, 3, 1, 2), w.half().double().permute(0, 3, 1, 2), b.double(), s, p)
    assert y.dtype == torch.float16
    assert _nrel(y.permute(0, 3, 1, 2), ref) < 1e-3
