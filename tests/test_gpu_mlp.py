"""BASELINE config 1: 2-layer MLP, batch 64, hidden 1024, per-channel INT8 with FP32
master weights -- forward + backward through the composed device path vs the
oracle composition (forward bit-exact, backward within tolerance)."""
import numpy as np
import pytest
import torch

from paper_2407_02327_b200.qlinear import INT8, QLinear

pytestmark = pytest.mark.gpu


def test_two_layer_mlp_int8_vs_oracle(cpuref):
    B, H = 64, 1024
    torch.manual_seed(0)
    l1 = QLinear(H, H, "fc1", precision=INT8).cuda()
    l2 = QLinear(H, H, "fc2", precision=INT8).cuda()
    rng = np.random.default_rng(11)
    x = rng.normal(size=(B, H)).astype(np.float32)
    g = rng.normal(size=(B, H)).astype(np.float32)
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    y1 = l1(xt)
    h = torch.relu(y1)
    y2 = l2(h)
    y2.backward(torch.from_numpy(g).cuda())
    torch.cuda.synchronize()

    w1, b1 = l1.weight.detach().cpu().numpy(), l1.bias.detach().cpu().numpy()
    w2, b2 = l2.weight.detach().cpu().numpy(), l2.bias.detach().cpu().numpy()
    o1 = cpuref.qlinear_int8(x, w1, b1, None)
    h_ref = np.maximum(o1["y"], 0.0)
    o2 = cpuref.qlinear_int8(h_ref, w2, b2, g)
    dy1 = o2["dx"] * (o1["y"] > 0)
    o1b = cpuref.qlinear_int8(x, w1, b1, dy1)

    # forward: quantized tensors, int32 GEMMs and dequant epilogues are bit-exact
    assert np.array_equal(y1.detach().cpu().numpy(), o1["y"])
    assert np.array_equal(y2.detach().cpu().numpy(), o2["y"])

    def rel(a, b):
        return np.abs(a - b).max() / max(np.abs(b).max(), 1e-12)

    assert rel(l2.weight.grad.cpu().numpy(), o2["dw"]) < 1e-3
    assert rel(l2.bias.grad.cpu().numpy(), o2["db"]) < 1e-5
    assert rel(l1.weight.grad.cpu().numpy(), o1b["dw"]) < 1e-2   # through the FP16 dgrad chain
    assert rel(l1.bias.grad.cpu().numpy(), o1b["db"]) < 1e-2
    assert rel(xt.grad.cpu().numpy(), o1b["dx"]) < 1e-2
