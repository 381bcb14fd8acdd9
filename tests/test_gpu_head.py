"""The classification head kernels (csrc/head.cu: pooler tanh + classifier +
mean cross entropy, forward and backward) against the same head in FP32 torch
(float64 for the reference), and the library zero kernel."""
import pytest
import torch
import torch.nn.functional as F

from paper_2407_02327_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,S,H,C", [(32, 128, 768, 2), (3, 5, 100, 7), (64, 16, 1024, 3)])
def test_cls_head_fwd_bwd_vs_fp64(B, S, H, C):
    g = torch.Generator(device="cuda").manual_seed(B + H)
    x = torch.randn(B, S, H, device="cuda", generator=g)
    wp = torch.randn(H, H, device="cuda", generator=g) / H ** 0.5
    bp = torch.randn(H, device="cuda", generator=g) * 0.1
    wc = torch.randn(C, H, device="cuda", generator=g) / H ** 0.5
    bc = torch.randn(C, device="cuda", generator=g) * 0.1
    labels = torch.randint(0, C, (B,), device="cuda", generator=g)
    loss, pooled, probs = ops.cls_head_fwd(x, wp, bp, wc, bc, labels)
    dwp, dbp, dwc, dbc = (torch.full_like(t, 0.5) for t in (wp, bp, wc, bc))  # ADDED into
    dloss = torch.tensor([2.0], device="cuda")
    dx = ops.cls_head_bwd(x, wp, wc, labels, pooled, probs, dloss, dwp, dbp, dwc, dbc)
    torch.cuda.synchronize()
    ref = [t.double().requires_grad_(True) for t in (x, wp, bp, wc, bc)]
    pr = torch.tanh(ref[0][:, 0] @ ref[1].t() + ref[2])
    lr = F.cross_entropy(pr @ ref[3].t() + ref[4], labels)
    (lr * 2.0).backward()

    def close(a, b, tol, what):
        err = (a.double() - b).abs().max().item() / max(b.abs().max().item(), 1e-30)
        assert err < tol, f"{what}: rel err {err}"
    close(loss.reshape(()), lr.detach(), 1e-5, "loss")
    close(pooled, pr.detach(), 1e-5, "pooled")
    close(dx, ref[0].grad, 1e-4, "dx")
    assert torch.count_nonzero(dx[:, 1:]) == 0
    for got, r, nm in ((dwp, ref[1], "dwp"), (dbp, ref[2], "dbp"), (dwc, ref[3], "dwc"), (dbc, ref[4], "dbc")):
        close(got - 0.5, r.grad, 1e-4, nm)
    # deterministic: a second run gives the same bits
    loss2, _, _ = ops.cls_head_fwd(x, wp, bp, wc, bc, labels)
    assert torch.equal(loss, loss2)


@pytest.mark.parametrize("n,dtype", [(1 << 20, torch.float32), (1000003, torch.float32), (77, torch.float16)])
def test_zero(n, dtype):
    t = torch.randn(n, device="cuda").to(dtype)
    ops.zero_(t)
    assert torch.count_nonzero(t) == 0
    u = torch.randn(n + 1, device="cuda").to(dtype) + 3
    ops.zero_(u[1:])  # not 16-byte aligned: byte head + vector body + byte tail
    assert torch.count_nonzero(u[1:]) == 0 and u[0] != 0
