"""The BF16 rung of the ladder (qlinear.BF16) and the stale-copy guard of the
fused path on the B200:

* BF16 QLinear forward / backward against an FP64 torch reference of the same
  op (BF16 operands: 2^-8 relative per element, FP32 accumulation): outputs
  within 2e-2 of the output scale, bias gradient exact to FP32 sums;
* a TrainStep whose plan mixes fused layers (INT8 / FP16) with a per-operator
  BF16 layer trains (finite, decreasing loss on a fixed batch);
* the fused forward never runs on weight copies older than the weights
  (load_state_dict after the optimizer wrote the copies)."""
import pytest
import torch

from paper_2407_02327_b200.qlinear import BF16, FP16, INT8, output_dtype, qlinear

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("M,N,K", [(256, 768, 768), (64, 3072, 768), (100, 200, 64)])
def test_bf16_qlinear_fwd_bwd(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", generator=g).requires_grad_(True)
    w = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).div_(K ** 0.5).requires_grad_(True)
    b = torch.randn(N, device="cuda", generator=g).mul_(0.1).requires_grad_(True)
    y = qlinear(x, w, b, BF16)
    assert y.dtype == output_dtype(BF16) == torch.bfloat16
    dy = torch.randn(M, N, device="cuda", generator=g)
    y.backward(dy)
    x64, w64, b64 = (t.detach().double() for t in (x, w, b))
    xb, wb = x64.bfloat16().double(), w64.bfloat16().double()
    assert _rel(y.float(), xb @ wb.t() + b64) < 2e-2
    dyb = dy.double().bfloat16().double()
    assert x.grad.dtype == torch.float32 and _rel(x.grad, dyb @ wb) < 2e-2
    assert _rel(w.grad, dyb.t() @ xb) < 2e-2
    assert _rel(b.grad, dyb.sum(0)) < 1e-5


def test_mixed_fused_and_bf16_layers_train():
    from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, _fusable
    cfg = BertConfig(vocab=1000, hidden=256, layers=3, heads=4, ffn=1024, max_pos=128, seq=128)
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    plan = {}
    for i, p in enumerate((INT8, BF16, FP16)):
        for op in ("qkv", "o", "ff1", "ff2"):
            plan[f"layer{i}.{op}"] = p
    m.apply_plan(plan)
    assert [_fusable(layer) for layer in m.layers] == [True, False, True]
    st = TrainStep(m, batch=4, graph=False, lr=1e-3)
    st.tokens.copy_(torch.randint(0, cfg.vocab, (4, cfg.seq), generator=torch.Generator().manual_seed(1)))
    st.labels.copy_(torch.tensor([0, 1, 0, 1]))
    losses = [float(st().item()) for _ in range(8)]
    assert all(abs(v) < 10 for v in losses)
    assert losses[-1] < losses[0], losses


def test_fused_forward_refreshes_stale_weight_copies():
    from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, mixed_plan
    cfg = BertConfig(vocab=1000, hidden=256, layers=2, heads=4, ffn=1024, max_pos=128, seq=128)
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(mixed_plan(cfg))
    st = TrainStep(m, batch=4, graph=False, lr=1e-2)
    tok = torch.randint(0, cfg.vocab, (4, cfg.seq), generator=torch.Generator().manual_seed(2))
    st.tokens.copy_(tok)
    st.labels.copy_(torch.tensor([0, 1, 1, 0]))
    st()  # the optimizer moved the weights and wrote the copies
    torch.manual_seed(5)
    fresh = BertEncoderStack(cfg).cuda()
    m.load_state_dict(fresh.state_dict())  # weights change outside the optimizer
    fresh.apply_plan(mixed_plan(cfg))
    st2 = TrainStep(fresh, batch=4, graph=False, lr=1e-2)  # copies made from these weights
    st2.tokens.copy_(tok)
    st2.labels.copy_(st.labels)
    with torch.no_grad():
        la = float(m(st.tokens, st.labels))
        lb = float(fresh(st2.tokens, st2.labels))
    assert abs(la - lb) <= 1e-5 * abs(lb), (la, lb)
