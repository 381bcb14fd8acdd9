"""GPU tests of the attention core (csrc/attn.cu) against an FP32 PyTorch
reference of softmax(Q K^T scale) V and its autograd backward.  Tolerances
(FP16 in/out, FP32 softmax): out and dQKV within 1e-2 of each tensor's max,
lse within 1e-3 absolute; absmax(out) exact."""
import pytest
import torch

from paper_2407_02327_b200 import ops

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _ref(qkv, dout, scale):
    q, k, v = (qkv[:, :, i].float().transpose(1, 2).detach().requires_grad_(True) for i in range(3))
    s = q @ k.transpose(-1, -2) * scale
    lse = torch.logsumexp(s, dim=-1)
    o = torch.softmax(s, dim=-1) @ v
    o.backward(dout.float().transpose(1, 2))
    dqkv = torch.stack([q.grad, k.grad, v.grad], dim=2).transpose(1, 3)  # [B, S, 3, H, D]
    return o.transpose(1, 2), lse, dqkv


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max()).item()


@pytest.fixture(params=[2, 1, 0], ids=["tc_2cta", "tc", "mma_sync"])
def attn_impl(request):
    """tcgen05 at 2 CTAs/SM (P^T in TMEM, the default), tcgen05 at 1 CTA/SM, mma.sync."""
    from paper_2407_02327_b200._lib import call
    call("qsync_attention_set_impl", request.param)
    yield request.param
    call("qsync_attention_set_impl", 2)


@pytest.mark.parametrize("B,H,amp", [(4, 12, 1.0), (2, 3, 4.0), (32, 12, 0.5)])
def test_attention_fwd_bwd_vs_fp32(B, H, amp, attn_impl):
    torch.manual_seed(B * 100 + H)
    S, D = 128, 64
    qkv = (torch.randn(B, S, 3, H, D, device=DEV) * amp).half()
    dout = torch.randn(B, S, H, D, device=DEV).half()
    scale = D ** -0.5
    out, lse, am = ops.attention_fwd(qkv, scale, want_absmax=True)
    o_ref, lse_ref, d_ref = _ref(qkv, dout, scale)
    assert _rel(out, o_ref) < 1e-2
    assert (lse - lse_ref).abs().max().item() < 1e-3
    assert am.item() == out.float().abs().max().item()
    dqkv = ops.attention_bwd(qkv, out, dout, lse, scale)
    for i, name in enumerate(("dq", "dk", "dv")):
        err = _rel(dqkv[:, :, i], d_ref[:, :, i])
        assert err < 2e-2, f"{name} rel err {err}"


def test_attention_rejects_unsupported_shapes():
    qkv = torch.zeros(1, 64, 3, 2, 64, device=DEV, dtype=torch.float16)
    with pytest.raises(Exception, match="seq 128"):
        ops.attention_fwd(qkv)


def test_attention_fwd_tcgen05_vs_mma_sync():
    """The tcgen05 forward (TMEM accumulators, TMA operands) and the mma.sync
    forward agree (same P rounding, different accumulation order)."""
    from paper_2407_02327_b200._lib import call
    torch.manual_seed(21)
    qkv = torch.randn(8, 128, 3, 12, 64, device=DEV).half()
    call("qsync_attention_set_impl", 1)
    o1, l1, a1 = ops.attention_fwd(qkv, want_absmax=True)
    call("qsync_attention_set_impl", 0)
    try:
        o0, l0, a0 = ops.attention_fwd(qkv, want_absmax=True)
    finally:
        call("qsync_attention_set_impl", 2)
    assert _rel(o1, o0) < 2e-3
    assert (l1 - l0).abs().max().item() < 1e-4
    assert a1.item() == o1.float().abs().max().item()


def test_attention_bwd_tmem_p_matches_smem_p():
    """The 2-CTA/SM backward (P^T kept in tensor memory, dV's A operand read from
    TMEM) equals the 1-CTA/SM one (P^T staged in shared memory): same FP16 P,
    same MMA shapes."""
    from paper_2407_02327_b200._lib import call
    torch.manual_seed(31)
    qkv = torch.randn(16, 128, 3, 12, 64, device=DEV).half()
    dout = torch.randn(16, 128, 12, 64, device=DEV).half()
    out, lse, _ = ops.attention_fwd(qkv)
    call("qsync_attention_set_impl", 1)
    try:
        d1 = ops.attention_bwd(qkv, out, dout, lse)
    finally:
        call("qsync_attention_set_impl", 2)
    d2 = ops.attention_bwd(qkv, out, dout, lse)
    assert _rel(d2, d1) < 1e-3


@pytest.mark.parametrize("B,H", [(32, 12), (2, 3), (600, 12)])
def test_attention_fwd_quant_bit_identical(B, H):
    """qsync_attention_fwd_quant (one kernel with a grid barrier when the blocks
    fit, B = 600 x 12 falls back) == attention_fwd + absmax + quantize_act."""
    from paper_2407_02327_b200 import ops
    torch.manual_seed(B)
    qkv = (torch.randn(B, 128, 3, H, 64, device="cuda") * 0.5).half()
    out, lse, q, s, q16 = ops.attention_fwd_quant(qkv)
    out0, lse0, am = ops.attention_fwd(qkv, want_absmax=True)
    q0, s0, h0 = ops.quantize_act(out0.view(B * 128, H * 64), am, want_q16=True)
    torch.cuda.synchronize()
    assert torch.equal(out, out0) and torch.equal(lse, lse0)
    assert torch.equal(q, q0) and torch.equal(s, s0) and torch.equal(q16, h0)
    out2, _, q2, s2, _ = ops.attention_fwd_quant(qkv)  # barrier slot reuse
    assert torch.equal(q2, q0) and torch.equal(s2, s0)
