"""FF1 with the GELU in the GEMM epilogue (qsync_gemm_gelu) against the unfused
pair it replaces in the fused layer: the plain INT8 / FP16 GEMM followed by the
FF2 operand kernel (gelu_absmax_store for an INT8 FF2, act_cast for FP16 / FP32).
Bit-exact: g, GELU'(h) (FP16) and absmax(g)."""
import pytest
import torch

from paper_2407_02327_b200 import ops

pytestmark = pytest.mark.gpu

SHAPES = [(4096, 3072, 768), (333, 136, 160), (128, 256, 64)]


def _operands(M, N, K, i8, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(M, K, device="cuda", generator=g)
    w = torch.randn(N, K, device="cuda", generator=g) / K ** 0.5
    bias = torch.randn(N, device="cuda", generator=g) * 0.1
    if i8:
        xq, xs, _ = ops.quantize_per_tensor(x)
        wq, ws, _ = ops.quantize_per_channel(w)
        return (xq, wq, xs[:1], ws), bias
    return (x.half(), w.half(), None, None), bias


def _unfused(opnd, bias, i8, g_dtype):
    a, b, sa, sb = opnd
    if i8:
        h = ops.gemm_s8_ex(a, b, sa, sb, bias, out_dtype=torch.float32)
    else:
        h = ops.gemm_f16(a, b, out_dtype=torch.float16, bias=bias)
    if g_dtype == h.dtype:  # what an INT8 FF2's operand kernel does
        am, g, d = ops.gelu_absmax_store(h)
        return am, g, d
    g, d = ops.act_cast(h, g_dtype, ops.ACT_GELU, want_dact=True)
    am = g.float().abs().max().reshape(1)
    return am, g, d


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("i8", [True, False])
@pytest.mark.parametrize("g_dtype", [torch.float32, torch.float16])
def test_gemm_gelu_bit_exact(shape, i8, g_dtype):
    M, N, K = shape
    opnd, bias = _operands(M, N, K, i8)
    a, b, sa, sb = opnd
    am, g, d = ops.gemm_gelu(a, b, sa, sb, bias, g_dtype=g_dtype)
    am_r, g_r, d_r = _unfused(opnd, bias, i8, g_dtype)
    torch.cuda.synchronize()
    assert g.dtype == g_dtype and d.dtype == torch.float16
    assert torch.equal(g.view(torch.int32 if g_dtype == torch.float32 else torch.int16),
                       g_r.view(torch.int32 if g_dtype == torch.float32 else torch.int16)), "g differs"
    assert torch.equal(d.view(torch.int16), d_r.view(torch.int16)), "GELU' differs"
    assert torch.equal(am, am_r.to(am.dtype)), f"absmax {am.item()} vs {am_r.item()}"


def test_gemm_gelu_no_bias_and_overwrites_absmax():
    opnd, _ = _operands(256, 512, 256, True, seed=3)
    a, b, sa, sb = opnd
    am1, g1, _ = ops.gemm_gelu(a, b, sa, sb, None)
    am2, g2, _ = ops.gemm_gelu(a, b, sa, sb, None)
    am_r, g_r, _ = _unfused(opnd, None, True, torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(g1, g_r) and torch.equal(g2, g_r)
    assert am1.item() == am2.item() == am_r.item()


def test_gemm_gelu_rejects_bad_n():
    a = torch.zeros(128, 64, device="cuda", dtype=torch.float16)
    b = torch.zeros(100, 64, device="cuda", dtype=torch.float16)
    with pytest.raises(Exception):
        ops.gemm_gelu(a, b)


@pytest.mark.parametrize("plan_kind", ["int8", "fp16", "mixed"])
def test_fused_stack_with_gelu_epilogue(plan_kind):
    """The fused encoder stack with FF1's GELU in the GEMM epilogue
    (fused.FF1_GELU_EPILOGUE) against the default operand-kernel path: the
    forward is bit-identical (same loss bits), gradients agree to atomics-order
    noise."""
    from paper_2407_02327_b200 import fused
    from paper_2407_02327_b200.qlinear import FP16, INT8
    from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, FlatGrads, mixed_plan, uniform_plan
    cfg = BertConfig(vocab=1000, hidden=256, layers=3, heads=4, ffn=1024, max_pos=128, seq=128)
    plans = {"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8), "fp16": uniform_plan(cfg, FP16)}
    g = torch.Generator().manual_seed(9)
    tok = torch.randint(0, cfg.vocab, (4, cfg.seq), generator=g).cuda()
    lab = torch.randint(0, 2, (4,), generator=g).cuda()
    res = {}
    old = fused.FF1_GELU_EPILOGUE
    try:
        for on in (False, True):
            fused.FF1_GELU_EPILOGUE = on
            torch.manual_seed(0)
            m = BertEncoderStack(cfg).cuda()
            m.apply_plan(plans[plan_kind])
            m.fused = True
            fg = FlatGrads(list(m.parameters()))
            fg.zero()
            loss = m(tok, lab)
            loss.backward()
            torch.cuda.synchronize()
            res[on] = (loss.detach().clone(), {n: p.main_grad.clone() for n, p in m.named_parameters()})
    finally:
        fused.FF1_GELU_EPILOGUE = old
    assert torch.equal(res[True][0], res[False][0])
    for n, g0 in res[False][1].items():
        g1 = res[True][1][n]
        if g0.abs().max().item() == 0:
            continue
        assert ((g1 - g0).norm() / g0.norm()).item() < 1e-3, n


def test_gelu_fp32_shortcut_preconditions():
    """k_gelu_quant's shortcut (absmax(gelu(h)) = gelu(max h)) rests on two
    properties of this library's float32 gelu, checked over EVERY float32 in
    [-16, 16]: non-decreasing wherever it exceeds 0.1701, and |gelu(h)| < 0.1701
    for h < 0."""
    viol, negmax = ops.gelu_fp32_check()
    assert viol == 0, f"{viol} monotonicity violations above 0.1701"
    assert 0.16 < negmax < 0.1701, negmax


@pytest.mark.parametrize("M,N,K", [(4096, 3072, 768), (333, 200, 160)])
@pytest.mark.parametrize("shift", [0.0, -6.0])
def test_gemm_ymax_then_gelu_quantize_bit_exact(M, N, K, shift):
    """qsync_gemm_s8_ymax + qsync_gelu_quantize == gemm_s8_ex + gelu_absmax_store +
    quantize_act (q, s, FP16(q), GELU').  shift -6 makes every h small, so the
    kernel takes its exact absmax fallback (grid barrier)."""
    opnd, bias = _operands(M, N, K, True, seed=5)
    a, b, sa, sb = opnd
    bias = bias + shift
    h, ym = ops.gemm_s8_ymax(a, b, sa, sb, bias)
    q, s, d, q16 = ops.gelu_quantize(h, ym)
    h0 = ops.gemm_s8_ex(a, b, sa, sb, bias, out_dtype=torch.float32)
    am, g0, d0 = ops.gelu_absmax_store(h0)
    q0, s0, h16 = ops.quantize_act(g0, am, want_q16=True)
    torch.cuda.synchronize()
    assert torch.equal(h, h0)
    assert ym.item() == max(0.0, h0.max().item())
    assert torch.equal(s, s0) and torch.equal(q, q0) and torch.equal(q16, h16)
    assert torch.equal(d.view(torch.int16), d0.view(torch.int16))
