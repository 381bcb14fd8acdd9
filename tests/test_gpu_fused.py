"""GPU tests of the layer-fused path (fused.py): each fused kernel against the
unfused kernels it replaces (bit-exact where the arithmetic is the same) or an
FP64/FP32 torch reference, the fused optimizer against torch.optim.AdamW, and
the fused encoder stack against the per-operator path on identical weights."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2407_02327_b200 import ops
from paper_2407_02327_b200.fused import FusedAdamW
from paper_2407_02327_b200.qlinear import FP16, FP32, INT8
from paper_2407_02327_b200.train_step import (BertConfig, BertEncoderStack, FlatGrads, TrainStep,
                                              mixed_plan, uniform_plan)

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("rows,cols,bdt", [(4096, 768, torch.float32), (333, 1024, torch.float16),
                                          (64, 128, None)])
def test_layernorm_fwd_ex_outputs(rows, cols, bdt):
    torch.manual_seed(0)
    a = torch.randn(rows, cols, device=DEV)
    b = torch.randn(rows, cols, device=DEV).to(bdt) if bdt else None
    g = torch.rand(cols, device=DEV) + 0.5
    be = torch.randn(cols, device=DEV)
    y0, s0, m0, r0 = ops.layernorm_fwd(a, b, g, be, 1e-12)
    y, s, m, r, y16, am = ops.layernorm_fwd_ex(a, b, g, be, 1e-12, want_f16=True, want_absmax=True)
    assert torch.equal(y, y0) and torch.equal(m, m0) and torch.equal(r, r0)
    assert torch.equal(y16, y.half())                  # FP16 operand of an FP16 op
    assert am.item() == y.abs().max().item()           # absmax for an INT8 op: exact


@pytest.mark.parametrize("rows,cols", [(4096, 768), (200, 256)])
def test_layernorm_bwd_ex_outputs(rows, cols):
    torch.manual_seed(1)
    a = torch.randn(rows, cols, device=DEV)
    g = torch.rand(cols, device=DEV) + 0.5
    be = torch.randn(cols, device=DEV)
    y, s, m, r = ops.layernorm_fwd(a, None, g, be, 1e-12)
    dy = torch.randn(rows, cols, device=DEV)
    dg0, db0 = torch.zeros(cols, device=DEV), torch.zeros(cols, device=DEV)
    dx0 = ops.layernorm_bwd(dy, s, m, r, g, dg0, db0)
    dg, db = torch.zeros(cols, device=DEV), torch.zeros(cols, device=DEV)
    col = torch.full((cols,), 0.5, device=DEV)
    dx, dx16 = ops.layernorm_bwd_ex(dy, s, m, r, g, dg, db, want_f16=True, colsum_into=col)
    assert torch.equal(dx, dx0)
    assert torch.equal(dx16, dx.half())
    want = dx.double().sum(0) + 0.5
    assert ((col.double() - want).abs().max() / want.abs().max()).item() < 1e-5
    # dgamma / dbeta: per-block partials combined by FP32 atomics (order varies)
    for got, ref in ((dg, dg0), (db, db0)):
        assert ((got - ref).abs().max() / ref.abs().max()).item() < 1e-4


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16])
@pytest.mark.parametrize("n", [4096 * 3072, 1000003])
def test_gelu_quantize_matches_unfused(dtype, n):
    """absmax(gelu(h)) / quantize(gelu(h)) with GELU in the prologue == the same
    kernels run on the materialised gelu(h) (bit-exact), and gelu ~ torch."""
    torch.manual_seed(2)
    h = (torch.randn(n, device=DEV) * 2).to(dtype)
    g = ops.act_cast(h, torch.float32, ops.ACT_GELU)
    # an FP16 producer's GELU runs (and rounds) in FP16, as torch's F.gelu(h16)
    tol = 2e-6 if dtype == torch.float32 else 1e-3
    torch.testing.assert_close(g, F.gelu(h).float(), rtol=tol, atol=tol / 10)
    am = ops.absmax_act(h, ops.ACT_GELU)
    assert am.item() == g.abs().max().item()
    q, s = ops.quantize_act(h, am, ops.ACT_GELU)
    q0, sc0, _ = ops.quantize_per_tensor(g.view(1, -1))
    assert torch.equal(q.view(-1), q0.view(-1))
    assert s.item() == sc0[0].item()
    g16 = ops.act_cast(h, torch.float16, ops.ACT_GELU)
    assert torch.equal(g16, g.half())


@pytest.mark.parametrize("rows,cols", [(4096, 3072), (4096, 768), (300, 200), (77, 1000)])
@pytest.mark.parametrize("dyt,ht", [(torch.float32, torch.float32), (torch.float16, torch.float16)])
def test_act_bwd_colsum_vs_fp64(rows, cols, dyt, ht):
    torch.manual_seed(3)
    dy = torch.randn(rows, cols, device=DEV).to(dyt)
    h = (torch.randn(rows, cols, device=DEV) * 2).to(ht)
    hd = h.double()
    grad = 0.5 * (1 + torch.erf(hd / 2 ** 0.5)) + hd * torch.exp(-0.5 * hd * hd) / (2 * np.pi) ** 0.5
    want = dy.double() * grad
    col = torch.zeros(cols, device=DEV)
    out = ops.act_bwd_colsum(dy, h, ops.ACT_GELU, torch.float16, colsum_into=col)
    assert ((out.double() - want).abs().max() / want.abs().max()).item() < 1e-3
    assert ((col.double() - want.sum(0)).abs().max() / want.sum(0).abs().max()).item() < 1e-4
    out32 = ops.act_bwd_colsum(dy, h, ops.ACT_GELU, torch.float32)
    assert ((out32.double() - want).abs().max() / want.abs().max()).item() < 1e-5
    # no activation: colsum only (the QKV bias gradient from the packed dQKV)
    col2 = torch.zeros(cols, device=DEV)
    assert ops.act_bwd_colsum(dy, None, ops.ACT_NONE, None, colsum_into=col2) is None
    w2 = dy.double().sum(0)
    assert ((col2.double() - w2).abs().max() / w2.abs().max()).item() < 1e-5


@pytest.mark.parametrize("mnk", [(4096, 2304, 768), (300, 200, 144)])
def test_gemm_s8_f16_epilogue_equals_cast(mnk):
    M, N, K = mnk
    torch.manual_seed(4)
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=DEV)
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=DEV)
    sa = torch.tensor([0.013], device=DEV)
    sb = torch.rand(N, device=DEV) * 0.01
    bias = torch.randn(N, device=DEV)
    _, y32 = ops.gemm_s8(a, b, sa, sb, bias)
    y16 = ops.gemm_s8_ex(a, b, sa, sb, bias, out_dtype=torch.float16)
    assert torch.equal(y16, y32.half())


def test_fused_adamw_matches_torch_and_prepares_weights():
    torch.manual_seed(5)
    shapes = [(2304, 768), (768,), (5, 3), (3072, 768), (7,)]
    ps = [torch.nn.Parameter(torch.randn(s, device=DEV) * 0.05) for s in shapes]
    ref = [torch.nn.Parameter(p.detach().clone()) for p in ps]
    for p in ps:
        p.main_grad = torch.zeros_like(p)
    opt = FusedAdamW(ps, lr=1e-3, weight_decay=0.01)

    class _M:  # a planned Linear's weight-copy holder
        def __init__(self, w, prec):
            self.weight, self.precision = w, prec

    mods = [_M(ps[0], INT8), _M(ps[3], FP16), _M(ps[2], INT8)]
    opt.attach(mods)
    topt = torch.optim.AdamW(ref, lr=1e-3, weight_decay=0.01)
    for it in range(4):
        for p, r in zip(ps, ref):
            g = torch.randn_like(p) * (0.1 + it)
            p.main_grad.copy_(g)
            r.grad = g.clone()
        opt.step()
        topt.step()
    for p, r in zip(ps, ref):
        torch.testing.assert_close(p.detach(), r.detach(), rtol=1e-5, atol=1e-6)
    # prepared copies == the standalone kernels on the updated weights, bit-exact
    wq, ws, _ = ops.quantize_per_channel(ps[0].detach())
    assert torch.equal(mods[0].wq, wq) and torch.equal(mods[0].ws, ws)
    assert torch.equal(mods[0].w16, ps[0].detach().half())
    assert torch.equal(mods[1].w16, ps[3].detach().half()) and mods[1].wq is None
    wq2, ws2, _ = ops.quantize_per_channel(ps[2].detach())
    assert torch.equal(mods[2].wq, wq2) and torch.equal(mods[2].ws, ws2)


def _tiny_cfg():
    return BertConfig(vocab=1000, hidden=256, layers=3, heads=4, ffn=1024, max_pos=128, seq=128)


def _random_plan(cfg, seed):
    rng = np.random.default_rng(seed)
    plan = {}
    for i in range(cfg.layers):
        for op in ("qkv", "o", "ff1", "ff2"):
            plan[f"layer{i}.{op}"] = [INT8, FP16, FP32][rng.integers(0, 3)]
    return plan


@pytest.mark.parametrize("plan_kind", ["mixed", "int8", "fp16", "fp32", "random0", "random1"])
def test_fused_stack_matches_per_operator_path(plan_kind):
    """Same weights, same batch: loss and every FP32 gradient of the fused stack
    agree with the per-operator path.  Tolerances: loss 1e-3; per gradient tensor
    ||g_fused - g_op|| / ||g_op|| < 1e-2 and max error < 5e-2 of its max (FP16
    backward; a GELU ulp difference can move an INT8 scale, i.e. re-round a whole
    quantized tensor, upstream)."""
    cfg = _tiny_cfg()
    plans = {"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8), "fp16": uniform_plan(cfg, FP16),
             "fp32": uniform_plan(cfg, FP32), "random0": _random_plan(cfg, 0), "random1": _random_plan(cfg, 1)}
    g = torch.Generator().manual_seed(9)
    tok = torch.randint(0, cfg.vocab, (4, cfg.seq), generator=g).to(DEV)
    lab = torch.randint(0, 2, (4,), generator=g).to(DEV)
    res = {}
    for fused in (False, True):
        torch.manual_seed(0)
        m = BertEncoderStack(cfg).to(DEV)
        m.apply_plan(plans[plan_kind])
        m.fused = fused
        fg = FlatGrads(list(m.parameters()))
        fg.zero()
        loss = m(tok, lab)
        loss.backward()
        torch.cuda.synchronize()
        res[fused] = (loss.item(), {n: p.main_grad.clone() for n, p in m.named_parameters()})
    assert abs(res[True][0] - res[False][0]) <= 1e-3 * max(1.0, abs(res[False][0]))
    for n, g0 in res[False][1].items():
        g1 = res[True][1][n]
        scale = g0.abs().max().item()
        if scale == 0:
            continue
        err = (g1 - g0).abs().max().item() / scale
        fro = ((g1 - g0).norm() / g0.norm()).item()
        assert fro < 1e-2 and err < 5e-2, f"{n}: rel err {fro} (max {err})"


def test_fused_trainstep_graph_learns():
    cfg = _tiny_cfg()
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).to(DEV)
    m.apply_plan(mixed_plan(cfg))
    st = TrainStep(m, batch=8, lr=3e-4, graph=True, fused=True)
    assert m.fused and isinstance(st.opt, FusedAdamW)
    g = torch.Generator().manual_seed(1)
    st.tokens.copy_(torch.randint(0, cfg.vocab, (8, cfg.seq), generator=g))
    st.labels.copy_(torch.randint(0, 2, (8,), generator=g))
    st.capture(warmup=3)
    ls = [float(st().item()) for _ in range(12)]
    assert ls[-1] < ls[0]
    assert int(st.opt.step_t.item()) == 3 + 12  # warm-up + replays (capture only records)


def test_embed_layernorm_vs_torch():
    """Gathered embedding sum + LN (fwd) and the scatter-add backward vs torch
    fp32 autograd of Embedding + LayerNorm."""
    from paper_2407_02327_b200.glue import embed_layernorm
    from paper_2407_02327_b200.glue import AddLayerNorm
    torch.manual_seed(11)
    V, P, H, B, S = 1000, 128, 768, 8, 128
    word, pos, typ = (torch.nn.Embedding(n, H).to(DEV) for n in (V, P, 2))
    ln = AddLayerNorm(H, eps=1e-12).to(DEV)
    with torch.no_grad():
        ln.weight.uniform_(0.5, 1.5)
        ln.bias.uniform_(-0.5, 0.5)
    tok = torch.randint(0, V, (B, S), device=DEV)
    tok[0, :10] = 7  # repeated ids: the scatter must accumulate
    y, am = embed_layernorm(tok, word, pos, typ, ln, want_absmax=True)
    ref_ln = torch.nn.LayerNorm(H, eps=1e-12).to(DEV)
    ref_ln.load_state_dict(ln.state_dict())
    params = [word.weight, pos.weight, typ.weight, ref_ln.weight, ref_ln.bias]
    x = word.weight[tok] + pos.weight[torch.arange(S, device=DEV)][None] + typ.weight[0][None, None]
    y_ref = ref_ln(x)
    torch.testing.assert_close(y, y_ref, rtol=1e-4, atol=1e-4)
    assert am.item() == y.abs().max().item()
    g = torch.randn_like(y_ref)
    y.backward(g)
    got = [word.weight.grad, pos.weight.grad, typ.weight.grad, ln.weight.grad, ln.bias.grad]
    for p in params:
        p.grad = None
    y_ref.backward(g)
    for name, a, b in zip(("word", "pos", "typ", "gamma", "beta"), got, [p.grad for p in params]):
        err = ((a - b).abs().max() / b.abs().max()).item()
        assert err < 1e-4, f"{name}: {err}"


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16])
def test_stored_gelu_derivative(dtype):
    """FF2's operand kernels also store GELU'(h) in FP16; the backward then
    multiplies by it (QSYNC_ACT_DERIV) -- matches the FP64 derivative to FP16
    rounding, and the fused backward equals dy * stored derivative exactly."""
    torch.manual_seed(12)
    T, F = 4096, 3072
    h = (torch.randn(T, F, device=DEV) * 2).to(dtype)
    hd = h.double()
    want = 0.5 * (1 + torch.erf(hd / 2 ** 0.5)) + hd * torch.exp(-0.5 * hd * hd) / (2 * np.pi) ** 0.5
    am = ops.absmax_act(h, ops.ACT_GELU)
    q, s, d = ops.quantize_act(h, am, ops.ACT_GELU, want_dact=True)
    q0, s0 = ops.quantize_act(h, am, ops.ACT_GELU)
    assert torch.equal(q, q0) and torch.equal(s, s0)        # the extra output changes nothing
    assert ((d.double() - want).abs().max() / want.abs().max()).item() < 1e-3
    g16, d2 = ops.act_cast(h, torch.float16, ops.ACT_GELU, want_dact=True)
    assert torch.equal(d2, d) and torch.equal(g16, ops.act_cast(h, torch.float16, ops.ACT_GELU))
    dy = torch.randn(T, F, device=DEV)
    col = torch.zeros(F, device=DEV)
    dh = ops.act_bwd_colsum(dy, d, ops.ACT_DERIV, torch.float16, colsum_into=col)
    assert torch.equal(dh, (dy * d.float()).half())
    ref = (dy.double() * d.double()).sum(0)
    assert ((col.double() - ref).abs().max() / ref.abs().max()).item() < 1e-4


def test_bucketwise_optimizer_matches_single_launch():
    """The bucket-wise AdamW (row ranges launched as gradient buckets become
    final, then one step advance) is bit-identical to one launch over all rows;
    in the train step the losses agree.  (Whole-model weights are not compared
    across runs: the bias-gradient FP32 atomics make gradients differ in the
    last bits, and Adam's first steps are sign-like on tiny gradients.)"""
    torch.manual_seed(7)
    shapes = [(2304, 768), (768,), (5, 3), (3072, 768), (7,), (768, 3072)]
    runs = []
    for mode in ("single", "ranges"):
        torch.manual_seed(7)
        ps = [torch.nn.Parameter(torch.randn(s, device=DEV) * 0.05) for s in shapes]
        for p in ps:
            p.main_grad = torch.randn_like(p) * 0.1
        opt = FusedAdamW(ps, lr=1e-3)
        for _ in range(3):
            if mode == "single":
                opt.step()
            else:
                for grp in ([ps[5], ps[4]], [ps[3]], [ps[0], ps[1], ps[2]]):
                    opt.step_range(*opt.rows_of(grp))
                opt.advance()
        runs.append([p.detach().clone() for p in ps] + [opt.step_t.clone()])
    for a, b in zip(*runs):
        assert torch.equal(a, b)
    cfg = _tiny_cfg()
    losses = {}
    for overlap in (False, True):
        torch.manual_seed(0)
        m = BertEncoderStack(cfg).to(DEV)
        m.apply_plan(mixed_plan(cfg))
        st = TrainStep(m, batch=4, lr=1e-3, graph=False, fused=True)
        st.overlap_opt = overlap
        g = torch.Generator().manual_seed(5)
        st.tokens.copy_(torch.randint(0, cfg.vocab, (4, cfg.seq), generator=g))
        st.labels.copy_(torch.randint(0, 2, (4,), generator=g))
        losses[overlap] = [float(st().item()) for _ in range(3)]
        assert int(st.opt.step_t.item()) == 3
    np.testing.assert_allclose(losses[True], losses[False], rtol=2e-3, atol=2e-3)


@pytest.mark.parametrize("act", [0, 1])
@pytest.mark.parametrize("n", [4096 * 768, 1001])
def test_quantize_act_q16_is_exact_copy(act, n):
    """The quantizer's FP16 copy of the grid values (the wgrad operand) equals
    FP16(q) exactly, and writing it changes nothing else."""
    torch.manual_seed(n + act)
    h = torch.randn(n, device="cuda") * 3
    am = ops.absmax_act(h, act)
    q0, s0 = ops.quantize_act(h, am, act)
    q, s, q16 = ops.quantize_act(h, am, act, want_q16=True)
    assert torch.equal(q, q0) and torch.equal(s, s0)
    assert q16.dtype == torch.float16 and torch.equal(q16, q.to(torch.float16))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16])
@pytest.mark.parametrize("n", [4096 * 3072, 1000003])
def test_gelu_absmax_store_then_quantize_is_bit_identical(dtype, n):
    """FF2's INT8 operand via gelu_absmax_store + a plain quantize equals the
    GELU-prologue absmax + quantize (q, s, FP16 q copy and GELU' all bit-identical)."""
    torch.manual_seed(n % 97)
    h = (torch.randn(n, device=DEV) * 2).to(dtype)
    am0 = ops.absmax_act(h, ops.ACT_GELU)
    q0, s0, d0, h0 = ops.quantize_act(h, am0, ops.ACT_GELU, want_dact=True, want_q16=True)
    am, g, d = ops.gelu_absmax_store(h)
    q, s, h16 = ops.quantize_act(g, am, want_q16=True)
    assert am.item() == am0.item()
    assert torch.equal(g, ops.act_cast(h, dtype, ops.ACT_GELU))
    assert torch.equal(q, q0) and torch.equal(s, s0) and torch.equal(h16, h0) and torch.equal(d, d0)


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,bdt", [(4096, 768, torch.float32), (4096, 768, torch.float16),
                                           (1000, 256, torch.float32), (9000, 768, torch.float32)])
def test_layernorm_fwd_quant_matches_two_pass(rows, cols, bdt):
    """LayerNorm fused with its INT8 quantizer (grid barrier on absmax; the
    9000-row case exceeds one row per resident warp and takes the two-launch
    fallback) is bit-identical to layernorm_fwd_ex(absmax) + quantize_act(q16)."""
    torch.manual_seed(3)
    a = torch.randn(rows, cols, device=DEV)
    b = torch.randn(rows, cols, device=DEV).to(bdt)
    g, be = torch.rand(cols, device=DEV) + 0.5, torch.randn(cols, device=DEV)
    y, s, m, r, q, sc, q16 = ops.layernorm_fwd_quant(a, b, g, be, 1e-12)
    y2, s2, m2, r2, _, am = ops.layernorm_fwd_ex(a, b, g, be, 1e-12, False, True)
    q2, sc2, q16b = ops.quantize_act(y2, am, want_q16=True)
    for x, z in ((y, y2), (s, s2), (m, m2), (r, r2), (q, q2), (q16, q16b)):
        assert torch.equal(x, z)
    assert torch.equal(sc[:1], sc2) and sc[1].item() == am.item()
    for _ in range(3):  # the barrier slot resets itself: repeated launches agree
        assert torch.equal(ops.layernorm_fwd_quant(a, b, g, be, 1e-12)[4], q)


@pytest.mark.gpu
def test_embed_layernorm_quant_matches_two_pass():
    from paper_2407_02327_b200.glue import AddLayerNorm, embed_layernorm
    torch.manual_seed(12)
    V, P, H, B, S = 1000, 128, 768, 32, 128
    word, pos, typ = (torch.nn.Embedding(n, H).to(DEV) for n in (V, P, 2))
    ln = AddLayerNorm(H, eps=1e-12).to(DEV)
    tok = torch.randint(0, V, (B, S), device=DEV)
    y, am = embed_layernorm(tok, word, pos, typ, ln, want_absmax=True)
    y2, op = embed_layernorm(tok, word, pos, typ, ln, want_quant=True)
    assert torch.equal(y, y2)
    q, s, q16 = ops.quantize_act(y.detach().reshape(-1, H), am, want_q16=True)
    assert op[0] == "i8" and torch.equal(op[1], q) and torch.equal(op[2], s) and torch.equal(op[3], q16)
