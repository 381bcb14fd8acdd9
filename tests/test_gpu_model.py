"""GPU tests of the composed path: quantized Linear fwd+bwd vs the oracle, the
main_grad accumulation path, and the BERT train step (graph == eager, loss
decreases, per-plan kernel selection)."""
import numpy as np
import pytest
import torch

from paper_2407_02327_b200 import ops
from paper_2407_02327_b200.qlinear import FP16, FP32, INT8, qlinear
from paper_2407_02327_b200.train_step import (BertConfig, BertEncoderStack, TrainStep,
                                              mixed_plan, uniform_plan)

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _case(M, N, K, seed):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(M, K)).astype(np.float32)
    w = (rng.uniform(-1, 1, size=(N, K)) / np.sqrt(K)).astype(np.float32)
    b = (rng.normal(size=N) * 0.1).astype(np.float32)
    dy = rng.normal(size=(M, N)).astype(np.float32)
    return x, w, b, dy


def _run(x, w, b, dy, precision, main_grad=False):
    xt = torch.from_numpy(x).to(DEV).requires_grad_(True)
    wt = torch.from_numpy(w).to(DEV).requires_grad_(True)
    bt = torch.from_numpy(b).to(DEV).requires_grad_(True)
    if main_grad:
        wt.main_grad = torch.full_like(wt, 0.5)
        bt.main_grad = torch.full_like(bt, 0.25)
    y = qlinear(xt, wt, bt, precision)
    y.backward(torch.from_numpy(dy).to(DEV).to(y.dtype))
    torch.cuda.synchronize()
    if main_grad:
        return y, xt.grad, wt.main_grad - 0.5, bt.main_grad - 0.25
    return y, xt.grad, wt.grad, bt.grad


def _rel(got, want):
    got = got.detach().float().cpu().numpy()
    return np.abs(got - want).max() / max(np.abs(want).max(), 1e-12)


@pytest.mark.parametrize("mnk", [(64, 1024, 1024), (4096, 768, 768), (300, 200, 144), (128, 2304, 768)])
@pytest.mark.parametrize("main_grad", [False, True])
def test_qlinear_int8_matches_oracle(mnk, main_grad, cpuref):
    x, w, b, dy = _case(*mnk, seed=sum(mnk))
    y, dx, dw, db = _run(x, w, b, dy, INT8, main_grad)
    o = cpuref.qlinear_int8(x, w, b, dy)
    assert np.array_equal(y.detach().cpu().numpy(), o["y"])  # bit-exact forward
    assert _rel(dx, o["dx"]) < 1e-2   # FP16 dgrad (tolerance 1e-2, north star)
    assert _rel(dw, o["dw"]) < 1e-3   # FP32-accumulated wgrad vs FP64 oracle
    assert _rel(db, o["db"]) < 1e-5


@pytest.mark.parametrize("mnk", [(64, 1024, 1024), (4096, 3072, 768), (200, 72, 64)])
def test_qlinear_fp16_matches_oracle(mnk, cpuref):
    x, w, b, dy = _case(*mnk, seed=7 + sum(mnk))
    y, dx, dw, db = _run(x, w, b, dy, FP16)
    o = cpuref.qlinear_f16(x, w, b, dy.astype(np.float16).astype(np.float32))
    assert y.dtype == torch.float16  # output_precision(FP16) = FP16
    assert _rel(y, o["y"]) < 1e-2
    assert _rel(dx, o["dx"]) < 1e-2
    assert _rel(dw, o["dw"]) < 1e-3
    assert _rel(db, o["db"]) < 1e-3


def test_qlinear_fp32_and_bad_precision():
    x, w, b, dy = _case(32, 48, 64, 3)
    y, dx, dw, db = _run(x, w, b, dy, FP32)
    assert y.dtype == torch.float32
    np.testing.assert_allclose(y.detach().cpu().numpy(), x @ w.T + b, rtol=1e-4, atol=1e-4)
    with pytest.raises(ValueError, match="unknown precision"):
        qlinear(torch.zeros(2, 4, device=DEV), torch.zeros(3, 4, device=DEV), None, "INT4")


def _tiny_cfg():
    return BertConfig(vocab=1000, hidden=256, layers=2, heads=4, ffn=1024, max_pos=128, seq=128)


def _batch(cfg, B, seed):
    g = torch.Generator().manual_seed(seed)
    return (torch.randint(0, cfg.vocab, (B, cfg.seq), generator=g),
            torch.randint(0, 2, (B,), generator=g))


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("plan_kind", ["mixed", "int8", "fp16"])
def test_train_step_graph_matches_eager_and_learns(plan_kind, fused):
    cfg = _tiny_cfg()
    plans = {"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8), "fp16": uniform_plan(cfg, FP16)}
    losses = {}
    for use_graph in (False, True):
        torch.manual_seed(0)
        m = BertEncoderStack(cfg).to(DEV)
        m.apply_plan(plans[plan_kind])
        st = TrainStep(m, batch=8, lr=3e-4, graph=use_graph, fused=fused)
        tok, lab = _batch(cfg, 8, 1)
        st.tokens.copy_(tok)
        st.labels.copy_(lab)
        st.capture(warmup=3)  # 3 eager warm-up steps (same in both modes)
        ls = [float(st().item()) for _ in range(12)]
        losses[use_graph] = ls
    # Same kernels, same order: graph replay reproduces eager exactly (up to
    # FP32 atomics in the bias-gradient column sums).
    np.testing.assert_allclose(losses[True], losses[False], rtol=2e-3, atol=2e-3)
    assert losses[True][-1] < losses[True][0]  # one fixed batch: the loss must fall


def test_plan_selects_kernels():
    cfg = _tiny_cfg()
    m = BertEncoderStack(cfg).to(DEV)
    m.apply_plan({"layer0.qkv": INT8, "layer1.ff2": FP16})
    ql = m.qlinears()
    assert ql["layer0.qkv"].precision == INT8
    assert ql["layer1.ff2"].precision == FP16
    assert ql["layer0.o"].precision == FP32  # omitted ops run FP32 (replayer.cpp:86-94)
    tok, lab = _batch(cfg, 2, 3)
    ops.GEMM_TIMER = []
    try:
        m(tok.to(DEV), lab.to(DEV)).backward()
        kinds = [k for k, *_ in ops.GEMM_TIMER]
    finally:
        ops.GEMM_TIMER = None
    assert kinds.count("gemm_s8") == 1          # one INT8 forward
    assert kinds.count("gemm_f16") == 2 + 1 + 2  # INT8 bwd (2) + FP16 fwd (1) + bwd (2)


@pytest.mark.parametrize("rows,cols,bdt", [(4096, 768, torch.float32), (333, 1024, torch.float16),
                                          (64, 128, None)])
def test_add_layernorm_vs_torch_fp32(rows, cols, bdt):
    from paper_2407_02327_b200.glue import AddLayerNorm
    torch.manual_seed(0)
    a = torch.randn(rows, cols, device=DEV, requires_grad=True)
    b = (torch.randn(rows, cols, device=DEV).to(bdt).requires_grad_(True) if bdt else None)
    ln = AddLayerNorm(cols, eps=1e-5).to(DEV)
    with torch.no_grad():
        ln.weight.uniform_(0.5, 1.5)
        ln.bias.uniform_(-0.5, 0.5)
    ref = torch.nn.LayerNorm(cols, eps=1e-5).to(DEV)
    ref.load_state_dict(ln.state_dict())
    a2 = a.detach().clone().requires_grad_(True)
    b2 = b.detach().clone().requires_grad_(True) if b is not None else None
    y = ln(a, b)
    y_ref = ref(a2 + (b2.float() if b2 is not None else 0))
    torch.testing.assert_close(y, y_ref, rtol=1e-4, atol=1e-4)
    g = torch.randn_like(y)
    y.backward(g)
    y_ref.backward(g)
    torch.testing.assert_close(a.grad, a2.grad, rtol=1e-4, atol=1e-4)
    if b is not None:
        torch.testing.assert_close(b.grad.float(), b2.grad.float(), rtol=1e-2, atol=1e-2)
    torch.testing.assert_close(ln.weight.grad, ref.weight.grad, rtol=1e-3, atol=1e-3)
    torch.testing.assert_close(ln.bias.grad, ref.bias.grad, rtol=1e-3, atol=1e-3)


@pytest.mark.parametrize("mnk", [(2304, 768, 4096), (768, 3072, 4096), (768, 768, 4096), (300, 200, 1000)])
def test_gemm_f16_splitk_accumulate(mnk):
    """wgrad shapes: accumulate into an FP32 buffer -> split-K + TMA reduce-add."""
    M, N, K = mnk
    torch.manual_seed(1)
    a = torch.randn(M, K, device=DEV).half()
    b = torch.randn(N, K, device=DEV).half()
    base = torch.randn(M, N, device=DEV)
    want = base.double() + 0.5 * (a.double() @ b.double().T)
    s = torch.tensor([0.25], device=DEV)
    ops.gemm_f16(a, b, alpha=2.0, alpha_dev=s, out=base, accumulate=True)
    err = (base.double() - want).abs().max().item()
    assert err <= 1e-3 * want.abs().max().item()
