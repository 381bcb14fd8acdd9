"""Isolated timing of the layer-fused path's streaming kernels at the BERT-base
step shapes (tokens 4096, hidden 768, ffn 3072), each launched back-to-back in a
CUDA graph, with achieved GB/s over the algorithmic bytes (compulsory reads +
writes) against the measured HBM peak.

    python tools/glue_bench.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import ops  # noqa: E402
from tools.gemm_overhead import graph_time_us  # noqa: E402

T, H, F = 4096, 768, 3072


def peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))["hbm_gbs"]
    except Exception:
        return 6650.0


def cases():
    d = "cuda"
    a = torch.randn(T, H, device=d)
    b = torch.randn(T, H, device=d)
    g = torch.rand(H, device=d) + 0.5
    be = torch.randn(H, device=d)
    y, s, m, r = ops.layernorm_fwd(a, b, g, be, 1e-12)
    dg, db, col = torch.zeros(H, device=d), torch.zeros(H, device=d), torch.zeros(H, device=d)
    yield "ln_fwd_ex (+y16)", lambda: ops.layernorm_fwd_ex(a, b, g, be, 1e-12, True, False), T * H * (4 + 4 + 4 + 4 + 2)
    yield "ln_fwd_ex (+absmax)", lambda: ops.layernorm_fwd_ex(a, b, g, be, 1e-12, False, True), T * H * 16
    yield "ln_bwd_ex (+dx16,colsum)", lambda: ops.layernorm_bwd_ex(a, s, m, r, g, dg, db, True, col), T * H * (4 + 4 + 4 + 2)
    h32 = torch.randn(T, F, device=d)
    h16 = h32.half()
    dg32 = torch.randn(T, F, device=d)
    dg16 = dg32.half()
    colF = torch.zeros(F, device=d)
    yield "act_bwd f32,f32->f16", lambda: ops.act_bwd_colsum(dg32, h32, ops.ACT_GELU, torch.float16, colF), T * F * 10
    yield "act_bwd f16,f16->f16", lambda: ops.act_bwd_colsum(dg16, h16, ops.ACT_GELU, torch.float16, colF), T * F * 6
    # as in the step: FP16 dG x the stored FP16 GELU'(h) -> FP16 dH + bias sums
    yield "act_bwd deriv f16 (step)", lambda: ops.act_bwd_colsum(dg16, h16, ops.ACT_DERIV, torch.float16, colF), T * F * 6
    q16 = torch.randn(T, 3 * H, device=d).half()
    col3 = torch.zeros(3 * H, device=d)
    yield "colsum f16 (qkv bias)", lambda: ops.act_bwd_colsum(q16, None, ops.ACT_NONE, None, col3), T * 3 * H * 2
    am = ops.absmax_act(h32, ops.ACT_GELU)
    yield "absmax gelu f32", lambda: ops.absmax_act(h32, ops.ACT_GELU, out=am), T * F * 4
    yield "quantize gelu f32", lambda: ops.quantize_act(h32, am, ops.ACT_GELU), T * F * 5
    # FF2's INT8 operand as the step builds it: the old two-erf form vs one erf + stored GELU
    yield "ff2 int8 operand: absmax+quantize gelu (2 erf)", lambda: ops.quantize_act(
        h32, ops.absmax_act(h32, ops.ACT_GELU), ops.ACT_GELU, want_dact=True, want_q16=True), T * F * (4 + 4 + 1 + 2 + 2)

    def one_erf():
        am2, g, _ = ops.gelu_absmax_store(h32)
        ops.quantize_act(g, am2, want_q16=True)
    yield "ff2 int8 operand: gelu_absmax_store+quantize (1 erf)", one_erf, T * F * (4 + 4 + 1 + 2 + 2)
    yield "absmax gelu f16", lambda: ops.absmax_act(h16, ops.ACT_GELU, out=am), T * F * 2
    yield "gelu cast f16->f16", lambda: ops.act_cast(h16, torch.float16, ops.ACT_GELU), T * F * 4
    yield "absmax f32 (act)", lambda: ops.absmax(a), T * H * 4
    yield "quantize_act f32", lambda: ops.quantize_act(a, am), T * H * 5
    xq = torch.randint(-127, 128, (T, F), dtype=torch.int8, device=d)
    yield "cast i8->f16", lambda: ops.cast(xq, torch.float16), T * F * 3
    a16 = torch.randn(T, H, device=d).half()
    yield "quantize_per_tensor f16", lambda: ops.quantize_per_tensor(a16), T * H * 3
    # optimizer over a BERT-base parameter set (110 M params)
    from paper_2407_02327_b200.fused import FusedAdamW
    from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, FlatGrads, mixed_plan
    cfg = BertConfig()
    mdl = BertEncoderStack(cfg).to(d)
    mdl.apply_plan(mixed_plan(cfg))
    params = list(mdl.parameters())
    FlatGrads(params)
    opt = FusedAdamW(params)
    opt.attach(mdl.qlinears().values())
    n = sum(p.numel() for p in params)
    prep = sum(m.weight.numel() * (3 if m.wq is not None else 2) for m in mdl.qlinears().values() if m.w16 is not None)
    yield "adamw + weight prep (BERT-base)", opt.step, n * 28 + prep


def main():
    pk = peak()
    print(f"{'kernel':34s} {'MB':>8s} {'us':>8s} {'GB/s':>8s} {'frac':>6s}")
    for name, fn, nbytes in cases():
        t = graph_time_us(fn, n=20)
        print(f"{name:34s} {nbytes / 1e6:8.1f} {t:8.1f} {nbytes / t / 1e3:8.0f} {nbytes / t / 1e3 / pk:6.2f}", flush=True)


if __name__ == "__main__":
    main()
