"""Run one hot kernel a few times for ncu (`ncu -k regex:... python tools/prof_targets.py <name>`).

Targets use the bench's shapes: BERT-base FF1 forward (4096x3072x768 INT8 with the
fused dequant epilogue), the INT8 GEMM at 8192^3, the FP16 dgrad shape, and the
1 GiB quantize / cast / stats sweep points.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import ops  # noqa: E402


def main(name: str, reps: int = 3) -> None:
    dev = "cuda"
    T, H, F = 4096, 768, 3072
    bert = {"qkv": (T, 3 * H, H), "o": (T, H, H), "ff1": (T, F, H), "ff2": (T, H, F), "8192": (8192, 8192, 8192)}
    if name.startswith("gemm_s8"):
        M, N, K = bert[name.split("_")[-1]]
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev)
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
        sa = torch.tensor([0.01], device=dev)
        sb = torch.rand(N, device=dev) * 0.01
        bias = torch.randn(N, device=dev)
        out = torch.empty((M, N), device=dev)
        fn = lambda: ops.gemm_s8(a, b, sa, sb, bias, out=out)  # noqa: E731
    elif name.startswith("gemm_f16"):
        M, N, K = {"gemm_f16_8192": (8192, 8192, 8192), "gemm_f16_ff1": (4096, 3072, 768)}.get(
            name, (4096, 768, 3072))
        a = torch.randn((M, K), device=dev).half()
        b = torch.randn((N, K), device=dev).half()
        out = torch.empty((M, N), device=dev, dtype=torch.float16 if name.endswith("ff1") else torch.float32)
        fn = lambda: ops.gemm_f16(a, b, out=out)  # noqa: E731
    elif name in ("attn_fwd", "attn_bwd"):
        qkv = torch.randn(32, 128, 3, 12, 64, device=dev).half()
        dout = torch.randn(32, 128, 12, 64, device=dev).half()
        out, lse, _ = ops.attention_fwd(qkv)
        fn = (lambda: ops.attention_fwd(qkv)) if name == "attn_fwd" else (  # noqa: E731
            lambda: ops.attention_bwd(qkv, out, dout, lse))
    elif name == "ln_bwd":
        a = torch.randn(T, H, device=dev)
        g, be = torch.rand(H, device=dev) + 0.5, torch.randn(H, device=dev)
        y, s_, m, r = ops.layernorm_fwd(a, a, g, be, 1e-12)
        dg, db, col = (torch.zeros(H, device=dev) for _ in range(3))
        fn = lambda: ops.layernorm_bwd_ex(a, s_, m, r, g, dg, db, True, col)  # noqa: E731
    elif name == "act_bwd":  # as in the step: FP16 dG (FF2's dgrad) x stored FP16 GELU'(h)
        dg = torch.randn(T, F, device=dev).half()
        gp = torch.rand(T, F, device=dev).half()
        col = torch.zeros(F, device=dev)
        fn = lambda: ops.act_bwd_colsum(dg, gp, ops.ACT_DERIV, torch.float16, col)  # noqa: E731
    elif name in ("conv_fwd", "conv_wgrad", "conv_dgrad"):
        # ResNet-50 res3 3x3 (batch 64, 28x28, 128 -> 128), FP16 implicit GEMM (TMA im2col)
        N, Hc, C, Co = 64, 28, 128, 128
        x = torch.randn(N, Hc, Hc, C, device=dev).half()
        w = (torch.randn(Co, 3, 3, C, device=dev) * 0.03).half()
        dy = torch.randn(N, Hc, Hc, Co, device=dev).half()
        dw = torch.zeros(Co, 9 * C, device=dev)
        fn = {"conv_fwd": lambda: ops.conv_fwd_implicit(x, w.view(Co, -1), 3, 3, (1, 1), (1, 1),
                                                        out_dtype=torch.float16),
              "conv_wgrad": lambda: ops.conv_wgrad_implicit(x, dy.view(-1, Co), 3, 3, (1, 1), (1, 1), out=dw,
                                                            accumulate=True),
              "conv_dgrad": lambda: ops.conv_dgrad_implicit(dy, w, (N, Hc, Hc, C), (1, 1), (1, 1))}[name]
    elif name == "adamw":
        from paper_2407_02327_b200.fused import FusedAdamW
        from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, FlatGrads, mixed_plan
        cfg = BertConfig()
        mdl = BertEncoderStack(cfg).to(dev)
        mdl.apply_plan(mixed_plan(cfg))
        params = list(mdl.parameters())
        FlatGrads(params)
        opt = FusedAdamW(params)
        opt.attach(mdl.qlinears().values())
        fn = opt.step
    else:
        n = (1 << 30) // 4
        x = torch.randn(n, device=dev)
        x2 = x.view(-1, 1024)
        q = torch.empty(n, dtype=torch.int8, device=dev)
        sc = torch.tensor([0.01], device=dev)
        h = torch.empty(n, dtype=torch.float16, device=dev)
        fn = {
            "quantize_per_tensor": lambda: ops.quantize_per_tensor(x2, out=q.view(x2.shape)),
            "quantize_with_scale": lambda: ops.quantize_with_scale(x, sc),
            "quantize_f16": lambda: ops.quantize_with_scale(h, sc),
            "quantize_per_channel": lambda: ops.quantize_per_channel(x2),
            "dequantize": lambda: ops.dequantize_per_tensor(q, sc),
            "cast": lambda: ops.cast(x, torch.float16, out=h),
            "stats": lambda: ops.tensor_stats(x),
            "absmax": lambda: ops.absmax(x),
        }[name]
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
