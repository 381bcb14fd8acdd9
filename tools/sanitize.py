"""One small launch of every kernel family with tricky synchronisation, for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py [group ...]

groups: gemm1 (1-CTA tcgen05 GEMM, INT8 + FP16, TMA store and reduce-add),
gemm2 (CTA-pair cta_group::2), conv_tma / conv_gather (implicit conv, both
operand loaders, fwd / dgrad / wgrad), attn1 / attn2 (tcgen05 attention, 1 and
2 CTAs/SM backward), sr (mt19937_64 jump-ahead + SR), pdl (PDL zeroing kernel +
atomic-max producer + quantizer chain), quant (streaming quantizers); round 2:
dual (two MMA issuers per CTA), streamk (stream-K fixup through the workspace +
arrival counters), gelu1 (FF1 GEMM with max(h) + the one-pass GELU quantizer,
shortcut and grid-barrier fallback), attnq (attention + quantizer behind a grid
barrier), head (classification head + the vector zero kernel), ln (LayerNorm
backward with bulk-copied row stages, plain and embedding scatter).
Shapes are small: the sanitizers replay every access.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import _lib, ops  # noqa: E402


def gemm(cta):
    ops.force_cta(cta)
    try:
        M, N, K = 512, 512, 256
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        sa = torch.tensor([0.01], device="cuda")
        sb = torch.rand(N, device="cuda") * 0.01
        ops.gemm_s8(a, b, sa, sb, torch.randn(N, device="cuda"))
        ah, bh = torch.randn(M, K, device="cuda").half(), torch.randn(N, K, device="cuda").half()
        ops.gemm_f16(ah, bh, out_dtype=torch.float16)
        if cta == 1:
            acc = torch.zeros(M, N, device="cuda")
            ops.gemm_f16(ah.t().contiguous(), bh.t().contiguous(), out=acc, accumulate=True, a_mn=True, b_mn=True)
    finally:
        ops.force_cta(0)


def conv(tma):
    ops.conv_set_impl(tma)
    try:
        N, H, C, Co = 2, 8, 128, 128
        x = torch.randn(N, H, H, C, device="cuda").half()
        w = (torch.randn(Co, 3, 3, C, device="cuda") * 0.03).half()
        ops.conv_fwd_implicit(x, w.view(Co, -1), 3, 3, (1, 1), (1, 1), out_dtype=torch.float16)
        dy = torch.randn(N, H, H, Co, device="cuda").half()
        ops.conv_dgrad_implicit(dy, w, (N, H, H, C), (1, 1), (1, 1))
        ops.conv_wgrad_implicit(x, dy.view(-1, Co), 3, 3, (1, 1), (1, 1))
        xq = torch.randint(-127, 128, (N, H, H, C), dtype=torch.int8, device="cuda")
        wq = torch.randint(-127, 128, (Co, 9 * C), dtype=torch.int8, device="cuda")
        ops.conv_fwd_implicit(xq, wq, 3, 3, (1, 1), (1, 1), torch.tensor([0.01], device="cuda"),
                              torch.rand(Co, device="cuda") * 0.01)
    finally:
        ops.conv_set_impl(1)


def attn(impl):
    _lib.call("qsync_attention_set_impl", impl)
    try:
        qkv = torch.randn(2, 128, 3, 2, 64, device="cuda").half()
        out, lse, _ = ops.attention_fwd(qkv, want_absmax=True)
        ops.attention_bwd(qkv, out, torch.randn_like(out), lse)
    finally:
        _lib.call("qsync_attention_set_impl", 2)


def sr():
    x = torch.rand(1 << 16, device="cuda")
    ops.quantize_sr(x, torch.tensor([0.01], device="cuda"), 7)
    ops.stochastic_round(x.double(), 0.01, 0.0, 3)


def pdl():
    x = torch.randn(4096, 768, device="cuda")
    am = ops.absmax_act(x)
    ops.quantize_act(x, am)
    ops.quantize_per_tensor(x)


def quant():
    x = torch.randn(1 << 16, device="cuda")
    ops.quantize_per_channel(x.view(64, -1))
    ops.cast(x, torch.float16)
    ops.tensor_stats(x)
    q, s, _ = ops.quantize_per_tensor(x.view(1, -1))
    ops.dequantize_per_tensor(q.view(-1), s[:1])


def dual():
    ops.set_dual_issue(True)
    M, N, K = 512, 384, 512  # 4 x 2 tiles of 128 x 192 <= SMs: one unit per CTA
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
    ops.gemm_s8_ex(a, b, torch.tensor([0.01], device="cuda"), torch.rand(N, device="cuda") * 0.01)
    ah, bh = torch.randn(M, K, device="cuda").half(), torch.randn(K, N, device="cuda").half()
    ops.gemm_f16(ah, bh, b_mn=True)


def streamk():
    ops.set_streamk(1)
    try:
        M, N, K = 384, 512, 1024
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        ops.gemm_s8_ex(a, b, torch.tensor([0.01], device="cuda"), torch.rand(N, device="cuda") * 0.01)
        acc = torch.zeros(M, N, device="cuda")
        ah, bh = torch.randn(K, M, device="cuda").half(), torch.randn(K, N, device="cuda").half()
        ops.gemm_f16(ah, bh, out=acc, accumulate=True, a_mn=True, b_mn=True)
    finally:
        ops.set_streamk(-1)


def gelu1():
    M, N, K = 256, 512, 256
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
    sb = torch.rand(N, device="cuda") * 0.01
    for shift in (0.0, -50.0):  # shortcut, then the grid-barrier fallback
        h, ym = ops.gemm_s8_ymax(a, b, torch.tensor([0.01], device="cuda"), sb,
                                 torch.full((N,), shift, device="cuda"))
        ops.gelu_quantize(h, ym)


def attnq():
    qkv = torch.randn(2, 128, 3, 2, 64, device="cuda").half()
    ops.attention_fwd_quant(qkv)


def head():
    x = torch.randn(4, 16, 256, device="cuda")
    wp, bp = torch.randn(256, 256, device="cuda") * 0.05, torch.zeros(256, device="cuda")
    wc, bc = torch.randn(3, 256, device="cuda") * 0.05, torch.zeros(3, device="cuda")
    labels = torch.randint(0, 3, (4,), device="cuda")
    loss, pooled, probs = ops.cls_head_fwd(x, wp, bp, wc, bc, labels)
    grads = [torch.zeros_like(t) for t in (wp, bp, wc, bc)]
    ops.cls_head_bwd(x, wp, wc, labels, pooled, probs, torch.ones(1, device="cuda"), *grads)
    ops.zero_(torch.randn(1001, device="cuda")[1:])


def ln():
    T, H, V = 300, 768, 50  # rows not a multiple of the 4 rows per block
    a, b = torch.randn(T, H, device="cuda"), torch.randn(T, H, device="cuda")
    g, be = torch.rand(H, device="cuda") + 0.5, torch.randn(H, device="cuda")
    y, s, m, r = ops.layernorm_fwd(a, b, g, be, 1e-12)
    dg, db, col = (torch.zeros(H, device="cuda") for _ in range(3))
    ops.layernorm_bwd_ex(torch.randn(T, H, device="cuda"), s, m, r, g, dg, db, True, col)
    tok = torch.randint(0, V, (3, T // 3), device="cuda")
    word, pos, typ = torch.randn(V, H, device="cuda"), torch.randn(T // 3, H, device="cuda"), torch.randn(2, H, device="cuda")
    y, s, m, r = ops.embed_layernorm_fwd(tok, word, pos, typ, g, be, 1e-12)[:4]
    ops.embed_layernorm_bwd(torch.randn(T, H, device="cuda"), s, m, r, g, tok, dg, db, torch.zeros_like(word),
                            torch.zeros_like(pos), torch.zeros(H, device="cuda"))


GROUPS = {"gemm1": lambda: gemm(1), "gemm2": lambda: gemm(2), "conv_tma": lambda: conv(1),
          "conv_gather": lambda: conv(0), "attn1": lambda: attn(1), "attn2": lambda: attn(2), "sr": sr,
          "pdl": pdl, "quant": quant, "dual": dual, "streamk": streamk, "gelu1": gelu1, "attnq": attnq,
          "head": head, "ln": ln}


def main():
    names = sys.argv[1:] or list(GROUPS)
    for n in names:
        GROUPS[n]()
        torch.cuda.synchronize()
        print(f"ran {n}", flush=True)


if __name__ == "__main__":
    main()
