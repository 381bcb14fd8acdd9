"""Attention core (BERT-base: batch 32, seq 128, 12 heads, d 64, FP16) fwd+bwd:
flash_attn 2 (packed QKV) vs torch SDPA backends, CUDA-graph timed."""
import os
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_overhead import graph_time_us  # noqa: E402

B, S, H, D = 32, 128, 12, 64
qkv = torch.randn(B, S, 3, H, D, device="cuda", dtype=torch.float16, requires_grad=True)
do = torch.randn(B, S, H, D, device="cuda", dtype=torch.float16)


def flash():
    from flash_attn import flash_attn_qkvpacked_func
    o = flash_attn_qkvpacked_func(qkv)
    o.backward(do)


def sdpa(backend):
    def f():
        q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
        with sdpa_kernel(backend):
            o = F.scaled_dot_product_attention(q, k, v)
        o.transpose(1, 2).backward(do)
    return f


def fwd_only(fn_kind):
    def f():
        with torch.no_grad():
            if fn_kind == "flash":
                from flash_attn import flash_attn_qkvpacked_func
                flash_attn_qkvpacked_func(qkv)
            else:
                q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
                with sdpa_kernel(fn_kind):
                    F.scaled_dot_product_attention(q, k, v)
    return f


from paper_2407_02327_b200 import ops  # noqa: E402


def ours():
    q = qkv.detach()
    out, lse, _ = ops.attention_fwd(q)
    ops.attention_bwd(q, out, do, lse)


def ours_fwd():
    ops.attention_fwd(qkv.detach())


for name, fn in [("qsync attn fwd+bwd", ours), ("qsync attn fwd", ours_fwd), ("flash_attn2 fwd+bwd", flash), ("sdpa cudnn fwd+bwd", sdpa(SDPBackend.CUDNN_ATTENTION)),
                 ("sdpa flash fwd+bwd", sdpa(SDPBackend.FLASH_ATTENTION)),
                 ("sdpa efficient fwd+bwd", sdpa(SDPBackend.EFFICIENT_ATTENTION)),
                 ("flash_attn2 fwd", fwd_only("flash")), ("sdpa cudnn fwd", fwd_only(SDPBackend.CUDNN_ATTENTION))]:
    try:
        t = graph_time_us(fn, n=10)
        print(f"{name:28s} {t:8.1f} us", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name:28s} failed: {str(e)[:120]}", flush=True)
    qkv.grad = None
