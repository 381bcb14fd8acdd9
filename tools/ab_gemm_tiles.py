"""Tile-shape A/B of the INT8 / FP16 GEMMs at the BERT step shapes (CUDA-graph timed)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import ops  # noqa: E402
from tools.gemm_overhead import graph_time_us  # noqa: E402

T, H, F = 4096, 768, 3072
for nm, (M, N, K) in {"qkv": (T, 3 * H, H), "o": (T, H, H), "ff1": (T, F, H), "ff2": (T, H, F)}.items():
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
    sa = torch.tensor([0.01], device="cuda")
    sb = torch.rand(N, device="cuda")
    bias = torch.randn(N, device="cuda")
    out = torch.empty(M, N, device="cuda", dtype=torch.float16 if nm == "qkv" else torch.float32)
    res = []
    for cta in (1, 2):
        for bn in (0, 64, 128, 256):
            if cta == 2 and bn == 64:
                continue
            ops.force_cta(cta)
            ops.force_tile_n(bn)
            res.append((f"cta{cta}/bn{bn or 'auto'}", graph_time_us(
                lambda: ops.gemm_s8_ex(a, b, sa, sb, bias, out_dtype=out.dtype, out=out))))
    ops.force_cta(0)
    ops.force_tile_n(0)
    auto = graph_time_us(lambda: ops.gemm_s8_ex(a, b, sa, sb, bias, out_dtype=out.dtype, out=out))
    print(f"s8 {nm:4s} auto {auto:6.1f}  " + "  ".join(f"{k} {v:6.1f}" for k, v in res), flush=True)
