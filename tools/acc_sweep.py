"""Tile width x split-K sweep of the ACCUMULATING FP32 GEMMs of the BERT-base
step (dgrad reduce-added into the residual gradient, wgrad into main_grad),
graph-timed back to back, next to the cost model's own choice (choose_acc).

    python tools/acc_sweep.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import ops  # noqa: E402
from tools.gemm_overhead import graph_time_us  # noqa: E402

T, H, F = 4096, 768, 3072
SHAPES = {  # name: (M, N, K, a_mn, b_mn)
    "dgrad_qkv": (T, H, 3 * H, False, True), "dgrad_ff1": (T, H, F, False, True),
    "wgrad_qkv": (3 * H, H, T, True, True), "wgrad_o": (H, H, T, True, True),
    "wgrad_ff1": (F, H, T, True, True), "wgrad_ff2": (H, F, T, True, True),
}


def main():
    for name, (M, N, K, amn, bmn) in SHAPES.items():
        a = torch.randn((K, M) if amn else (M, K), device="cuda").half()
        b = torch.randn((K, N) if bmn else (N, K), device="cuda").half()
        out = torch.zeros(M, N, device="cuda")
        fn = lambda: ops.gemm_f16(a, b, out=out, accumulate=True, a_mn=amn, b_mn=bmn)  # noqa: E731
        ops.set_streamk(-1)
        res = {"model": graph_time_us(fn)}
        ops.set_streamk(1)
        res["streamk"] = graph_time_us(fn)
        ops.set_streamk(0)
        res["model+sk"] = graph_time_us(fn)
        ops.set_streamk(-1)
        for bn in (128, 192, 256):
            for ks in (1, 2, 3, 4, 6):
                ops.force_tile_n(bn)
                ops.force_splitk(ks)
                res[f"{bn}/{ks}"] = graph_time_us(fn)
        ops.force_tile_n(0)
        ops.force_splitk(0)
        ops.set_streamk(-1)
        best = min(res, key=res.get)
        print(f"{name:10s} tiles {res['model']:6.1f} sk {res['streamk']:6.1f} model+sk {res['model+sk']:6.1f} us"
              f" | best {best} {res[best]:6.1f} | " +
              " ".join(f"{k}:{v:.1f}" for k, v in res.items() if "/" in k), flush=True)


if __name__ == "__main__":
    main()
