"""Per-shape timing of the BERT-base backward GEMMs (dgrad / wgrad) across tile
N and split-K choices.  Launches are queued behind a device spin so the CUDA
events bracket kernels only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import ops  # noqa: E402

T = 4096
H, F = 768, 3072
SHAPES = {  # name: (M, N, K, accumulate)
    "dgrad_qkv": (T, H, 3 * H, False), "dgrad_o": (T, H, H, False),
    "dgrad_ff1": (T, H, F, False), "dgrad_ff2": (T, F, H, False),
    "wgrad_qkv": (3 * H, H, T, True), "wgrad_o": (H, H, T, True),
    "wgrad_ff1": (F, H, T, True), "wgrad_ff2": (H, F, T, True),
    "fwd_qkv": (T, 3 * H, H, False), "fwd_ff1": (T, F, H, False), "fwd_ff2": (T, H, F, False),
}


def timeit(fn, iters=20):
    fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def main():
    for name, (M, N, K, acc) in SHAPES.items():
        a = torch.randn(M, K, device="cuda").half()
        b = torch.randn(N, K, device="cuda").half()
        out = torch.zeros(M, N, device="cuda")
        flops = 2.0 * M * N * K
        res = []
        for cta in (1, 2):
            for bn in (0, 64, 128, 256):
                if cta == 2 and bn == 64:
                    continue
                for ks in ((1, 0, 2, 4) if acc else (1,)):
                    ops.force_tile_n(bn)
                    ops.force_splitk(ks)
                    ops.force_cta(cta)
                    try:
                        us = timeit(lambda: ops.gemm_f16(a, b, out=out, accumulate=acc))
                    finally:
                        ops.force_tile_n(0)
                        ops.force_splitk(0)
                        ops.force_cta(0)
                    res.append((us, f"c{cta}b{bn}", ks))
        auto = timeit(lambda: ops.gemm_f16(a, b, out=out, accumulate=acc))
        ref = timeit(lambda: torch.matmul(a, b.t()))
        res.sort()
        best = res[0]
        print(f"{name:10s} {M:5d}x{N:5d}x{K:5d} acc={int(acc)} cublas {ref:6.1f}us auto {auto:6.1f}us | "
              + " ".join(f"{bn}/ks{ks}:{us:.1f}" for us, bn, ks in res[:5])
              + f" | best {flops/best[0]/1e6:.0f} TF")
        a8 = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b8 = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        if name.startswith("fwd"):
            sa = torch.tensor([0.01], device="cuda")
            sb = torch.rand(N, device="cuda")
            r8 = []
            for cta in (1, 2):
                for bn in (64, 128, 256):
                    if cta == 2 and bn == 64:
                        continue
                    ops.force_tile_n(bn)
                    ops.force_cta(cta)
                    try:
                        r8.append((timeit(lambda: ops.gemm_s8(a8, b8, sa, sb, out=out)), f"c{cta}b{bn}"))
                    finally:
                        ops.force_tile_n(0)
                        ops.force_cta(0)
            r8.sort()
            ref8 = timeit(lambda: torch._int_mm(a8, b8.t()))
            auto8 = timeit(lambda: ops.gemm_s8(a8, b8, sa, sb, out=out))
            print(f"   int8   cublasLt {ref8:6.1f}us auto {auto8:6.1f}us | " + " ".join(f"{bn}:{us:.1f}" for us, bn in r8))


if __name__ == "__main__":
    main()
