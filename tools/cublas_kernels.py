"""Which cuBLAS / cuBLASLt kernels (tile shape, cluster shape) run at the
BERT-base step GEMM shapes, and their device time (CUPTI via torch.profiler).
A reference point for the tile / cluster choice of csrc/gemm.cu.

    python tools/cublas_kernels.py
"""
import torch
from torch.profiler import ProfilerActivity, profile

T, H, F = 4096, 768, 3072


def cases():
    for nm, (M, N, K) in {"qkv": (T, 3 * H, H), "o": (T, H, H), "ff1": (T, F, H), "ff2": (T, H, F)}.items():
        a = torch.randn(M, K, device="cuda").half()
        w = torch.randn(N, K, device="cuda").half()
        dy = torch.randn(M, N, device="cuda").half()
        yield f"fwd f16 {nm}", lambda a=a, w=w: torch.mm(a, w.t())
        yield f"dgrad f16 {nm}", lambda dy=dy, w=w: torch.mm(dy, w)
        yield f"wgrad f16 {nm}", lambda dy=dy, a=a: torch.mm(dy.t(), a)
        a8 = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        w8 = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        yield f"fwd s8 {nm}", lambda a8=a8, w8=w8: torch._int_mm(a8, w8.t())
    a = torch.randn(8192, 8192, device="cuda").half()
    yield "f16 8192^3", lambda: torch.mm(a, a)


def main():
    for name, fn in cases():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(10):
                fn()
            torch.cuda.synchronize()
        ks = {}
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                k = ks.setdefault(e.name, [0, 0.0])
                k[0] += 1
                k[1] += e.device_time
        for k, (n, t) in ks.items():
            print(f"{name:16s} {t / n:8.1f} us  x{n // 10}  {k}", flush=True)


if __name__ == "__main__":
    main()
