"""Per-launch time of the tcgen05 GEMMs at the BERT-base step shapes, launched
back-to-back inside a CUDA graph (as in the train step), with the epilogue
math/stores on or skipped and programmatic dependent launch on or off, next to
cuBLAS / cuBLASLt on the same operands (torch.mm FP16 out; torch._int_mm int32
out with no epilogue, FP16 wgrad without the FP32 accumulate).  The
difference to the MMA-only bound is the fixed cost (prologue, pipeline fill,
exposed epilogue) the small GEMMs of the step pay.

    python tools/gemm_overhead.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import _lib, ops  # noqa: E402

T, H, F = 4096, 768, 3072
PEAK_F16 = 1.65e15  # measured burst bf16/fp16 dense (MEASURED_PEAKS.json)


def graph_time_us(fn, n=40, reps=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    return best


def cases():
    def f16(M, N, K, lay=0, acc=False, out16=True):
        a = torch.randn((K, M) if lay == 3 else (M, K), device="cuda").half()
        b = torch.randn((K, N) if lay & 2 else (N, K), device="cuda").half()
        out = torch.zeros(M, N, device="cuda", dtype=torch.float16 if out16 and not acc else torch.float32)
        am = a.t() if lay == 3 else a
        bm = b if lay & 2 else b.t()
        ref = (lambda: torch.mm(am, bm)) if not acc else (lambda: torch.mm(am, bm))
        return (lambda: ops.gemm_f16(a, b, out=out, accumulate=acc, a_mn=lay == 3, b_mn=bool(lay & 2))), 2.0 * M * N * K, ref

    def s8(M, N, K):
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        sa = torch.tensor([0.01], device="cuda")
        sb = torch.rand(N, device="cuda")
        bias = torch.randn(N, device="cuda")
        out = torch.empty(M, N, device="cuda")
        bt = b.t()
        return (lambda: ops.gemm_s8(a, b, sa, sb, bias, out=out)), 2.0 * M * N * K, (lambda: torch._int_mm(a, bt))

    yield "big  f16 8192^3", *f16(8192, 8192, 8192, out16=False)
    yield "big  s8  8192^3", *s8(8192, 8192, 8192)
    yield "tiny f16 128x256x64", *f16(128, 256, 64)
    yield "tiny f16 128x256x768", *f16(128, 256, 768)
    for nm, (M, N, K) in {"qkv": (T, H, 3 * H), "ff1": (T, H, F)}.items():
        yield f"dgac f16 {nm}", *f16(M, N, K, lay=2, acc=True)
    for nm, (M, N, K) in {"qkv": (T, 3 * H, H), "o": (T, H, H), "ff1": (T, F, H), "ff2": (T, H, F)}.items():
        yield f"fwd  f16 {nm}", *f16(M, N, K)
        yield f"fwd  s8  {nm}", *s8(M, N, K)
        yield f"dgrd f16 {nm}", *f16(M, K, N, lay=2, out16=False)
        yield f"wgrd f16 {nm}", *f16(N, K, M, lay=3, acc=True)


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--bn", type=int, default=0, help="force the tile width (0 = cost model)")
    ap.add_argument("--only", default="", help="substring filter on the case name")
    ap.add_argument("--streamk", type=int, default=-1, help="-1 never (default), 0 cost model, 1 always")
    args = ap.parse_args()
    ops.set_streamk(args.streamk)
    _lib.call("qsync_gemm_force_tile_n", args.bn)
    print(f"{'case':22s} {'GFLOP':>7s} {'ideal':>7s} {'us':>7s} {'noepi':>7s} {'nopdl':>7s} {'cublas':>7s}  TF/s  (bn={args.bn})")
    for name, fn, flops, ref in cases():
        if args.only and args.only not in name:
            continue
        t = graph_time_us(fn)
        _lib.call("qsync_gemm_debug_epilogue", 1)
        t_ne = graph_time_us(fn)
        _lib.call("qsync_gemm_debug_epilogue", 0)
        _lib.call("qsync_gemm_set_pdl", 0)
        t_np = graph_time_us(fn)
        _lib.call("qsync_gemm_set_pdl", 1)
        t_ref = graph_time_us(ref)
        ideal = flops / PEAK_F16 * 1e6 / (2 if "s8" in name else 1)
        print(f"{name:22s} {flops / 1e9:7.2f} {ideal:7.1f} {t:7.1f} {t_ne:7.1f} {t_np:7.1f} {t_ref:7.1f}  {flops / t / 1e6:6.0f}",
              flush=True)


if __name__ == "__main__":
    main()
