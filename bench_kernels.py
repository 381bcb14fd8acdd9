"""Kernel microbenchmarks (config 5 sweep + GEMM roofline), CUDA-event timed.

    python bench_kernels.py [--sweep] [--gemm] [--json out.json]

Every kernel is launched through the C ABI on torch's current stream and timed
with CUDA events on that stream after warm-up.  Bandwidth kernels use inputs
>= 64 MB (larger than nothing in L2 between iterations: a 256 MB scratch write
flushes L2 between timed iterations for the smaller sizes).  Roofline
denominators come from MEASURED_PEAKS.json; the INT8 dense peak is measured here
with cuBLASLt (torch._int_mm) at 8192^3, best of 10.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
from paper_2407_02327_b200 import ops  # noqa: E402


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    _flush.zero_()


def time_ms(fn, iters=20, warmup=3, flush=False) -> float:
    """Mean device time of fn() over iters (flushing L2 before each if asked).
    The stream is held behind a ~100 us device spin while the host enqueues
    the start event, fn's launches and the end event, so the events bracket
    the kernels only -- not the host launch latency of the ctypes calls."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        if flush:
            flush_l2()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    times.sort()
    return sum(times[: max(1, len(times) * 3 // 4)]) / max(1, len(times) * 3 // 4)


def int8_peak_cublas(n=8192) -> float:
    a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda").t()
    best = 1e9
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def gemm_bench(results: dict) -> None:
    pk = peaks()
    i8_peak = int8_peak_cublas()
    results["int8_peak_cublaslt_tops"] = i8_peak
    rows = []
    shapes = [(8192, 8192, 8192), (4096, 2304, 768), (4096, 768, 768), (4096, 3072, 768),
              (4096, 768, 3072), (64, 1024, 1024)]
    for (M, N, K) in shapes:
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        sa = torch.tensor([0.01], device="cuda")
        sb = torch.rand(N, device="cuda") * 0.01
        out = torch.empty((M, N), device="cuda")
        for bn in (0, 128, 256):
            ops.force_tile_n(bn)
            t = time_ms(lambda: ops.gemm_s8(a, b, sa, sb, out=out))
            rows.append({"kind": "i8", "M": M, "N": N, "K": K, "bn": bn, "ms": t,
                         "tops": 2.0 * M * N * K / (t * 1e-3) / 1e12})
        ops.force_tile_n(0)
        # FP8 rung (E4M3, kind::f8f6f4) beside cuBLASLt FP8 (torch._scaled_mm)
        if K % 16 == 0 and M >= 128:
            a8, s8a = ops.quantize_fp8(torch.randn((M, K), device="cuda"))
            b8, s8b = ops.quantize_fp8_rows(torch.randn((N, K), device="cuda"))
            out8 = torch.empty((M, N), device="cuda")
            t = time_ms(lambda: ops.gemm_f8(a8, b8, s8a, s8b, out=out8))
            rows.append({"kind": "f8", "M": M, "N": N, "K": K, "bn": 0, "ms": t,
                         "tops": 2.0 * M * N * K / (t * 1e-3) / 1e12})
            try:
                one = torch.ones((), device="cuda")
                t = time_ms(lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one,
                                                     out_dtype=torch.float32))
                rows.append({"kind": "cublaslt_f8", "M": M, "N": N, "K": K, "ms": t,
                             "tops": 2.0 * M * N * K / (t * 1e-3) / 1e12})
            except Exception as e:  # noqa: BLE001
                print(f"cuBLASLt FP8 unavailable: {e}")
        ah = torch.randn((M, K), device="cuda").half()
        bh = torch.randn((N, K), device="cuda").half()
        outf = torch.empty((M, N), device="cuda")
        t = time_ms(lambda: ops.gemm_f16(ah, bh, out=outf))
        rows.append({"kind": "f16", "M": M, "N": N, "K": K, "bn": 0, "ms": t,
                     "tops": 2.0 * M * N * K / (t * 1e-3) / 1e12})
        t = time_ms(lambda: torch.matmul(ah, bh.t()))
        rows.append({"kind": "cublas_f16", "M": M, "N": N, "K": K, "ms": t,
                     "tops": 2.0 * M * N * K / (t * 1e-3) / 1e12})
        if M % 8 == 0 and K % 8 == 0 and N % 8 == 0 and M > 16:
            t = time_ms(lambda: torch._int_mm(a, b.t()))
            rows.append({"kind": "cublaslt_i8", "M": M, "N": N, "K": K, "ms": t,
                         "tops": 2.0 * M * N * K / (t * 1e-3) / 1e12})
    results["gemm"] = rows
    for r in rows:
        frac = r["tops"] / (i8_peak if ("i8" in r["kind"] or "f8" in r["kind"]) else pk["bf16_tflops"])
        print(f"{r['kind']:12s} {r['M']:5d}x{r['N']:5d}x{r['K']:5d} bn={r.get('bn', '-')!s:4s}"
              f" {r['ms']*1e3:9.1f} us {r['tops']:8.1f} TOPS  frac={frac:.3f}")
    print(f"int8 peak (cuBLASLt 8192^3 best of 10): {i8_peak:.1f} TOPS")


def graph_time_us(fn, n=10, reps=5):
    """Per-call device time of fn() captured n times into one CUDA graph."""
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
    torch.cuda.current_stream().wait_stream(st)
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


def spin_time_ms(fn, reps=5, spin_cycles=100_000_000):
    """Median device time of fn() with its launches queued behind a device spin."""
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(spin_cycles)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def resnet50_convs(batch: int = 64):
    """The 53 Conv2d layers of ResNet-50 at 224x224 (NHWC): (name, N, H, W, C, Cout, R, stride, pad)."""
    convs = [("conv1", batch, 224, 224, 3, 64, 7, 2, 3)]
    h, cin = 56, 64
    for stage, (width, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)]):
        for b in range(blocks):
            s = stride if b == 0 else 1
            hin = h
            ho = h // s
            convs.append((f"res{stage + 2}.{b}.a", batch, hin, hin, cin, width, 1, 1, 0))
            convs.append((f"res{stage + 2}.{b}.b", batch, hin, hin, width, width, 3, s, 1))
            convs.append((f"res{stage + 2}.{b}.c", batch, ho, ho, width, 4 * width, 1, 1, 0))
            if b == 0:
                convs.append((f"res{stage + 2}.{b}.ds", batch, hin, hin, cin, 4 * width, 1, s, 0))
            cin, h = 4 * width, ho
    return convs


def conv_bench(results: dict, batch: int = 64) -> None:
    """BASELINE configs[2]: the ResNet-50 convolutions as GEMMs (INT8 / FP16 plans),
    forward and forward+backward per distinct layer shape, summed over the 53 layers."""
    from paper_2407_02327_b200.qconv import qconv2d
    from paper_2407_02327_b200.qlinear import FP16, INT8
    convs = resnet50_convs(batch)
    if os.environ.get("QSB_CONV_BWD_COL"):  # A/B: materialised im2col / col2im backward
        ops.implicit_dgrad_ok = lambda *a: False
        ops.implicit_wgrad_ok = lambda *a: False
    distinct = {}
    for c in convs:
        distinct.setdefault(c[1:], []).append(c[0])
    rows = []
    totals = {INT8: [0.0, 0.0], FP16: [0.0, 0.0]}
    flops_fwd = 0.0
    for key, names in distinct.items():
        N, H, W, C, Cout, R, st, pd = key
        P = (H + 2 * pd - R) // st + 1
        fl = 2.0 * N * P * P * Cout * R * R * C
        flops_fwd += fl * len(names)
        x = torch.randn(N, H, W, C, device="cuda")
        w = (torch.randn(Cout, R, R, C, device="cuda") / (R * R * C) ** 0.5).requires_grad_(True)
        b = torch.zeros(Cout, device="cuda", requires_grad=True)
        for prec in (INT8, FP16):
            xin = x if prec == INT8 else x.half()
            # the stem's input is the image: no dgrad (as in training)
            xg = xin.detach().clone().requires_grad_(C != 3)
            wrt = [t for t in (xg, w, b) if t.requires_grad]
            # Device time with the launches queued behind a device spin, so the
            # host's launch overhead is excluded (as in the CUDA-graphed step).
            tf = spin_time_ms(lambda: qconv2d(xin, w, b, (st, st), (pd, pd), prec))
            y = qconv2d(xg, w, b, (st, st), (pd, pd), prec)
            gy = torch.randn_like(y)

            def fb():  # gradients returned, not accumulated into .grad
                yy = qconv2d(xg, w, b, (st, st), (pd, pd), prec)
                torch.autograd.grad(yy, wrt, gy)
            tfb = spin_time_ms(fb)
            totals[prec][0] += tf * len(names)
            totals[prec][1] += tfb * len(names)
            rows.append({"layers": names, "N": N, "H": H, "C": C, "Cout": Cout, "R": R, "stride": st,
                         "precision": prec, "fwd_ms": tf, "fwd_bwd_ms": tfb,
                         "fwd_tops": fl / (tf * 1e-3) / 1e12, "fwd_bwd_tops": 3 * fl / (tfb * 1e-3) / 1e12})
            print(f"{names[0]:10s} x{len(names)} {prec} C={C:4d}->{Cout:4d} R={R} s={st} H={H:3d}: "
                  f"fwd {tf*1e3:8.1f} us ({fl/(tf*1e-3)/1e12:6.1f} TOPS)  fwd+bwd {tfb*1e3:8.1f} us", flush=True)
        del x, w, b
        torch.cuda.empty_cache()
    results["resnet50_convs"] = {
        "batch": batch, "layers": len(convs), "fwd_gflop": flops_fwd / 1e9, "rows": rows,
        "stack": {p: {"fwd_ms": v[0], "fwd_bwd_ms": v[1], "fwd_tflops": flops_fwd / (v[0] * 1e-3) / 1e12,
                      "fwd_bwd_tflops": 3 * flops_fwd / (v[1] * 1e-3) / 1e12} for p, v in totals.items()}}
    for p, v in totals.items():
        print(f"ResNet-50 conv stack (53 layers, batch {batch}) {p}: fwd {v[0]:.2f} ms, fwd+bwd {v[1]:.2f} ms "
              f"({3 * flops_fwd / (v[1] * 1e-3) / 1e12:.0f} TFLOP/s)")


L2_BYTES = 126 << 20


def rotating_graph_us(make_call, nbytes_per_call: int, max_copies: int = 64, reps: int = 5):
    """Per-call device time of a streaming kernel, CUDA-graph timed (no launch
    gaps) with cold inputs: ``make_call(k)`` returns the k-th call over its own
    input/output copy; the graph cycles through enough copies that the bytes
    touched between two uses of one copy exceed 2x L2 (126 MB), so every call
    streams from HBM.  Returns (us per call, "cold" | "warm": warm when the copy
    cap leaves the working set L2-resident)."""
    copies = max(1, min(max_copies, -(-2 * L2_BYTES // max(1, nbytes_per_call))))
    calls = [make_call(k) for k in range(copies)]
    n = copies if copies >= 8 else max(8, copies)
    seq = [calls[i % copies] for i in range(n)]
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for c in calls:
            c()
    torch.cuda.current_stream().wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for c in seq:
            c()
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
    cold = copies * nbytes_per_call >= 2 * L2_BYTES
    del g
    return best, "cold" if cold else "warm"


def sweep_bench(results: dict, sizes=None) -> None:
    """Config 5: FP32 tensors of 2^16 .. 2^30 bytes, x ~ U(-1, 1)
    (seed 1); the absmax / per-tensor quantizer also on N(0,1) with 0.1% x100
    outliers; FP16 -> INT8; SR quantize (seed 7, parity mode: the reference's
    mt19937_64 stream, so FP64 + twist bound -- reported against HBM all the
    same).  Every kernel is CUDA-graph timed over rotating copies (cold L2)."""
    pk = peaks()
    bw = pk["hbm_gbs"]
    rows = []
    sizes = sizes or [1 << k for k in range(16, 31)]
    gen = torch.Generator(device="cuda").manual_seed(1)
    for nbytes in sizes:
        n = nbytes // 4
        per = max(1, min(64, -(-2 * L2_BYTES // nbytes)))
        xs = [torch.rand(n, device="cuda", generator=gen) * 2 - 1 for _ in range(per)]
        xo = torch.randn(n, device="cuda", generator=gen)
        idx = torch.randint(0, n, (max(1, n // 1000),), device="cuda", generator=gen)
        xo[idx] *= 100.0
        xos = [xo] + [xo.clone() for _ in range(per - 1)]
        x16 = [x.half() for x in xs]
        rowsn = max(1, n // 1024)
        qs = [torch.empty(n, dtype=torch.int8, device="cuda") for _ in range(per)]
        hs = [torch.empty(n, dtype=torch.float16, device="cuda") for _ in range(per)]
        sc = torch.tensor([0.01], device="cuda")
        cases = {
            "absmax": (lambda k: (lambda: ops.absmax(xs[k])), 4),
            "absmax_outliers": (lambda k: (lambda: ops.absmax(xos[k])), 4),
            "quantize_per_tensor": (lambda k: (lambda: ops.quantize_per_tensor(
                xs[k].view(rowsn, -1), out=qs[k].view(rowsn, -1))), 5),
            "quantize_per_tensor_outliers": (lambda k: (lambda: ops.quantize_per_tensor(
                xos[k].view(rowsn, -1), out=qs[k].view(rowsn, -1))), 5),
            "quantize_with_scale": (lambda k: (lambda: ops.quantize_with_scale(xs[k], sc)), 5),
            "quantize_f16_with_scale": (lambda k: (lambda: ops.quantize_with_scale(x16[k], sc)), 3),
            "quantize_per_channel": (lambda k: (lambda: ops.quantize_per_channel(xs[k].view(rowsn, -1))), 5),
            "dequantize": (lambda k: (lambda: ops.dequantize_per_tensor(qs[k], sc)), 5),
            "cast_f32_f16": (lambda k: (lambda: ops.cast(xs[k], torch.float16, out=hs[k])), 6),
            "tensor_stats": (lambda k: (lambda: ops.tensor_stats(xs[k])), 4),
        }
        for name, (mk, bpe) in cases.items():
            us, l2 = rotating_graph_us(mk, n * bpe, max_copies=per)
            gbs = n * bpe / (us * 1e-6) / 1e9
            rows.append({"kernel": name, "bytes_in": nbytes, "n": n, "us": us, "alg_bytes_per_elem": bpe,
                         "gbs": gbs, "frac_hbm": gbs / bw, "l2": l2, "timing": "cuda-graph, rotating copies"})
            print(f"{name:30s} {nbytes/2**20:9.3f} MiB {us:10.2f} us {gbs:8.1f} GB/s  frac={gbs/bw:.3f} {l2}",
                  flush=True)
        # SR quantize (parity mode): eager (its jump-ahead workspace is not capturable),
        # launches queued behind a device spin.
        if nbytes <= (1 << 28):
            t = spin_time_ms(lambda: ops.quantize_sr(xs[0], sc, 7))
            gbs = n * 5 / (t * 1e-3) / 1e9
            rows.append({"kernel": "quantize_sr_mt19937", "bytes_in": nbytes, "n": n, "us": t * 1e3,
                         "alg_bytes_per_elem": 5, "gbs": gbs, "frac_hbm": gbs / bw,
                         "melem_per_s": n / (t * 1e-3) / 1e6, "l2": "warm",
                         "timing": "eager behind a device spin", "bound": "FP64 SR + mt19937_64 twist"})
            print(f"{'quantize_sr_mt19937':30s} {nbytes/2**20:9.3f} MiB {t*1e3:10.2f} us {gbs:8.1f} GB/s "
                  f"({n / (t * 1e-3) / 1e6:.0f} Melem/s)", flush=True)
        del xs, xos, x16, qs, hs
        torch.cuda.empty_cache()
    results["sweep"] = rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--gemm", action="store_true")
    ap.add_argument("--conv", action="store_true")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    res: dict = {"peaks": peaks()}
    everything = not (args.gemm or args.sweep or args.conv)
    if args.gemm or everything:
        gemm_bench(res)
    if args.conv or everything:
        conv_bench(res)
    if args.sweep or everything:
        sweep_bench(res)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
