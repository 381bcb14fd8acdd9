"""Backward GEMM pairs of one BERT-base layer (dgrad on the critical path, wgrad
into the FP32 main_grad) at batch 32 x 128 tokens, CUDA-graph timed: each GEMM
alone, the pair back-to-back on one stream, and the pair on two streams (as the
train step runs them), with optional grid caps -- how much of the pair's time is
fixed cost and SM contention rather than tensor-core work.

    python tools/bwd_pair_bench.py [--caps 0:0,96:52]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import _lib, ops  # noqa: E402

T, H, F = 4096, 768, 3072
PEAK = 1.65e15


def graph_us(fns, streams, n=20, reps=5):
    """fns[i] enqueued on streams[i] (None = capture stream), joined each rep."""
    main = torch.cuda.Stream()
    main.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(main):
        for f in fns:
            f()
    torch.cuda.current_stream().wait_stream(main)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        for _ in range(n):
            if any(streams):  # fork before either GEMM is enqueued: the two run concurrently
                side.wait_stream(cur)
            for f, s in zip(fns, streams):
                if s:
                    with torch.cuda.stream(side):
                        f()
                else:
                    f()
            if any(streams):
                cur.wait_stream(side)
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


def with_cap(fn, cap):
    def run():
        if cap:
            _lib.call("qsync_gemm_set_max_ctas", cap)
        fn()
        if cap:
            _lib.call("qsync_gemm_set_max_ctas", 0)
    return run


def pairs():
    for nm, (N, K) in {"qkv": (3 * H, H), "o": (H, H), "ff1": (F, H), "ff2": (H, F)}.items():
        dy = torch.randn(T, N, device="cuda").half()
        w = torch.randn(N, K, device="cuda").half()
        x = torch.randn(T, K, device="cuda").half()
        acc = nm in ("qkv", "ff1")  # these dgrads reduce-add into the residual gradient (FP32)
        dx = torch.zeros(T, K, device="cuda", dtype=torch.float32 if acc else torch.float16)
        dw = torch.zeros(N, K, device="cuda")
        dgrad = lambda dy=dy, w=w, dx=dx, acc=acc: ops.gemm_f16(dy, w, out=dx, accumulate=acc, b_mn=True)  # noqa: E731
        wgrad = lambda dy=dy, x=x, dw=dw: ops.gemm_f16(dy, x, out=dw, accumulate=True, a_mn=True, b_mn=True)  # noqa: E731
        yield nm, dgrad, wgrad, 2.0 * T * N * K


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--caps", default="0:0,96:52,74:74,112:36")
    args = ap.parse_args()
    caps = [tuple(int(c) for c in v.split(":")) for v in args.caps.split(",")]
    print(f"{'pair':5s} {'ideal':>6s} {'dgrad':>6s} {'wgrad':>6s} {'seq':>6s} " +
          " ".join(f"{'2s ' + str(d) + ':' + str(w):>10s}" for d, w in caps))
    tot = {}
    for nm, dg, wg, fl in pairs():
        t_d = graph_us([dg], [False])
        t_w = graph_us([wg], [False])
        t_s = graph_us([dg, wg], [False, False])
        row = [t_d, t_w, t_s]
        for d, w in caps:
            row.append(graph_us([with_cap(dg, d), with_cap(wg, w)], [False, True]))
        for i, v in enumerate(row):
            tot[i] = tot.get(i, 0.0) + v
        print(f"{nm:5s} {2 * fl / PEAK * 1e6:6.1f} " + " ".join(f"{v:6.1f}" for v in row[:3]) + " " +
              " ".join(f"{v:10.1f}" for v in row[3:]), flush=True)
    print("sum   " + " " * 7 + " ".join(f"{tot[i]:6.1f}" for i in range(3)) + " " +
          " ".join(f"{tot[i]:10.1f}" for i in range(3, len(tot))))


if __name__ == "__main__":
    main()
