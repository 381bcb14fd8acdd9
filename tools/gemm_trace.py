"""Per-CTA phase timeline of the tcgen05 GEMM at the BERT-base step shapes
(the "measure, don't guess" step before changing the GEMM's scheduling).

    tools/build_variant.sh /tmp/libtrace.so -DQSB_GEMM_TRACE
    QSYNC_B200_LIB=/tmp/libtrace.so python tools/gemm_trace.py [--json out.json]

For every CTA the kernel records (gemm.cu, QSB_GEMM_TRACE): entry, end of the
prologue, and per work unit the producer's first load, the MMA thread's
accumulator-free / first-stage-full / last-commit times and the epilogue's
accumulator-full / last-store times.  Printed: medians over CTAs, in us.
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import _lib, ops  # noqa: E402

T, H, F = 4096, 768, 3072


def cases():
    out = {}
    for nm, (M, N, K) in {"qkv": (T, 3 * H, H), "o": (T, H, H), "ff1": (T, F, H), "ff2": (T, H, F)}.items():
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
        sa = torch.tensor([0.01], device="cuda")
        sb = torch.rand(N, device="cuda") * 0.01
        c = torch.empty((M, N), device="cuda")
        out[f"s8_{nm}"] = (lambda a=a, b=b, sa=sa, sb=sb, c=c: ops.gemm_s8(a, b, sa, sb, out=c), 2.0 * M * N * K)
    # FP16: forward FF1 (FP16 out), dgrad FF1 (B MN-major), wgrad FF1 (both MN-major, FP32 accumulate)
    a = torch.randn(T, H, device="cuda").half()
    w = torch.randn(F, H, device="cuda").half()
    c16 = torch.empty(T, F, device="cuda", dtype=torch.float16)
    out["f16_ff1_fwd"] = (lambda: ops.gemm_f16(a, w, out=c16), 2.0 * T * F * H)
    dy = torch.randn(T, F, device="cuda").half()
    dx = torch.empty(T, H, device="cuda", dtype=torch.float16)
    out["f16_ff1_dgrad"] = (lambda: ops.gemm_f16(dy, w, out=dx, b_mn=True), 2.0 * T * F * H)
    dw = torch.zeros(F, H, device="cuda")
    out["f16_ff1_wgrad"] = (lambda: ops.gemm_f16(dy, a, out=dw, accumulate=True, a_mn=True, b_mn=True),
                            2.0 * T * F * H)
    aq = torch.randn(T, H, device="cuda").half()
    wq = torch.randn(3 * H, H, device="cuda").half()
    cq = torch.empty(T, 3 * H, device="cuda", dtype=torch.float16)
    out["f16_qkv_fwd"] = (lambda: ops.gemm_f16(aq, wq, out=cq), 2.0 * T * 3 * H * H)
    dyq = torch.randn(T, 3 * H, device="cuda").half()
    out["f16_qkv_dgrad"] = (lambda: ops.gemm_f16(dyq, wq, out=aq, b_mn=True), 2.0 * T * 3 * H * H)
    return out


def analyse(buf: torch.Tensor, grid: int) -> dict:
    t = buf.view(-1, 72)[:grid].cpu().tolist()
    rows = [r for r in t if r[1]]
    if not rows:
        return {}
    freq = statistics.median((r[3] - r[1]) / max(1, (r[4] - r[0])) for r in rows)  # cycles per ns
    gt0 = min(r[0] for r in rows)

    def us(c):
        return c / freq / 1e3
    res = {"ctas": len(rows), "ghz": freq, "span_us": (max(r[4] for r in rows) - gt0) / 1e3,
           "entry_skew_us": (max(r[0] for r in rows) - gt0) / 1e3,
           "prologue_us": statistics.median(us(r[2] - r[1]) for r in rows),
           "cta_busy_us": statistics.median(us(r[3] - r[1]) for r in rows)}
    res["epi_warp2_us"] = {k: statistics.median(us(r[i]) for r in rows)
                           for k, i in (("tmem_ld", 5), ("math", 6), ("staging_wait", 7), ("store", 71))}
    units = []
    for k in range(8):
        ev = [r[8 + 8 * k: 14 + 8 * k] for r in rows if r[8 + 8 * k + 3]]
        if not ev:
            break
        base = {id(e): None for e in ev}
        del base
        units.append({
            "ctas": len(ev),
            "first_load_us": statistics.median(us(e[0] - r[1]) for e, r in zip(ev, rows)),
            "acc_free_us": statistics.median(us(e[1] - r[1]) for e, r in zip(ev, rows)),
            "first_full_us": statistics.median(us(e[2] - r[1]) for e, r in zip(ev, rows)),
            "last_commit_us": statistics.median(us(e[3] - r[1]) for e, r in zip(ev, rows)),
            "epi_start_us": statistics.median(us(e[4] - r[1]) for e, r in zip(ev, rows)),
            "epi_end_us": statistics.median(us(e[5] - r[1]) for e, r in zip(ev, rows)),
        })
    res["units"] = units
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--modes", default="0", help="comma list of isolation modes (trace build): 0 full, "
                    "1 no epilogue math/stores, 2 MMA only (no loads), 4 loads only (no MMAs, single CTA)")
    ap.add_argument("--only", default="")
    ap.add_argument("--streamk", type=int, default=-1, help="-1 never (default), 0 cost model, 1 always")
    ap.add_argument("--variants", default="0:0", help="comma list of cta:tile_n overrides, e.g. 0:0,2:256,2:128")
    args = ap.parse_args()
    ops.set_streamk(args.streamk)
    buf = torch.zeros(1024 * 72, dtype=torch.int64, device="cuda")
    out = {}
    variants = [tuple(int(x) for x in v.split(":")) for v in args.variants.split(",")]
    modes = [int(m) for m in args.modes.split(",")]
    todo = [(f"{name}[cta{c},bn{b}]" if (c, b) != (0, 0) else name, fn, flops, c, b, m)
            for name, (fn, flops) in cases().items() for c, b in variants for m in modes
            if args.only in name]
    for name, fn, flops, cta, bn, mode in todo:
        if mode:
            name += f"[mode{mode}]"
        _lib.call("qsync_gemm_debug_epilogue", mode)
        ops.force_cta(cta)
        ops.force_tile_n(bn)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        plain_us = e0.elapsed_time(e1) * 1e3
        buf.zero_()
        _lib.call("qsync_gemm_trace_buffer", buf.data_ptr())
        fn()
        torch.cuda.synchronize()
        _lib.call("qsync_gemm_trace_buffer", None)
        r = analyse(buf, 1024)
        ops.force_cta(0)
        ops.force_tile_n(0)
        _lib.call("qsync_gemm_debug_epilogue", 0)
        r["event_us"] = plain_us
        r["tflops_event"] = flops / (plain_us * 1e-6) / 1e12
        out[name] = r
        print(f"== {name}: event {plain_us:.1f} us ({r['tflops_event']:.0f} TF/s), span {r.get('span_us', 0):.1f} us,"
              f" ctas {r.get('ctas')}, entry skew {r.get('entry_skew_us', 0):.2f}, prologue {r.get('prologue_us', 0):.2f},"
              f" busy {r.get('cta_busy_us', 0):.2f} us @ {r.get('ghz', 0):.2f} GHz")
        print("   epilogue warp 2 totals (us):", {k: round(v, 2) for k, v in r.get("epi_warp2_us", {}).items()})
        for i, u in enumerate(r.get("units", [])):
            print(f"   unit {i} ({u['ctas']} CTAs): load {u['first_load_us']:.2f} accfree {u['acc_free_us']:.2f} "
                  f"full {u['first_full_us']:.2f} commit {u['last_commit_us']:.2f} | epi {u['epi_start_us']:.2f}"
                  f" -> {u['epi_end_us']:.2f}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
