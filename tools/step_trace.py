"""Measured-step trace of the graphed BERT-base train step.

Runs the bench's step (CUDA graph replay) under the CUPTI kernel tracer
(torch.profiler, no nsys on the box) and writes
  * a Chrome trace in the reference replayer's format (replayer.cpp:126-148:
    {"traceEvents": [{name, ph "X", ts/dur in us, pid = device, tid}], "displayTimeUnit": "ms"}),
    one tid per CUDA stream, so the measured step opens in the same viewer as the
    replayer's predicted timeline;
  * a per-kernel summary (device time per step, launches per step, share) and the
    step span / busy / idle time, as JSON.

    python tools/step_trace.py --out gpurun_out/step_trace [--plan mixed] [--steps 5]
"""
import argparse
import collections
import gzip
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200.qlinear import FP16, INT8  # noqa: E402
from paper_2407_02327_b200.train_step import (BertConfig, BertEncoderStack, TrainStep,  # noqa: E402
                                              mixed_plan, uniform_plan)


def short(name: str) -> str:
    for pre in ("void ", "(anonymous namespace)::", "<unnamed>::", "qsb::", "at::native::"):
        name = name.replace(pre, "")
    return name.split("(")[0][:80]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/step_trace")
    ap.add_argument("--plan", default="mixed", choices=["mixed", "int8", "fp16", "fp32"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--no-fused", action="store_true")
    ap.add_argument("--no-pdl", action="store_true",
                    help="launch without programmatic dependent launch, so each kernel's traced duration "
                         "is its own (with PDL a kernel starts early and waits in griddepcontrol.wait)")
    args = ap.parse_args()
    if args.no_pdl:
        from paper_2407_02327_b200 import _lib
        _lib.call("qsync_gemm_set_pdl", 0)
    cfg = BertConfig()
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    plan = {"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8), "fp16": uniform_plan(cfg, FP16),
            "fp32": {}}[args.plan]
    m.apply_plan(plan)
    st = TrainStep(m, batch=args.batch, graph=True, fused=not args.no_fused)
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=3)
    for _ in range(5):
        st()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            st()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern = []
    for e in evs:
        tr = e.time_range
        kern.append((tr.start, tr.end, e.name, getattr(e, "device_resource_id", 0)))
    kern.sort()
    if not kern:
        raise SystemExit("no kernels traced")
    t0 = kern[0][0]
    # Chrome trace in the replayer's event format (times in us).
    events = [{"name": short(n), "ph": "X", "ts": (s - t0), "dur": (e - s), "pid": "b200",
               "tid": int(sid)} for s, e, n, sid in kern]
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with gzip.open(args.out + ".trace.json.gz", "wt") as f:
        json.dump({"traceEvents": events, "displayTimeUnit": "ms"}, f)
    # Busy time = union of kernel intervals (streams overlap).
    busy, cur_s, cur_e = 0.0, None, None
    for s, e, _, _ in kern:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    busy += cur_e - cur_s
    span = kern[-1][1] - kern[0][0]
    per = collections.defaultdict(lambda: [0.0, 0])
    for s, e, n, _ in kern:
        per[short(n)][0] += e - s
        per[short(n)][1] += 1
    tot = sum(v[0] for v in per.values())
    rows = sorted(per.items(), key=lambda kv: -kv[1][0])
    summary = {
        "plan": args.plan, "fused": not args.no_fused, "batch": args.batch, "steps": args.steps,
        "step_span_us": span / args.steps, "step_busy_us": busy / args.steps,
        "step_idle_us": (span - busy) / args.steps, "kernel_sum_us": tot / args.steps,
        "kernels": [{"kernel": k, "us_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps,
                     "share": v[0] / tot} for k, v in rows],
    }
    with open(args.out + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "kernels"}))
    for r in summary["kernels"][:40]:
        print(f"{r['us_per_step']:9.1f} us {r['launches_per_step']:6.1f}x {100 * r['share']:5.1f}%  {r['kernel']}")


if __name__ == "__main__":
    main()
