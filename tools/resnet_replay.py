"""Config 3 in the planner's world: profile ResNet-50 (224^2, batch 64) on this B200
into a ProfileBundle (profiler_resnet), let the UNMODIFIED reference planner plan it
under a memory cap and the reference replayer predict each plan's iteration time,
and measure the same plans' forward+backward on the model (resnet.ResNet50).

    python tools/resnet_replay.py --out gpurun_out/rn50_replay.json
"""
import argparse
import gzip
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.cpu_ref import RefLib  # noqa: E402  (test/measurement infrastructure)
from paper_2407_02327_b200.profiler import default_cap  # noqa: E402
from paper_2407_02327_b200.profiler_resnet import profile_resnet50  # noqa: E402
from paper_2407_02327_b200.qlinear import FP16, FP32, INT8  # noqa: E402
from paper_2407_02327_b200.resnet import ResNet50, conv_specs  # noqa: E402


def step_ms(model, batch, plan, reps=5):
    """Device time of one forward+backward (launches queued behind a device spin)."""
    model.apply_plan(plan)
    img = torch.randn(batch, 224, 224, 3, device="cuda")
    lab = torch.randint(0, 1000, (batch,), device="cuda")

    def run():
        model.zero_grad(set_to_none=True)
        model(img, lab).backward()
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(400_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/rn50_replay.json")
    ap.add_argument("--bundle", default="gpurun_out/r2_resnet50_b200_bundle.json.gz")
    ap.add_argument("--batch", type=int, default=64)
    args = ap.parse_args()
    b = profile_resnet50(args.batch)
    b["devices"] = [{"id": "b200", "is_inference": True, "mem_capacity_bytes": 183_000_000_000}]
    with gzip.open(args.bundle, "wt") as f:
        json.dump(b, f)
    plain = args.bundle[:-3]
    with open(plain, "w") as f:
        json.dump(b, f)
    ref = RefLib()
    convs = [s[0] for s in conv_specs(1)]
    plans = {"fp32": {}, "int8": {n: INT8 for n in convs + ["fc"]},
             "fp16": {n: FP16 for n in convs + ["fc"]}}
    cap = default_cap(b["graph"], b["op_costs"], 0.75)
    rep = ref.plan_bundle(plain, 1, args.batch, 50, "b200", cap)
    plans["planner_cap75"] = {k: v for k, v in rep["devices"]["b200"].items() if v != FP32}
    model = ResNet50().cuda()
    rows = {}
    for name, plan in plans.items():
        full = {n["id"]: plan.get(n["id"], FP32) for n in b["graph"]["nodes"]}
        pred = ref.replay_bundle(plain, {"per_device": {"b200": full}}) / 1e6
        meas = step_ms(model, args.batch, plan)
        rows[name] = {"predicted_ms": pred, "measured_fwd_bwd_ms": meas, "error": pred / meas - 1,
                      "ops_int8": sum(v == INT8 for v in plan.values()),
                      "ops_fp16": sum(v == FP16 for v in plan.values())}
        print(name, rows[name], flush=True)
    os.remove(plain)
    out = {"workload": f"ResNet-50 224^2 batch {args.batch}, synthetic images", "cap_bytes": cap,
           "planner_memory_ok": rep["memory_ok"], "plans": rows,
           "note": "measured = eager forward+backward (no optimizer; max-pool/mean/CE unmodelled "
                   "in the graph); predicted = reference replayer makespan on the measured bundle"}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
