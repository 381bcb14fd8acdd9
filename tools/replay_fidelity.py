"""Replayer fidelity on B200 (PAPER.md:691-719 reports
<5% error): profile the BERT-base step on this GPU into a ProfileBundle, let the
UNMODIFIED reference replayer (oracle/_ref) predict the iteration time of a plan,
and compare with the measured CUDA-graph step of the same plan.

    python tools/replay_fidelity.py --out gpurun_out/fidelity.json
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.cpu_ref import RefLib  # noqa: E402  (test/measurement infrastructure)
from paper_2407_02327_b200.profiler import (bert_graph, build_bundle, collect_tensor_stats,  # noqa: E402
                                            measure_cast_samples, measure_op_costs)
from paper_2407_02327_b200.qlinear import FP16, INT8  # noqa: E402
from paper_2407_02327_b200.train_step import (BertConfig, BertEncoderStack, TrainStep,  # noqa: E402
                                              mixed_plan, uniform_plan)


def measured_step_ms(cfg, batch, plan, steps=20):
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(plan)
    st = TrainStep(m, batch=batch, graph=True)
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=3)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        st()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    del st, m
    torch.cuda.empty_cache()
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/fidelity.json")
    ap.add_argument("--bundle", default="gpurun_out/bert_base_b200_bundle.json")
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--batch", type=int, default=32)
    args = ap.parse_args()
    cfg = BertConfig(layers=args.layers)
    model = BertEncoderStack(cfg).cuda()
    model.apply_plan({})
    stats = collect_tensor_stats(model, args.batch, 3)
    del model
    costs = measure_op_costs(cfg, args.batch, reps=10)
    casts = measure_cast_samples(reps=10)
    graph = bert_graph(cfg, args.batch)
    devices = [{"id": "b200", "is_inference": True, "mem_capacity_bytes": 183_000_000_000}]
    bundle = build_bundle(graph, costs, casts, stats, devices)
    with open(args.bundle, "w") as f:
        json.dump(bundle, f)
    ref = RefLib()
    plans = {"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8), "fp16": uniform_plan(cfg, FP16),
             "fp32": {}}
    rows = {}
    for name, plan in plans.items():
        pred_ns = ref.replay_bundle(args.bundle, {"per_device": {"b200": plan}})
        meas = measured_step_ms(cfg, args.batch, plan)
        rows[name] = {"predicted_ms": pred_ns / 1e6, "measured_ms": meas,
                      "error": (pred_ns / 1e6 - meas) / meas}
        print(name, rows[name], flush=True)
    with open(args.out, "w") as f:
        json.dump({"config": {"layers": args.layers, "batch": args.batch, "seq": cfg.seq},
                   "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
