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

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.cpu_ref import RefLib  # noqa: E402  (test/measurement infrastructure)
from paper_2407_02327_b200.profiler import (bert_graph, build_bundle, collect_tensor_stats,  # noqa: E402
                                            graph_step_ms, measure_cast_samples, measure_comm_slots,
                                            measure_fused_cast_samples, measure_fused_costs, measure_op_costs,
                                            measured_op_trace, net_weight_casts)
from paper_2407_02327_b200.qlinear import FP16, INT8  # noqa: E402
from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, mixed_plan, uniform_plan  # noqa: E402


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
    graph = bert_graph(cfg, args.batch)
    devices = [{"id": "b200", "is_inference": True, "mem_capacity_bytes": 183_000_000_000}]
    # Two bundles: the fused implementation the train step runs (operator regions of
    # the fused step, conversions as the marginal cost of the fused producers) and
    # the per-operator implementation (each op's GEMMs alone, standalone cast kernels).
    fused_casts = measure_fused_cast_samples(cfg)
    raw_costs = net_weight_casts(cfg, measure_fused_costs(cfg, args.batch, reps=5, calibrate=False), fused_casts)
    cal_costs = net_weight_casts(cfg, measure_fused_costs(cfg, args.batch, reps=5, calibrate=True), fused_casts)
    diag = measure_fused_costs.last_diag
    # Measured gradient-exchange slots (C ABI NCCL all-reduce; one rank on this box).
    comm = {"b200": measure_comm_slots(cfg, args.batch)}
    bundles = {
        "fused": build_bundle(graph, cal_costs, fused_casts, stats, devices, comm=comm),
        "fused_uncalibrated": build_bundle(graph, raw_costs, fused_casts, stats, devices, comm=comm),
        "per_op": build_bundle(graph, measure_op_costs(cfg, args.batch, reps=10),
                               measure_cast_samples(reps=10), stats, devices),
    }
    ref = RefLib()
    plans = {"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8), "fp16": uniform_plan(cfg, FP16),
             "fp32": {}}
    measured = {name: graph_step_ms(cfg, args.batch, plan) for name, plan in plans.items()}
    out = {"config": {"layers": args.layers, "batch": args.batch, "seq": cfg.seq,
                      "measured": "CUDA-graph train step (wgrad side stream, optimizer included)"}}
    for kind, bundle in bundles.items():
        path = args.bundle.replace(".json", f"_{kind}.json")
        with open(path, "w") as f:
            json.dump(bundle, f)
        rows = {}
        for name, plan in plans.items():
            pred_ns = ref.replay_bundle(path, {"per_device": {"b200": plan}})
            meas = measured[name]
            rows[name] = {"predicted_ms": pred_ns / 1e6, "measured_ms": meas,
                          "error": (pred_ns / 1e6 - meas) / meas}
            print(kind, name, rows[name], flush=True)
        out["rows" if kind == "fused" else f"rows_{kind}_bundle"] = rows
    out["calibration"] = diag
    out["comm_slots"] = comm["b200"]
    # Measured vs predicted operator-level traces of the mixed plan, same event ids
    # (replayer.cpp:126-148): the measured eager single-stream step against the
    # uncalibrated fused bundle (built from the same eager regions).
    import gzip
    meas = measured_op_trace(cfg, args.batch, plans["mixed"], "b200")
    pred = ref.replay_trace(args.bundle.replace(".json", "_fused_uncalibrated.json"),
                            {"per_device": {"b200": plans["mixed"]}})
    base = args.out[:-5] if args.out.endswith(".json") else args.out
    for tag, tr in (("measured", meas), ("predicted", pred)):
        with gzip.open(f"{base}_{tag}_mixed.trace.json.gz", "wt") as f:
            json.dump(tr, f)

    def by_id(tr):
        d = {}
        for e in tr["traceEvents"]:
            d[e["name"]] = d.get(e["name"], 0.0) + e["dur"]
        return d
    m_id, p_id = by_id(meas), by_id(pred)
    common = sorted(set(m_id) & set(p_id))
    out["trace_diff_mixed"] = {
        "ids_measured": len(m_id), "ids_predicted": len(p_id), "ids_common": len(common),
        "only_measured": sorted(set(m_id) - set(p_id)), "only_predicted": sorted(set(p_id) - set(m_id)),
        "sum_us_measured": sum(m_id[k] for k in common), "sum_us_predicted": sum(p_id[k] for k in common),
        "worst": sorted(({"id": k, "measured_us": m_id[k], "predicted_us": p_id[k]} for k in common),
                        key=lambda r: -abs(r["measured_us"] - r["predicted_us"]))[:10],
    }
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
