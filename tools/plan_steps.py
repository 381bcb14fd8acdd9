"""Graphed BERT-base train-step time per uniform plan (INT8 / FP16 / FP32) and
the mixed bench plan, batch 32 (profiler.graph_step_ms).

    python tools/plan_steps.py [--json out.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200.profiler import graph_step_ms  # noqa: E402
from paper_2407_02327_b200.qlinear import FP16, INT8  # noqa: E402
from paper_2407_02327_b200.train_step import BertConfig, mixed_plan, uniform_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--plans", default="mixed,int8,fp16,fp32")
    args = ap.parse_args()
    cfg = BertConfig()
    plans = {"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8), "fp16": uniform_plan(cfg, FP16), "fp32": {}}
    out = {}
    for name in args.plans.split(","):
        out[name] = graph_step_ms(cfg, 32, plans[name])
        print(f"{name:6s} {out[name]:8.3f} ms", flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
