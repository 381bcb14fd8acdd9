"""In-step GEMM throughput (bench.gemm_durations: events around each GEMM launch
inside a captured copy of the step) for an A/B of a GEMM switch.

    python tools/gemm_in_step.py [--plan mixed] [--dual 1,0]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2407_02327_b200 import ops  # noqa: E402
from paper_2407_02327_b200.qlinear import FP16, INT8  # noqa: E402
from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, mixed_plan, uniform_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default="mixed")
    ap.add_argument("--dual", default="1,0")
    args = ap.parse_args()
    cfg = BertConfig()
    for rep in range(2):
        for d in args.dual.split(","):
            ops.set_dual_issue(d == "1")
            torch.manual_seed(0)
            m = BertEncoderStack(cfg).cuda()
            m.apply_plan({"mixed": mixed_plan(cfg), "int8": uniform_plan(cfg, INT8),
                          "fp16": uniform_plan(cfg, FP16)}[args.plan])
            st = TrainStep(m, batch=32, graph=True)
            st.tokens.random_(0, cfg.vocab)
            st.capture(warmup=3)
            kern, _ = bench.gemm_durations(st, torch, ops)
            print(f"rep {rep} dual={d} " + " ".join(
                f"{k}: {v['flops'] / v['ms'] / 1e9:.0f} TF/s ({v['ms']:.3f} ms, {v['launches']})"
                for k, v in sorted(kern.items())), flush=True)
            del st, m
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
