"""Device time of the fused AdamW step (k_adamw) over BERT-base's parameters at
the bench's mixed plan, CUDA-graph timed (back-to-back updates), and its HBM
fraction by the algorithmic bytes (28 B/param + 2 B per planned weight for the
FP16 copy + 1 B for the INT8 copy).

    python tools/opt_bench.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_kernels import graph_time_us, peaks  # noqa: E402
from paper_2407_02327_b200.fused import FusedAdamW  # noqa: E402
from paper_2407_02327_b200.qlinear import FP16, INT8  # noqa: E402
from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, FlatGrads, mixed_plan  # noqa: E402


def main():
    cfg = BertConfig()
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(mixed_plan(cfg))
    params = list(m.parameters())
    FlatGrads(params)
    opt = FusedAdamW(params)
    opt.attach(m.qlinears().values())
    n = sum(p.numel() for p in params)
    extra = sum(q.weight.numel() * (2 + (1 if q.precision == INT8 else 0))
                for q in m.qlinears().values() if q.precision in (INT8, FP16))
    alg = 28 * n + extra
    us = graph_time_us(opt.step, n=10, reps=5)
    gbs = alg / (us * 1e-6) / 1e9
    out = {"params": n, "alg_bytes": alg, "us": us, "gbs": gbs, "frac_hbm": gbs / peaks()["hbm_gbs"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
