"""A/B the graphed BERT-base step over the side-stream wgrad GEMM grid cap."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200 import fused  # noqa: E402
from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, mixed_plan  # noqa: E402


def step_ms(cap, steps=30):
    cfg = BertConfig()
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(mixed_plan(cfg))
    st = TrainStep(m, batch=32, graph=True)
    fused.WGRAD_CTAS = cap  # after TrainStep, which sets its default (2/3 of the SMs)
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=3)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        st()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


for cap in [int(c) for c in (sys.argv[1:] or ["0", "64", "80", "98", "112", "128", "98"])]:
    print(f"wgrad cap={cap:4d} step_ms={step_ms(cap):.3f}", flush=True)
