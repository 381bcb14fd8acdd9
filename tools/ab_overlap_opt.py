"""A/B the graphed BERT-base step on one GPU: AdamW once after the backward vs
bucket-wise on the comm stream as each gradient bucket becomes final."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, mixed_plan  # noqa: E402


def step_ms(overlap, steps=50):
    cfg = BertConfig()
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(mixed_plan(cfg))
    st = TrainStep(m, batch=32, graph=True, overlap_opt=overlap)
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=3)
    for _ in range(5):
        st()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        st()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


for ov in (False, True, False, True):
    print(f"overlap_opt={ov} step_ms={step_ms(ov):.3f}", flush=True)
