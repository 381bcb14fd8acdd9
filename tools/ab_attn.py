"""A/B the graphed BERT-base step over the attention-core implementations
(0 mma.sync, 1 tcgen05, 2 tcgen05 backward at 2 CTAs / SM):
    python tools/ab_attn.py [impl ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200._lib import call  # noqa: E402
from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, mixed_plan  # noqa: E402


def step_ms(tc, steps=50):
    call("qsync_attention_set_impl", tc)
    cfg = BertConfig()
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(mixed_plan(cfg))
    st = TrainStep(m, batch=32, graph=True)
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=3)
    for _ in range(10):
        st()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        st()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


for tc in [int(a) for a in (sys.argv[1:] or ["2", "1", "2", "1", "0"])]:
    print(f"attn_tc={tc} step_ms={step_ms(tc):.3f}", flush=True)
