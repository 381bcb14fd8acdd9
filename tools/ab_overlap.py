"""A/B the graphed BERT-base step with / without the wgrad side stream."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, mixed_plan  # noqa: E402


def step_ms(overlap, steps=30):
    cfg = BertConfig()
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    m.apply_plan(mixed_plan(cfg))
    st = TrainStep(m, batch=32, graph=True, overlap_wgrad=overlap)
    st.tokens.random_(0, cfg.vocab)
    st.capture(warmup=3)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        loss = st()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps, float(loss)


for ov in (True, False, True, False):
    ms, l = step_ms(ov)
    print(f"overlap={ov} step_ms={ms:.3f} loss={l:.5f}", flush=True)
